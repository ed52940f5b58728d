DYNRAD_K6=ag timeout 600 python -m pytest tests/test_attention_gpu.py -x -q -k "bf16 or wan_shape or empty_row or host_pipeline or layer_host" 2>&1 | tail -3
DYNRAD_K6=ag timeout 600 python -m pytest tests/test_soft_attention_gpu.py -x -q 2>&1 | tail -2
for rep in 1 2; do
  for v in db ag; do DYNRAD_K6=$v TAG=$v timeout 300 python tools/ab_k6.py; done
done
