set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_features_gpu.py -x -q 2>&1 | tail -15
for v in pp db; do DYNRAD_K6=$v TAG=$v timeout 300 python tools/ab_k6.py; done
for v in pp db; do DYNRAD_K6=$v TAG=$v timeout 300 python tools/ab_k6.py; done
timeout 900 python -m pytest tests/test_mask_gpu.py -x -q -k "production" 2>&1 | tail -15
