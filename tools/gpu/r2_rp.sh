DYNRAD_K6=rp timeout 600 python -m pytest tests/test_attention_gpu.py -x -q -k "bf16 or wan_shape or empty_row or host_pipeline" 2>&1 | tail -3
for rep in 1 2; do
  for v in db rp; do DYNRAD_K6=$v TAG=$v timeout 300 python tools/ab_k6.py; done
done
for v in rp db; do DYNRAD_K6=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-lib --no-dense --no-cpu --no-e2e --no-rebuild > gpurun_out/rp_$v.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/rp_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['roofline']['achieved'], d['hunyuan_dynamic']['value'], d['hunyuan_dynamic']['roofline']['achieved'], d['hunyuan_dynamic']['roofline']['kernel'])"; done
