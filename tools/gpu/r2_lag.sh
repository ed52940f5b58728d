DYNRAD_DB_LAG=1 timeout 600 python -m pytest tests/test_attention_gpu.py -x -q -k "bf16 or wan_shape" 2>&1 | tail -2
for rep in 1 2 3; do
for lag in 0 1; do
  DYNRAD_DB_LAG=$lag timeout 600 python bench.py --steps 20 --warmup 5 --no-dynamic --no-lib --no-dense --no-cpu --no-e2e --no-rebuild > gpurun_out/lag$lag.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/lag$lag.json').read().strip().splitlines()[-1]); print('lag=$lag', round(d['value'],3), round(d['roofline']['kernel_ms'],3), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'], d['gpu_launches'])"
done; done
