timeout 900 python -m pytest tests/test_mask_gpu.py tests/test_select_ops_gpu.py -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 5 --warmup 3 --no-lib --no-dense --no-cpu --no-e2e --no-rebuild > gpurun_out/score_bench.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/score_bench.json').read().strip().splitlines()[-1]); h=d['hunyuan_dynamic']; print(h['value'], h['mask_equals_reference_golden'], json.dumps(h['stages_ms']['per_stage_device_ms']), json.dumps({k:v['frac'] for k,v in h['scoring_roofline'].items()}))"
