# A/B of the experimental ppc stage-(d) kernel (tools/experiments/k6_variants/
# attn_sm100_ppc.cu, wired as DYNRAD_K6=ppc while measured) against db:
# parity subset, Wan config-3 and dense-mask timings, HBM traffic per launch.
mkdir -p gpurun_out
DYNRAD_K6=ppc timeout 300 python -m pytest -q -x -p no:cacheprovider tests/test_attention_gpu.py -k "bf16 or wan_shape or empty_row or host_pipeline" 2>&1 | tail -2
for v in db ppc; do
  DYNRAD_K6=$v TAG=$v timeout 120 python tools/ab_k6.py
  DENSE=1 DYNRAD_K6=$v TAG=dense_$v timeout 120 python tools/ab_k6.py
  DYNRAD_K6=$v timeout 300 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:bsfa -c 1 python tools/ab_k6.py 2>/dev/null | grep -E "dram__|lts__|tensor"
done
