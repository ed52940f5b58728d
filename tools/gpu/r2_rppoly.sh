for rep in 1 2; do
  for v in base rp01 rp11; do
    if [ $v = base ]; then LIB=""; else LIB="variants/$v.so"; fi
    env ${LIB:+DYNRAD_LIB=$LIB} DYNRAD_K6=rp timeout 600 python bench.py --steps 10 --warmup 3 --no-lib --no-dense --no-cpu --no-e2e --no-rebuild > gpurun_out/rpp_$v.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/rpp_$v.json').read().strip().splitlines()[-1]); h=d['hunyuan_dynamic']; print('$v', round(d['roofline']['kernel_ms'],3), round(d['roofline']['achieved'],1), round(h['roofline']['kernel_ms'],3), round(h['roofline']['achieved'],1))"
  done
done
