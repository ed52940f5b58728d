mkdir -p gpurun_out
(python tools/cpu_reference_full.py gpurun_out/r2_cpu_reference_build_mask.json > gpurun_out/cpu_ref.log 2>&1 &)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsfa -s 1 -c 1 -o gpurun_out/r2_k6db_wan python tools/prof_layer.py wan > gpurun_out/ncu_wan.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bsfa -s 1 -c 1 -o gpurun_out/r2_k6rp_hunyuan python tools/prof_layer.py hunyuan > gpurun_out/ncu_hy.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_hunyuan.csv python tools/prof_layer.py hunyuan > /dev/null 2>&1
# wait for the CPU reference run
for i in $(seq 1 120); do
  if grep -q hunyuan_dynamic gpurun_out/cpu_ref.log 2>/dev/null; then break; fi
  sleep 10
done
cat gpurun_out/cpu_ref.log
