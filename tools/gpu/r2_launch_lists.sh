mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-lib --no-cpu --no-e2e --no-dense --no-rebuild > gpurun_out/launch_bench.log 2>&1
echo rc=$?
