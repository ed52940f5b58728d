# Round-end validation: GPU tests, smoke, the default bench line, the
# reference arm and the ncu launch list of a short bench run.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/r2_bench_ref_final.json 2> gpurun_out/r2_bench_ref_final.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-lib --no-cpu --no-e2e --no-dense --no-rebuild > gpurun_out/launch_bench.log 2>&1; echo "ncu rc=$?"
