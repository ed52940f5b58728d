mkdir -p gpurun_out
s=$(date +%s); timeout 1800 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/ref_full.json 2> gpurun_out/ref_full.err; echo "ref rc=$? $(( $(date +%s) - s )) s"
s=$(date +%s); timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$? $(( $(date +%s) - s )) s"
tail -c 600 gpurun_out/bench_full.err
