timeout 600 python -m pytest tests/test_attention_gpu.py -x -q -k "layer_host or empty_row" 2>&1 | tail -5
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench1.err
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --gather --no-lib --no-dense --no-cpu --no-e2e > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench2 rc=$?"; tail -c 1500 gpurun_out/bench2.err
