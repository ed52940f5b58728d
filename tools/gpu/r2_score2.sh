mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mask_gpu.py tests/test_select_ops_gpu.py -x -q > gpurun_out/score2_tests.log 2>&1
tail -3 gpurun_out/score2_tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 2 -c 2 -o gpurun_out/r2_score2_hunyuan python tools/prof_layer.py hunyuan > gpurun_out/ncu_score2.log 2>&1
tail -3 gpurun_out/ncu_score2.log
