mkdir -p gpurun_out
bash tools/score_ab.sh $1 > gpurun_out/score_ab.log 2>&1
timeout 900 python -m pytest tests/test_mask_gpu.py tests/test_select_ops_gpu.py -x -q > gpurun_out/score3_tests.log 2>&1
tail -3 gpurun_out/score3_tests.log
