mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 2 -c 2 -o gpurun_out/r2_score_hunyuan python tools/prof_layer.py hunyuan > gpurun_out/ncu_score.log 2>&1
tail -3 gpurun_out/ncu_score.log
