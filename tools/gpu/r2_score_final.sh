mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_kernel|recheck_kernel|apply_tiles|job_stats" -s 4 -c 5 -o gpurun_out/r2_score_final python tools/prof_layer.py hunyuan > gpurun_out/ncu_score_final.log 2>&1
tail -2 gpurun_out/ncu_score_final.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/dyn_stats.py > gpurun_out/r2_dyn_launches.csv 2>/dev/null
tail -1 gpurun_out/r2_dyn_launches.csv | cut -c1-200
