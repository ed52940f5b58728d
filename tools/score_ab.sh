#!/bin/bash
# Interleaved A/B of the dynamic-mask build (tools/dyn_stats.py) between the
# in-tree libdynrad.so and variants/$1.so, plus one ncu launch list each.
mkdir -p gpurun_out
for r in 1 2 3; do
  echo "== new";  timeout 200 python tools/dyn_stats.py | grep hunyuan | grep -o "rechecked_pairs[^,]*\|build ms.*"
  echo "== $1"; DYNRAD_LIB=$PWD/variants/$1.so timeout 200 python tools/dyn_stats.py | grep hunyuan | grep -o "rechecked_pairs[^,]*\|build ms.*"
done
for v in new $1; do
  echo "== ncu $v"
  if [ $v = new ]; then L=; else L=DYNRAD_LIB=$PWD/variants/$v.so; fi
  env $L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"score_kernel|recheck_kernel|apply|job_stats" -c 5 --csv python tools/dyn_stats.py 2>/dev/null | grep -E "score_kernel|recheck_kernel|apply|job_stats" | awk -F'","' '{print substr($5,1,40), $NF}'
done
