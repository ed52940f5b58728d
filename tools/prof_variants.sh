#!/bin/bash
# one ncu --set full capture of the stage-(d) kernel per library variant
mkdir -p gpurun_out
for so in "$@"; do
  n=$(basename $so .so)
  QUICK=1 DYNRAD_LIB=$PWD/$so timeout 300 ncu --set full --clock-control none --import-source on -k regex:bsfa -s 2 -c 1 -o gpurun_out/prof_$n python tools/attn_perf.py > gpurun_out/prof_$n.log 2>&1
  echo "$n rc=$?"
done
