#!/bin/bash
# time every library variant under variants/ on the Wan stage-(d) workload
for so in variants/*.so; do
  echo "== $so"; DYNRAD_LIB=$PWD/$so timeout 120 python tools/attn_perf.py 2>&1 | head -1

done
