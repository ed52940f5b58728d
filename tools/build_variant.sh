#!/bin/bash
# build_variant.sh NAME "EXTRA nvcc flags" [SOURCE] -> variants/NAME.so
# Recompiles only capi.cu (stage d + CSR + C ABI) with the extra flags and
# links it with the already-built mask objects under build/.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_2604_20470_b200/csrc
B=$ROOT/paper_2604_20470_b200/build
mkdir -p $ROOT/variants $B/var
[ -f $B/mask_build.o ] && [ -f $B/mask_score_sm100.o ] || make -s -C $C >/dev/null
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -I$ROOT/include -I$C --expt-relaxed-constexpr -Xptxas -v $2 -c -o $B/var/$1.o ${3:-$C/capi.cu} 2> $B/var/$1.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/variants/$1.so $B/var/$1.o $(ls $B/*.o | grep -v "/capi.o")
grep -A1 "pp_kernelILi128" $B/var/$1.log | grep -o "Used [0-9]* registers.*" | head -1
