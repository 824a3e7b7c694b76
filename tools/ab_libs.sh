#!/bin/bash
# Interleaved A/B of library builds on one box: ab_libs.sh "<ab_time args>" libA libB ...
# (each build/lib_<name>.so, twice in alternation; output gpurun_out/ab_libs.log)
ARGS=$1; shift
for rep in 1 2; do
  for L in "$@"; do
    COMMDET_CUDA_LIB=build/lib_$L.so timeout 900 python tools/ab_time.py --tag $L.$rep $ARGS >> gpurun_out/ab_libs.log 2>&1
  done
done
