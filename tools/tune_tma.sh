#!/bin/bash
# Tuning sweep of the TMA plan knobs on a C5-shaped slab (results: gpurun_out/tune_*.log).
A="python bench.py --config c5 --dims 128,128,128,32 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-compare-fp64"
for v in "256 64 2 3" "256 64 3 3" "256 12 2 3" "128 64 2 2" "256 64 2 2" "256 64 2 4" "256 24 2 3"; do
  set -- $v
  SLDG_TMA_W=$1 SLDG_TMA_TSUB=$2 SLDG_TMA_SDIV=$3 SLDG_TMA_D0DIV=$4 timeout 200 $A > gpurun_out/tune2_$1_$2_$3_$4.log 2>&1
done
