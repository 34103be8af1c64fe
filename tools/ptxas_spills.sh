#!/bin/bash
# ptxas register / spill report of one csrc file (sm_100a): tools/ptxas_spills.sh sldg_sweep_tma.cu [regex]
cd "$(dirname "$0")/../paper_1603_07008_b200"
NCCL_INC=$(python -c "import nvidia.nccl as n; print(list(n.__path__)[0])")/include
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I../include -I"$NCCL_INC" -Xptxas -v -c -o /tmp/ptxas_spills.o "csrc/$1" 2>&1 |
  awk '/Compiling entry function/ {f=$0; sub(/.*function ./, "", f); sub(/. for .*/, "", f)}
       /spill stores/ {sp=$0} /Used [0-9]+ registers/ {r=$0; sub(/.*Used /, "", r); sub(/ registers.*/, "", r); print f, "regs=" r, sp}' |
  grep -E "${2:-.}" | sed -e 's/bytes stack frame, /stack /' -e 's/ bytes spill stores, / st /' -e 's/ bytes spill loads/ ld/'
