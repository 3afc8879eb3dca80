#!/bin/bash
# Quick register / spill check of one translation unit (no link):
#   tune/regs.sh trace.cu 'trace_kernelILi1ENS_22alpha_bits' [-DFOO]
SRC=$1; PAT=$2; shift 2
cd "$(dirname "$0")/../paper_1912_12786_b200/csrc"
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
  -prec-div=true -prec-sqrt=true -ftz=false -Xptxas -v -I ../../include "$@" -cubin -o /tmp/regs.cubin $SRC 2>&1 \
  | grep -A3 "$PAT" | grep -E "Compiling|spill|Used" | sed 's/ptxas info    : //'
