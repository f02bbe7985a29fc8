#!/bin/bash
# ncu --set full of the fused SwiGLU-backward pair GEMM (1B shape) -> gpurun_out/dswiglu.ncu-rep
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:Li256ELb1ELi5EE -s 3 -c 1 -o gpurun_out/dswiglu -f python tools/swiglu_bench.py > gpurun_out/dswiglu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:Li256ELb0ELi4EE -s 3 -c 1 -o gpurun_out/swiglu_fwd -f python tools/swiglu_bench.py >> gpurun_out/dswiglu.log 2>&1
tail -3 gpurun_out/dswiglu.log
