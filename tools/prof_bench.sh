#!/bin/bash
# Round profile of the bench command itself (1 GPU):
#  1. launch list of one timed stable step (ncu gpu__time_duration, profiler range = timed steps)
#  2. ncu --set full of the roofline kernel (K1 pair GEMM, gate|up + SwiGLU epilogue) inside the timed step
mkdir -p gpurun_out
PF_NCU_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/bench_launches.csv python bench.py --steps 1 --warmup 3 > gpurun_out/prof_bench_launch.log 2>&1
tail -2 gpurun_out/prof_bench_launch.log | cut -c1-300
PF_NCU_RANGE=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  --kernel-name-base mangled -k regex:Li256ELb0ELi4EE -c 2 -o gpurun_out/roofline -f \
  python bench.py --steps 1 --warmup 3 > gpurun_out/prof_bench_full.log 2>&1
tail -2 gpurun_out/prof_bench_full.log | cut -c1-300
ls -la gpurun_out | tail -5
