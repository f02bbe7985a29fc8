#!/bin/bash
# Round-2 profile of the bench command (LLaMA-8B 1F1B M32, 1 GPU), one timed stable step:
#  1. launch list (ncu gpu__time_duration, profiler range = the timed step)
#  2. ncu --set full of the roofline kernel (K1 pair GEMM, gate|up + SwiGLU epilogue)
#  3. ncu --set full of the masked dW (K3 row pairs) and of the flash attention fwd / bwd
mkdir -p gpurun_out
export PF_NCU_RANGE=1 PF_SKIP_CPU_BASELINE=1
B="python bench.py --steps 1 --warmup 3"
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2_bench_launches.csv $B > gpurun_out/r2_prof_launch.log 2>&1
tail -1 gpurun_out/r2_prof_launch.log | cut -c1-200
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  --kernel-name-base mangled -k regex:Li256ELb0ELi4EE -c 1 -o gpurun_out/r2_roofline -f $B > gpurun_out/r2_prof_roof.log 2>&1
tail -1 gpurun_out/r2_prof_roof.log | cut -c1-200
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:gemm_dw_rowpair -c 1 -o gpurun_out/r2_dw -f $B > gpurun_out/r2_prof_dw.log 2>&1
tail -1 gpurun_out/r2_prof_dw.log | cut -c1-200
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:flash_ -c 4 -o gpurun_out/r2_attn -f $B > gpurun_out/r2_prof_attn.log 2>&1
tail -1 gpurun_out/r2_prof_attn.log | cut -c1-200
ls -la gpurun_out | tail -8
