#!/bin/bash
# Round-2 end-of-round profile of the bench command (LLaMA-8B 1F1B M=32, 1 GPU): the launch list of one
# whole timed step (ncu serialises ~16.7k launches: ~45 min), then --set full of the attention kernels.
mkdir -p gpurun_out
export PF_NCU_RANGE=1 PF_SKIP_CPU_BASELINE=1
B="python bench.py --steps 1 --warmup 3"
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:flash_ -c 4 -o gpurun_out/r2b_attn -f $B > gpurun_out/r2b_prof_attn.log 2>&1
tail -1 gpurun_out/r2b_prof_attn.log | cut -c1-200
timeout 3300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2b_bench_launches.csv $B > gpurun_out/r2b_prof_launch.log 2>&1
tail -1 gpurun_out/r2b_prof_launch.log | cut -c1-200
ls -la gpurun_out | tail -4
