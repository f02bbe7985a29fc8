#!/bin/bash
# usage: bash tools/prof_launch.sh <tag> [ratio]   -> gpurun_out/launches_<tag>.csv
tag=${1:-run}; ratio=${2:-0.8}
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${tag}.csv python tools/profile_step.py --model llama-1b --ratio ${ratio} \
  > gpurun_out/prof_launch_${tag}.log 2>&1
tail -2 gpurun_out/prof_launch_${tag}.log
