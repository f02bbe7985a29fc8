#!/bin/bash
# Raster group height on the LLaMA-8B N = 4096 GEMM shapes (standalone, same box).
cd $GRAFT_REPO_ROOT
for g in 0 4 8 16 4; do
  echo "== PF_GEMM_GROUP_M=$g (0: default)"
  if [ $g = 0 ]; then timeout 300 python tools/gemm_bench8b.py 2>&1 | tail -6; else PF_GEMM_GROUP_M=$g timeout 300 python tools/gemm_bench8b.py 2>&1 | tail -6; fi
done
