#!/bin/bash
# A/B on C3: wide forward GEMMs (gate|up, LM head) with every tile row in one raster group (weight read once).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
summ() { tail -1 $1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('value', d['value'], 'nofreeze', d['nofreeze']['value'], 'ms', d['ms_per_step'], 'roof', d['roofline']['achieved'], 'clk', d['clocks']['sm_mhz'])"; }
for v in 0 1 0 1; do
  echo "== FULLM=$v"; PF_GEMM_FULLM=$v PF_SKIP_CPU_BASELINE=1 timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/i_c3_$v.log 2>&1; summ gpurun_out/i_c3_$v.log
done
