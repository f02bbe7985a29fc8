#!/bin/bash
# bench.py on each schedule (1 GPU): value / nofreeze / batch-vs-LP per schedule
mkdir -p gpurun_out
for sch in "$@"; do
  echo "== $sch"
  timeout 300 python bench.py --steps 4 --warmup 3 --schedule $sch > gpurun_out/sched_$sch.log 2>&1
  tail -1 gpurun_out/sched_$sch.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value', d['value'], 'nofreeze', d['nofreeze']['value'], 'speedup', d['freeze_speedup'], 'batch/lp', d['batch_vs_lp']['ratio'], 'plan', d['batch_vs_lp']['plan_makespan_base_ms'], d['batch_vs_lp']['plan_makespan_opt_ms'])" 2>/dev/null || tail -5 gpurun_out/sched_$sch.log
done
