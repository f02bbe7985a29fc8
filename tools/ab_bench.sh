#!/bin/bash
# A/B of bench.py on one box: each arg is "ENV=VAL ..." (or "-" for defaults); prints value lines.
for cfg in "$@"; do
  if [ "$cfg" = "-" ]; then envs=""; else envs="$cfg"; fi
  echo "== $cfg"
  env $envs timeout 240 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value', d['value'], 'nofreeze', d['nofreeze']['value'], 'ms', d['ms_per_step'], 'clk', d['clocks'])"
done
