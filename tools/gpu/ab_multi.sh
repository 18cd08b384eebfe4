#!/bin/bash
# bench under several environment settings, alternating (3 rounds); args: settings ("" = none)
for i in 1 2 3; do
  for E in "$@"; do
    v=$(env $E timeout 200 python bench.py --precision ${PREC:-bf16} --steps 300 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))")
    echo "[$E] $v"
  done
done
