#!/bin/bash
# A/B of an environment toggle on the bf16 bench (3 alternating runs each)
for i in 1 2 3; do
  for E in "" "$1"; do
    v=$(env $E timeout 200 python bench.py --precision ${2:-bf16} --steps 300 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']))")
    echo "[$E] $v"
  done
done
