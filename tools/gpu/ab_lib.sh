#!/bin/bash
# A/B of two builds of the library (paths $1, $2) on the bf16 bench, 3 alternating runs each
L=paper_2206_08888_b200/libpbrl_b200.so
for i in 1 2 3; do
  for V in "$1" "$2"; do
    cp "$V" $L
    v=$(timeout 200 python bench.py --precision ${3:-bf16} --steps 300 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']))")
    echo "[$V] $v"
  done
done
cp "$1" $L
