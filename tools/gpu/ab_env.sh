#!/bin/bash
# A/B of an environment toggle on the default bench (alternating runs), after the parity tests
# named in $TESTS.  usage: TESTS="tests/x.py" bash tools/gpu/ab_env.sh VAR=1 [precision]
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -q -x -p no:cacheprovider 2>&1 | tail -4; fi
for i in 1 2 3; do
  for E in "" "$1"; do
    v=$(env $E timeout 200 python bench.py --precision ${2:-bf16} --steps 300 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))")
    echo "[$E] $v"
  done
done
