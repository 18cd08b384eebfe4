#!/bin/bash
# marginal cost of each launch class inside the replayed graph (diagnostics: results are not a
# valid update, only the step time is read)
for M in 0 1 2 4 8 16 32 63; do
  v=$(PBRL_SKIP_CLASSES=$M timeout 200 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1))")
  echo "skip mask $M: $v us/step"
done
