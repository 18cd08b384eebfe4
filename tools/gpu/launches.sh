#!/bin/bash
# eager-mode ncu launch list of a short bf16 bench (per-kernel durations)
PBRL_NO_GRAPH=1 timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches_${1:-bf16}.csv python bench.py --precision ${1:-bf16} --steps 4 --warmup 3 \
  --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -q 2>&1 | tail -2
