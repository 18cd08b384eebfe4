#!/bin/bash
PBRL_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 120 --csv \
  --log-file gpurun_out/launches_E.csv python bench.py --config E --pop ${POP:-64} --steps 2 --warmup 1 \
  --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/launches_E.csv
