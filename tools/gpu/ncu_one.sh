#!/bin/bash
# ncu --set full of one kernel (regex $1, skip $2 launches) in an eager bf16 bench run
PBRL_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$1" \
  --launch-skip ${2:-0} --launch-count ${3:-1} -o gpurun_out/one -f python bench.py --steps 2 --warmup 3 \
  --no-cpu-baseline --no-e2e > gpurun_out/ncu_one.log 2>&1
tail -1 gpurun_out/ncu_one.log
