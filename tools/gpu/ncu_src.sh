#!/bin/bash
# source-level warp-stall sampling (densest interval) of one kernel launch, eager bf16 bench run
PBRL_NO_GRAPH=1 timeout 600 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 \
  --clock-control none --import-source on -k regex:"$1" --launch-skip ${2:-0} --launch-count 1 \
  -o gpurun_out/src -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_src.log 2>&1
tail -1 gpurun_out/ncu_src.log
