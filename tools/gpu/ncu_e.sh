#!/bin/bash
# ncu --set full of the K=512 forward GEMM at config E (pop 64), eager replay
PBRL_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none -k regex:"k_tc_gemm" --launch-skip 2 --launch-count 2 \
  -o gpurun_out/full_E -f python bench.py --config E --pop 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_e.log 2>&1
tail -1 gpurun_out/ncu_e.log
