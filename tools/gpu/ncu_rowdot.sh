#!/bin/bash
# ncu --set full of the output-layer row-dot kernels at config E (pop 64), eager replay
mkdir -p gpurun_out
PBRL_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none -k regex:"k_fwd_rowdot" --launch-count 3 \
  -o gpurun_out/full_rowdot -f python bench.py --config E --pop 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_rowdot.log 2>&1
tail -1 gpurun_out/ncu_rowdot.log
ncu -i gpurun_out/full_rowdot.ncu-rep --page details --csv 2>/dev/null | grep -E '"(Duration|Registers Per Thread|Achieved Occupancy|Theoretical Occupancy|Memory Throughput|DRAM Throughput|Compute \(SM\) Throughput|Block Limit Registers|Block Limit Shared Mem|Executed Instructions|Waves Per SM|L2 Hit Rate|L1/TEX Hit Rate)"' | cut -d, -f5,13-16 | head -60
