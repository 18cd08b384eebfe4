#!/bin/bash
# Round evidence on one B200: GPU tests, bench lines (tf32 + bf16), ncu launch lists and one
# `ncu --set full` capture of the forward GEMM launches of one step per precision.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for P in tf32 bf16; do
  timeout 300 python bench.py --precision $P > gpurun_out/bench_$P.json 2> gpurun_out/bench_$P.err
  head -c 400 gpurun_out/bench_$P.json; echo
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$P.csv python bench.py --precision $P --steps 4 --warmup 3 \
    --no-cpu-baseline --no-e2e > /dev/null 2>&1
  PBRL_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm \
    --launch-skip 60 --launch-count 10 -o gpurun_out/full_gemm_$P -f python bench.py --precision $P \
    --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$P.log 2>&1
  tail -2 gpurun_out/ncu_full_$P.log
  PBRL_NO_GRAPH=1 timeout 300 ncu --set full --clock-control none -k regex:k_adam --launch-skip 6 --launch-count 2 \
    -o gpurun_out/full_adam_$P -f python bench.py --precision $P --steps 2 --warmup 3 \
    --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1
tail -1 gpurun_out/bench_ref.json | head -c 300; echo
ls gpurun_out
