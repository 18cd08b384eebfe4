#!/bin/bash
# Round evidence on one B200: GPU tests, bench lines (bf16 default + tf32), the reference arm,
# ncu launch lists (eager replay) and `ncu --set full` captures of the top kernels.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err; head -c 300 gpurun_out/bench_bf16.json; echo
timeout 300 python bench.py --precision tf32 --no-cpu-baseline > gpurun_out/bench_tf32.json 2> gpurun_out/bench_tf32.err; head -c 300 gpurun_out/bench_tf32.json; echo
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json | head -c 200; echo
for P in bf16 tf32; do
  PBRL_NO_GRAPH=1 timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$P.csv python bench.py --precision $P --steps 4 --warmup 3 \
    --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
# one full capture per top kernel class (bf16): fused forward, dW GEMM, dX GEMM, Adam, output backward
PBRL_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_mlp_fwd2|k_tc_gemm|k_adam|k_out_backward" --launch-skip 60 --launch-count 24 \
  -o gpurun_out/full_bf16 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_full_bf16.log 2>&1
tail -2 gpurun_out/ncu_full_bf16.log
ls gpurun_out
# summarise on the box (the .ncu-rep files would exceed the 64 MiB copy-back limit)
python profiles/summarize.py r1_final_bf16 gpurun_out/launches_bf16.csv gpurun_out/full_bf16.ncu-rep > /dev/null 2>&1
python profiles/summarize.py r1_final_tf32 gpurun_out/launches_tf32.csv > /dev/null 2>&1
mkdir -p gpurun_out/profiles_box
cp profiles/r1_final_bf16_*.md profiles/r1_final_tf32_*.md profiles/traffic_bf16_D.json gpurun_out/profiles_box/
rm -f gpurun_out/*.ncu-rep
