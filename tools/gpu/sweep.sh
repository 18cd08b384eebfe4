#!/bin/bash
# quick A/B of bench configurations (diagnostics): precision x tile-width policy
mkdir -p gpurun_out
for P in tf32 bf16; do
  for BN in auto 256; do
    if [ "$BN" = auto ]; then unset PBRL_TC_BN; else export PBRL_TC_BN=$BN; fi
    v=$(timeout 200 python bench.py --precision $P --steps 200 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))")
    echo "$P BN=$BN: $v"
  done
done
unset PBRL_TC_BN
timeout 300 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_bf16.py -q 2>&1 | tail -2
