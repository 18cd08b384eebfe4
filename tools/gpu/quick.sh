#!/bin/bash
# fast GPU check: full GPU test suite + short bench per precision
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; tail -1 gpurun_out/q_pytest.log
for P in tf32 bf16; do
  timeout 200 python bench.py --precision $P --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/q_$P.json 2>gpurun_out/q_$P.err
  python -c "import json; d=json.load(open('gpurun_out/q_$P.json')); print('$P', round(d['value']), round(d['ms_per_step']*1e3,1), {k: round(v['ms'],3) for k,v in d['profile'].items()})" || tail -3 gpurun_out/q_$P.err
done
tail -1 gpurun_out/q_pytest.log
