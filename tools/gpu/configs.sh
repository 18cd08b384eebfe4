#!/bin/bash
# throughput of the other BASELINE configs (parity-test cases, not bench lines): B (pop 1 vs 10),
# C (SAC pop 32), E (TD3 3x512, batch 1024, pop 1..256)
run() { timeout 300 python bench.py --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$*', round(d['value']), 'agent-updates/s', round(d['ms_per_step']*1e3,1), 'us/step')" ; }
run --config B --pop 1
run --config B --pop 10
run --config C
run --config C --precision tf32
STEPS=20 run --config E --pop 1
STEPS=20 run --config E --pop 8
STEPS=20 run --config E --pop 64
STEPS=10 run --config E --pop 256
