#!/bin/bash
# Round-2 bench lines on one B200: bench tests, default (config D BF16), TF32, FFMA32, configs
# B / C / E, --gpus 2 (ranks sharing the GPU), and the GPU parity printouts.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bench.py -q -p no:cacheprovider > gpurun_out/r2_bench_tests.log 2>&1; tail -3 gpurun_out/r2_bench_tests.log
timeout 300 python bench.py > gpurun_out/r2_bench_D_bf16.json 2> gpurun_out/r2_bench_D_bf16.err; head -c 400 gpurun_out/r2_bench_D_bf16.json; echo
timeout 300 python bench.py --precision tf32 --no-cpu-baseline > gpurun_out/r2_bench_D_tf32.json 2>&1
timeout 300 python bench.py --precision ffma32 --no-cpu-baseline --steps 20 > gpurun_out/r2_bench_D_ffma32.json 2>&1
timeout 300 python bench.py --config B --no-cpu-baseline > gpurun_out/r2_bench_B.json 2>&1
timeout 300 python bench.py --config C --no-cpu-baseline > gpurun_out/r2_bench_C.json 2>&1
for P in 1 8 64 256; do
  timeout 300 python bench.py --config E --pop $P --no-cpu-baseline --steps 20 --warmup 3 > gpurun_out/r2_bench_E_$P.json 2>&1
done
timeout 300 python bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r2_bench_D_2ranks.json 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.json 2>&1
timeout 600 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_bf16.py tests/test_gpu_tf32.py -q -s -p no:cacheprovider 2>&1 | grep -E "^[A-Z]_|passed|failed" > gpurun_out/r2_parity.log
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r2_bench_*.json")):
    try:
        d = [json.loads(l) for l in open(f) if l.startswith("{")][-1]
    except Exception as e:
        print(f, "ERR", open(f).read()[-300:]); continue
    pe = d.get("pbt_exchange") or {}
    print(f.split("/")[-1], round(d.get("value", 0)), "e2e", round((d.get("e2e") or {}).get("value", 0)),
          "ms", round(d.get("ms_per_step", 0) * 1e3, 1), "frac", round((d.get("step_roofline") or {}).get("frac", 0), 3),
          "pbt_ms", round(pe.get("ms", 0), 2), "vec", (d.get("vectorization_overhead") or {}).get("ratio"))
PY
cat gpurun_out/r2_parity.log
