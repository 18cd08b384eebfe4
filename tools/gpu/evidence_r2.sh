#!/bin/bash
# Round-2 evidence at HEAD on one B200: GPU tests, bench lines (bf16 default, tf32, ffma32,
# configs B / C / E, 2 ranks, reference arm), ncu launch lists (eager replay) and `ncu --set full`
# captures of the top kernels, summarised into profiles/ on the box.
set -u
TAG=${TAG:-r2}
mkdir -p gpurun_out/profiles_box
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/${TAG}_bench_D_bf16.json 2> gpurun_out/${TAG}_bench_D_bf16.err; head -c 300 gpurun_out/${TAG}_bench_D_bf16.json; echo
timeout 300 python bench.py --precision tf32 --no-cpu-baseline > gpurun_out/${TAG}_bench_D_tf32.json 2>&1
timeout 300 python bench.py --precision ffma32 --no-cpu-baseline --steps 20 > gpurun_out/${TAG}_bench_D_ffma32.json 2>&1
timeout 300 python bench.py --config B --no-cpu-baseline > gpurun_out/${TAG}_bench_B.json 2>&1
timeout 300 python bench.py --config C --no-cpu-baseline > gpurun_out/${TAG}_bench_C.json 2>&1
for P in 1 8 64 256; do
  timeout 300 python bench.py --config E --pop $P --no-cpu-baseline --steps 20 --warmup 3 > gpurun_out/${TAG}_bench_E_$P.json 2>&1
done
timeout 300 python bench.py --gpus 2 --no-cpu-baseline > gpurun_out/${TAG}_bench_D_2ranks.json 2>&1
timeout 600 python bench.py --replay --no-cpu-baseline > gpurun_out/${TAG}_bench_D_replay.json 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2>&1
for P in bf16 tf32; do
  PBRL_NO_GRAPH=1 timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}_$P.csv python bench.py --precision $P --steps 4 --warmup 3 \
    --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
PBRL_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_mlp_fwd2|k_tc_gemm|k_adam|k_out_backward|k_pack_batch" --launch-skip 62 --launch-count 26 \
  -o gpurun_out/full_${TAG}_bf16 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_full_${TAG}.log
# graph-mode kernel timeline (CUPTI through torch.profiler): a fire step and a non-fire step
timeout 200 python tools/gpu/timeline.py ${TAG}_graph 0.5 > /dev/null 2>&1
{ echo "# ${TAG}: graph-mode kernel timeline, config D BF16 (CUPTI, tools/gpu/timeline.py)"; echo;
  echo "start / duration / end in us from the step's batch pack; sN = graph branch (stream id)"; echo;
  echo '```'; python tools/gpu/tl_show.py ${TAG}_graph 4 2; echo '```'; } > gpurun_out/profiles_box/${TAG}_graph_timeline.md
rm -f gpurun_out/trace_${TAG}_graph.json
python profiles/summarize.py ${TAG}_bf16 gpurun_out/launches_${TAG}_bf16.csv gpurun_out/full_${TAG}_bf16.ncu-rep > /dev/null 2>&1
python profiles/summarize.py ${TAG}_tf32 gpurun_out/launches_${TAG}_tf32.csv > /dev/null 2>&1
cp profiles/${TAG}_bf16_*.md profiles/${TAG}_tf32_*.md profiles/traffic_bf16_D.json gpurun_out/profiles_box/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
python - <<'PY'
import json, glob, os
tag = os.environ.get("TAG", "r2")
for f in sorted(glob.glob(f"gpurun_out/{tag}_bench_*.json")):
    try:
        d = [json.loads(l) for l in open(f) if l.startswith("{")][-1]
    except Exception as e:
        print(f, "ERR", open(f).read()[-300:]); continue
    print(f.split("/")[-1], round(d.get("value", 0)), "e2e", round((d.get("e2e") or {}).get("value", 0)),
          "ms", round(d.get("ms_per_step", 0) * 1e3, 1), "frac", round((d.get("step_roofline") or {}).get("frac", 0), 3),
          "vec", (d.get("vectorization_overhead") or {}).get("ratio"))
PY
