#!/bin/bash
# launch list + ncu --set full of the output-layer backward and batch pack kernels (bf16, config D)
mkdir -p gpurun_out
PBRL_NO_GRAPH=1 timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches_${TAG:-x}.csv python bench.py --steps 4 --warmup 3 \
  --no-cpu-baseline --no-e2e > /dev/null 2>&1
PBRL_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"${KRE:-k_out_backward|k_pack_batch}" --launch-skip ${SKIP:-10} --launch-count ${CNT:-8} \
  -o gpurun_out/full_${TAG:-x} -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_full_${TAG:-x}.log 2>&1
tail -2 gpurun_out/ncu_full_${TAG:-x}.log
python profiles/summarize.py ${TAG:-x} gpurun_out/launches_${TAG:-x}.csv gpurun_out/full_${TAG:-x}.ncu-rep > /dev/null 2>&1
mkdir -p gpurun_out/profiles_box
cp profiles/${TAG:-x}_*.md gpurun_out/profiles_box/ 2>/dev/null
ls -la gpurun_out/*.ncu-rep
