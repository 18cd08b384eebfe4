#!/bin/bash
# Adam kernel A/B in the graph: per-kernel durations from the CUPTI timeline; args: env settings
mkdir -p gpurun_out
for E in "$@"; do
  for R in 1.0 0.0001; do
    T=ab_$(echo "$E" | tr -c 'A-Za-z0-9' '_')_$R
    env $E timeout 120 python tools/gpu/timeline.py $T $R > /dev/null 2>&1
    rm -f gpurun_out/trace_$T.json
    echo "== [$E] $R"; python tools/gpu/tl_show.py $T 6 1 | grep -E "adam|^ +[0-9.]+ +[0-9.]+ +[0-9.]+ s[0-9]+ $|next"
  done
done
