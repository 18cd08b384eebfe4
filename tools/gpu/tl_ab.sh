#!/bin/bash
# fire-step (policy_delay_ratio 1) CUPTI timelines under several environment settings
mkdir -p gpurun_out
R=${RATIO:-1.0}
for E in "$@"; do
  T=tl_$(echo "$E" | tr -c 'A-Za-z0-9' '_')_$R
  env $E timeout 120 python tools/gpu/timeline.py $T $R > /dev/null 2>&1
  rm -f gpurun_out/trace_$T.json
  echo "== [$E] $R"; python tools/gpu/tl_show.py $T 6 1
done
