"""Print steps of a timeline_<tag>.json (tools/gpu/timeline.py): start / dur / end per kernel,
relative to each step's batch pack.  args: tag [first_step] [count]"""
import json
import re
import sys

tag = sys.argv[1]
j0 = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cnt = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ks = json.load(open(f"gpurun_out/timeline_{tag}.json"))


def short(n):
    n = re.sub(r"\(.*", "", n).replace("void ", "").replace("__nv_bfloat16", "bf16")
    return n.replace("unsigned int", "u32").replace("pbrl::", "")[:44]


starts = [i for i, k in enumerate(ks) if "pack_batch" in k["name"] or "replay_gather" in k["name"]]
for j in range(j0, min(j0 + cnt, len(starts) - 1)):
    s, e = starts[j], starts[j + 1]
    base = ks[s]["start"]
    for k in ks[s:e]:
        st = k["start"] - base
        print(f"{st:8.1f} {k['dur']:7.1f} {st + k['dur']:8.1f} s{k['stream']} {short(k['name'])}")
    print("--- next step at", round(ks[e]["start"] - base, 1))
