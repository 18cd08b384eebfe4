"""Graph-mode kernel timeline of config D steps through CUPTI (torch.profiler / kineto records
the kernels of graph launches one by one): writes gpurun_out/timeline_<tag>.json with
(name, stream, start_us, dur_us) per kernel.  args: tag [ratio] [precision] [pop] [batch]
[hidden, e.g. 512,512,512]"""
import json
import sys
import torch
sys.path.insert(0, ".")
import paper_2206_08888_b200 as pb
from paper_2206_08888_b200 import _lib

tag = sys.argv[1] if len(sys.argv) > 1 else "d"
ratio = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
prec = sys.argv[3] if len(sys.argv) > 3 else "bf16"
n = int(sys.argv[4]) if len(sys.argv) > 4 else 80
B = int(sys.argv[5]) if len(sys.argv) > 5 else 256
hidden = [int(h) for h in sys.argv[6].split(",")] if len(sys.argv) > 6 else [256, 256]
st = pb.make_td3_state(n, 17, 6, hidden, 1.0, 7, precision=prec, device=0)
hy = pb.Td3Hyper.defaults(n)
hy.policy_delay_ratio = [ratio] * n
st._sync_hyper(hy)
gb = pb.make_synthetic_batches(4 if n * B > 100000 else 8, n, B, 17, 6, 7, device=torch.device("cuda", 0))
structs = [_lib.Batch(*[x.data_ptr() for x in (b.s, b.a, b.r, b.s2, b.done)]) for b in gb]


def run(i, cnt=1):
    arr = (_lib.Batch * cnt)(*[structs[(i + j) % len(structs)] for j in range(cnt)])
    _lib.call("pbrl_update_batches_device", st.handle, arr, cnt, B, None)


for i in range(6 if n * B > 100000 else 30):
    run(i)
st.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    steps = 4 if n * B > 100000 else 12
    run(0, steps)  # one call: the packs after the first overlap the previous step's last Adam
    st.synchronize()
prof.export_chrome_trace(f"gpurun_out/trace_{tag}.json")
ev = json.load(open(f"gpurun_out/trace_{tag}.json"))["traceEvents"]
ks = [dict(name=e["name"], stream=e.get("args", {}).get("stream", e.get("tid")),
           start=float(e["ts"]), dur=float(e.get("dur", 0)))
      for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ks.sort(key=lambda k: k["start"])
t0 = ks[0]["start"] if ks else 0.0
for k in ks:
    k["start"] -= t0
json.dump(ks, open(f"gpurun_out/timeline_{tag}.json", "w"), indent=0)
print(len(ks), "kernels")
