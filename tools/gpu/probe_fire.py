"""Graph-mode step time split by whether the policies fire (config D, BF16): every step fires
(policy_delay_ratio 1) vs none in the timed window (ratio 1e-4) vs the default 0.5."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2206_08888_b200 as pb
from paper_2206_08888_b200 import _lib

n, B = 80, 256
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
st = pb.make_td3_state(n, 17, 6, [256, 256], 1.0, 7, precision=prec, device=0)
gb = pb.make_synthetic_batches(8, n, B, 17, 6, 7, device=torch.device("cuda", 0))
structs = [_lib.Batch(*[x.data_ptr() for x in (b.s, b.a, b.r, b.s2, b.done)]) for b in gb]
ls = st.lib_stream()
for ratio in (1.0, 1e-4, 0.5, 1.0, 1e-4, 0.5):
    hy = pb.Td3Hyper.defaults(n)
    hy.policy_delay_ratio = [ratio] * n
    st._sync_hyper(hy)

    def run(i):
        arr = (_lib.Batch * 1)(structs[i % len(structs)])
        _lib.call("pbrl_update_batches_device", st.handle, arr, 1, B, None)
    for i in range(20):
        run(i)
    st.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 400
    a.record(ls)
    for i in range(K):
        run(i)
    b.record(ls)
    b.synchronize()
    print(f"{prec} ratio {ratio}: {a.elapsed_time(b) / K * 1e3:.1f} us/step", flush=True)
