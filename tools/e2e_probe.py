import ctypes as C, sys, time, torch
sys.path.insert(0, '.')
import paper_2206_08888_b200 as pb
from paper_2206_08888_b200 import _lib
n, B = 80, 256
st = pb.make_td3_state(n, 17, 6, [256, 256], 1.0, 7, precision="bf16")
hy = pb.Td3Hyper.defaults(n); st._sync_hyper(hy)
gb = pb.make_synthetic_batches(10, n, B, 17, 6, 7, device=torch.device("cuda", 0))
hb = [[x.cpu().pin_memory() for x in (b.s, b.a, b.r, b.s2, b.done)] for b in gb]
hs = [_lib.Batch(*[x.data_ptr() for x in h]) for h in hb]
ds = [_lib.Batch(*[x.data_ptr() for x in (b.s, b.a, b.r, b.s2, b.done)]) for b in gb]
loss = torch.empty(50 * 3 * n, dtype=torch.float64).pin_memory()
lp = C.cast(loss.data_ptr(), _lib.f64p)
def run(KC, structs, with_loss, calls=10):
    arr = (_lib.Batch * KC)(*[structs[j % 10] for j in range(KC)])
    f = (lambda: _lib.call("pbrl_update_batches_losses", st.handle, arr, KC, B, None, lp)) if with_loss else (lambda: _lib.call("pbrl_update_batches", st.handle, arr, KC, B, None))
    f(); st.synchronize()
    t0 = time.perf_counter()
    for _ in range(calls): f()
    st.synchronize()
    dt = (time.perf_counter() - t0) / (calls * KC)
    return n / dt
for KC in (10, 50):
    print(KC, "host+loss %.0f" % run(KC, hs, True), "host nolos %.0f" % run(KC, hs, False), "dev+loss %.0f" % run(KC, ds, True), "dev nolos %.0f" % run(KC, ds, False))
