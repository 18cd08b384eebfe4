"""TEST HELPER (launched by tests/test_gpu_dist_native.py): one rank of a sharded population on
the shared GPU, PBT exchange through the library (pbrl_pbt_evolve_sharded) over a host transport
(torch.distributed gloo).  Writes its shard's final state to --out."""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def scenario(pb, st, hy, batches, pbt, rng, evolve, off, n, k=2):
    """K updates, returns recorded by global id, evolve, K more updates (shared by the sharded
    ranks and the single-process reference run)."""
    upd = pb.td3_update_step if isinstance(st, pb.Td3State) else pb.sac_update_step
    for i in range(k):
        upd(st, batches[i], hy)
    for m in range(n):
        g = off + m
        for j in range(1 + g % 3):
            pbt.record_return(m, float((g * 7 + j * 3) % 11) - 0.5 * j)
    plan = evolve()
    for i in range(k, 2 * k):
        upd(st, batches[i], hy)
    return plan


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int)
    ap.add_argument("--world", type=int)
    ap.add_argument("--port", type=int)
    ap.add_argument("--algo", default="td3")
    ap.add_argument("--precision", default="ffma32")
    ap.add_argument("--n-total", type=int, default=12)
    ap.add_argument("--unready", action="store_true")
    ap.add_argument("--out")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(a.port)
    dist.init_process_group("gloo", rank=a.rank, world_size=a.world)
    import paper_2206_08888_b200 as pb
    from paper_2206_08888_b200.dist import Comm, NativeShardedPBT
    from helpers import SAC_NETS, TD3_NETS

    n = a.n_total // a.world
    off = a.rank * n
    make = pb.make_td3_state if a.algo == "td3" else pb.make_sac_state
    st = make(n, 5, 2, [32, 32], 1.0, 60, precision=a.precision, device=0, member_offset=off,
              n_global=a.n_total)
    hy = pb.Td3Hyper.defaults(n) if a.algo == "td3" else pb.SacHyper.defaults(n, 2)
    gb = pb.make_synthetic_batches(4, a.n_total, 32, 5, 2, 9)
    batches = [pb.TransitionBatch(*[x[off:off + n].contiguous() for x in
                                    (b.s, b.a, b.r, b.s2, b.done)]) for b in gb]
    pbt = pb.PBTState(n)
    rng = pb.RngSequence(1, 2, "kDonorChoice")
    comm = Comm.host(device=0)
    sharded = NativeShardedPBT(st, hy, comm)
    if a.unready:  # rank 1 leaves its member 0 unscored: every rank must raise together
        for m in range(n):
            if not (a.rank == 1 and m == 0):
                pbt.record_return(m, 1.0)
        try:
            sharded.evolve(pbt, rng)
            res = "no error"
        except pb.NotReadyError as e:
            res = "NotReadyError: " + str(e)
        Path(a.out).write_text(res)
        dist.destroy_process_group()
        return
    plan = scenario(pb, st, hy, batches, pbt, rng, lambda: sharded.evolve(pbt, rng), off, n)
    nets = TD3_NETS if a.algo == "td3" else SAC_NETS
    out = {f"net_{k}": st.params(k) for k in nets}
    for f in hy.FIELDS:
        out[f"hyper_{f}"] = np.asarray(getattr(hy, f))
    out["replaced"] = np.asarray(plan.replaced)
    out["donors"] = np.asarray(plan.donors)
    out["rng_next"] = np.asarray([rng.next], np.uint64)
    out["exchange_ms"] = np.asarray(list(sharded.last_exchange_ms.values()))
    out["ring_lens"] = np.asarray([len(r) for r in pbt.returns])
    for k in ("policy", "critic1", "critic2"):
        out[f"adam_t_{k}"] = np.asarray([st.adam(k, i)[2] for i in range(n)])
    np.savez(a.out, **out)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
