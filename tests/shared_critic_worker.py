"""TEST HELPER (launched by tests/test_gpu_shared_critic_dist.py): one rank of a shared-critic
TD3 population sharded over ranks that share the GPU.  Every step sums the critic gradients over
the ranks (pbrl_attach_comm; host transport = torch.distributed gloo), so each rank's critic
replica takes the step of the unsharded population.  Writes the shard's state to --out."""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int)
    ap.add_argument("--world", type=int)
    ap.add_argument("--port", type=int)
    ap.add_argument("--n-total", type=int, default=8)
    ap.add_argument("--precision", default="ffma32")
    ap.add_argument("--out")
    a = ap.parse_args()
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(a.port)
    dist.init_process_group("gloo", rank=a.rank, world_size=a.world)
    import paper_2206_08888_b200 as pb
    from paper_2206_08888_b200.dist import Comm

    n = a.n_total // a.world
    off = a.rank * n
    st = pb.make_td3_state(n, 17, 6, [32, 32], 1.0, 5, mode="shared_critic",
                           precision=a.precision, member_offset=off, n_global=a.n_total)
    comm = Comm.host(device=0)
    st.attach_comm(comm)
    hy = pb.Td3Hyper.defaults(n)
    gb = pb.make_synthetic_batches(4, a.n_total, 32, 17, 6, 6)
    gmask = [1 if m < a.n_total // 2 else 0 for m in range(a.n_total)]  # CEM-RL train mask
    for i, b in enumerate(gb):
        sb = pb.TransitionBatch(*[x[off:off + n].contiguous() for x in
                                  (b.s, b.a, b.r, b.s2, b.done)])
        mask = gmask[off:off + n] if i % 2 else None
        pb.td3_update_step(st, sb, hy, policy_member_mask=mask)
    out = {f"net_{k}": st.params(k) for k in ("policy", "policy_target", "critic1", "critic2",
                                               "critic1_target", "critic2_target")}
    out["losses"] = np.stack(st.last_losses())
    np.savez(a.out, **out)
    st.attach_comm(None)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
