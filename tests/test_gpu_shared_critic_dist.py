"""Shared-critic TD3 sharded over two ranks: the per-step
critic-gradient all-reduce inside the library (pbrl_attach_comm) keeps one identical critic
replica per rank, and the result equals the single-process shared-critic population up to the
summation order of the critic gradient (the two shards' partial sums are added instead of one
running sum over all n*B rows): FFMA32 within 1e-5 relative; policies, steps and masks per shard."""
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from helpers import bits_equal

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("precision,tol", [("ffma32", 1e-5), ("bf16", 2e-2)])
def test_two_rank_shared_critic_equals_single_process(cuda, tmp_path, precision, tol):
    import paper_2206_08888_b200 as pb
    n_total, world = 8, 2
    port = _port()
    procs, outs = [], []
    for r in range(world):
        out = tmp_path / f"rank{r}.npz"
        outs.append(out)
        procs.append(subprocess.Popen(
            [sys.executable, str(ROOT / "tests" / "shared_critic_worker.py"), "--rank", str(r),
             "--world", str(world), "--port", str(port), "--out", str(out), "--n-total",
             str(n_total), "--precision", precision],
            stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    for p in procs:
        o, _ = p.communicate(timeout=300)
        assert p.returncode == 0, o[-3000:]
    st = pb.make_td3_state(n_total, 17, 6, [32, 32], 1.0, 5, mode="shared_critic",
                           precision=precision)
    hy = pb.Td3Hyper.defaults(n_total)
    gmask = [1 if m < n_total // 2 else 0 for m in range(n_total)]
    for i, b in enumerate(pb.make_synthetic_batches(4, n_total, 32, 17, 6, 6)):
        pb.td3_update_step(st, b, hy, policy_member_mask=gmask if i % 2 else None)
    z = [np.load(p) for p in outs]
    n = n_total // world

    def rel(a, b):
        a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
        return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))

    for net in ("critic1", "critic2", "critic1_target", "critic2_target"):
        assert bits_equal(z[0][f"net_{net}"], z[1][f"net_{net}"]), net  # identical replicas
        assert rel(z[0][f"net_{net}"], st.params(net)) < tol, net
    for r in range(world):
        for net in ("policy", "policy_target"):
            assert rel(z[r][f"net_{net}"], st.params(net)[r * n:(r + 1) * n]) < tol, (r, net)
    # the shard losses are partial sums of the whole population's critic loss
    full = np.stack(st.last_losses())
    tot = z[0]["losses"][0, 0] + z[1]["losses"][0, 0]
    assert abs(tot - full[0, 0]) <= 1e-5 * abs(full[0, 0])
