"""The native PBT exchange (pbrl_pbt_evolve_sharded) with two ranks sharing the
one GPU: each rank owns half of a population, the exchange runs inside the library over a host
transport (gloo through torch.distributed, Comm.host), and the result must equal -- bit for bit --
the single-process pbt_evolve_trainer (evolve.hpp:169-213) run on the whole population: the
plan, the RngSequence position, every member's weights after further updates, the re-drawn
hypers, the optimiser resets and the cleared return rings.  Plus the single-rank NCCL
transport (Comm.nccl) on the same path."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from helpers import SAC_NETS, TD3_NETS, bits_equal

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))


@pytest.fixture(scope="module")
def pb(cuda):
    import paper_2206_08888_b200 as pb
    return pb


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_ranks(tmp_path, world, extra):
    port = _port()
    procs, outs = [], []
    for r in range(world):
        out = tmp_path / f"rank{r}.npz"
        outs.append(out)
        procs.append(subprocess.Popen(
            [sys.executable, str(ROOT / "tests" / "dist_native_worker.py"), "--rank", str(r),
             "--world", str(world), "--port", str(port), "--out", str(out)] + extra,
            stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    for p in procs:
        out, _ = p.communicate(timeout=300)
        assert p.returncode == 0, out[-3000:]
    return outs


def _single_process(pb, algo, n_total, precision):
    from dist_native_worker import scenario
    make = pb.make_td3_state if algo == "td3" else pb.make_sac_state
    st = make(n_total, 5, 2, [32, 32], 1.0, 60, precision=precision)
    hy = pb.Td3Hyper.defaults(n_total) if algo == "td3" else pb.SacHyper.defaults(n_total, 2)
    batches = pb.make_synthetic_batches(4, n_total, 32, 5, 2, 9)
    pbt = pb.PBTState(n_total)
    rng = pb.RngSequence(1, 2, "kDonorChoice")
    prior = pb.Td3Prior() if algo == "td3" else pb.SacPrior()
    plan = scenario(pb, st, hy, batches, pbt, rng,
                    lambda: pb.pbt_evolve_trainer(pbt, st, hy, prior, rng), 0, n_total)
    return st, hy, plan, rng, pbt


@pytest.mark.parametrize("algo,precision", [("td3", "ffma32"), ("sac", "ffma32"),
                                            ("td3", "bf16")])
def test_two_ranks_equal_single_process(pb, tmp_path, algo, precision):
    n_total, world = 12, 2
    outs = _run_ranks(tmp_path, world, ["--algo", algo, "--precision", precision,
                                        "--n-total", str(n_total)])
    st, hy, plan, rng, pbt = _single_process(pb, algo, n_total, precision)
    n = n_total // world
    cross = sum(1 for d, s in zip(plan.replaced, plan.donors) if d // n != s // n)
    assert cross > 0, "scenario must exercise a cross-rank exploit copy"
    nets = TD3_NETS if algo == "td3" else SAC_NETS
    for r, path in enumerate(outs):
        z = np.load(path)
        assert z["replaced"].tolist() == plan.replaced
        assert z["donors"].tolist() == plan.donors
        assert int(z["rng_next"][0]) == rng.next
        sl = slice(r * n, (r + 1) * n)
        for net in nets:
            assert bits_equal(z[f"net_{net}"], st.params(net)[sl]), (r, net)
        for f in hy.FIELDS:
            assert np.array_equal(z[f"hyper_{f}"], np.asarray(getattr(hy, f))[sl]), (r, f)
        for k in ("policy", "critic1", "critic2"):
            want = [st.adam(k, i)[2] for i in range(r * n, (r + 1) * n)]
            assert z[f"adam_t_{k}"].tolist() == want, (r, k)
        assert z["ring_lens"].tolist() == [len(x) for x in pbt.returns[sl]]
        assert np.all(z["exchange_ms"] >= 0)


def test_not_ready_on_one_rank_raises_on_every_rank(pb, tmp_path):
    outs = _run_ranks(tmp_path, 2, ["--unready"])
    for path in outs:
        msg = Path(path).read_text()
        assert msg.startswith("NotReadyError") and "ranks not ready: 1" in msg, msg


def test_single_rank_nccl_transport_matches_trainer(pb, cuda):
    import torch.distributed as dist
    from paper_2206_08888_b200.dist import Comm, NativeShardedPBT
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        n = 10
        x = pb.make_td3_state(n, 5, 2, [16], 1.0, 60)
        y = pb.make_td3_state(n, 5, 2, [16], 1.0, 60)
        hx, hy_ = pb.Td3Hyper.defaults(n), pb.Td3Hyper.defaults(n)
        px, py = pb.PBTState(n), pb.PBTState(n)
        for m in range(n):
            px.record_return(m, float((m * 3) % 7))
            py.record_return(m, float((m * 3) % 7))
        rx, ry = pb.RngSequence(1, 2, "kDonorChoice"), pb.RngSequence(1, 2, "kDonorChoice")
        comm = Comm.nccl(device=0)
        assert comm.kind == "nccl"
        plan_x = NativeShardedPBT(x, hx, comm).evolve(px, rx)
        plan_y = pb.pbt_evolve_trainer(py, y, hy_, pb.Td3Prior(), ry)
        comm.close()
        assert plan_x.replaced == plan_y.replaced and plan_x.donors == plan_y.donors
        assert rx.next == ry.next
        for f in pb.Td3Hyper.FIELDS:
            assert getattr(hx, f) == getattr(hy_, f)
        for net in TD3_NETS:
            assert bits_equal(x.params(net), y.params(net))
    finally:
        dist.destroy_process_group()
