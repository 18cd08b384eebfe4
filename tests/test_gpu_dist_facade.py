"""Device-side pieces of the multi-GPU path and the C++ facade, on one GPU:
member-state blobs (export/import, the payload of cross-GPU exploit copies), ShardedPBT with the
device adapter in a single-rank NCCL group (== pbt_evolve_trainer), and the C++ demo binary."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from helpers import TD3_NETS, bits_equal, raw_at, to_batch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def pb(cuda):
    import paper_2206_08888_b200 as pb
    return pb


def test_member_blob_roundtrip(pb, ora, cuda):
    import torch
    from paper_2206_08888_b200.pbrl import export_member, import_member, member_blob_size
    a = pb.make_td3_state(4, 5, 2, [16, 16], 1.0, 1)
    b = pb.make_td3_state(4, 5, 2, [16, 16], 1.0, 2)
    raw = ora.synthetic_batches(2, 4, 8, 5, 2, 3)
    for k in range(2):
        pb.td3_update_step(a, to_batch(pb, raw, k), pb.Td3Hyper.defaults(4))
    blob = torch.empty(member_blob_size(a), dtype=torch.float32, device=cuda)
    export_member(a, 3, blob.data_ptr())
    import_member(b, 1, blob.data_ptr())
    for net in TD3_NETS:
        assert bits_equal(a.flatten_member(net, 3), b.flatten_member(net, 1)), net


def test_sharded_pbt_single_rank_matches_trainer(pb, ora, cuda):
    import torch.distributed as dist
    from paper_2206_08888_b200.dist import DeviceShard, ShardedPBT
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1)
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
        plan_x = ShardedPBT(DeviceShard(x, hx), n).evolve(px, rx, pb.Td3Prior())
        plan_y = pb.pbt_evolve_trainer(py, y, hy_, pb.Td3Prior(), ry)
        assert plan_x.replaced == plan_y.replaced and plan_x.donors == plan_y.donors
        assert rx.next == ry.next
        for f in pb.Td3Hyper.FIELDS:
            assert getattr(hx, f) == getattr(hy_, f)
        for net in TD3_NETS:
            assert bits_equal(x.params(net), y.params(net))
    finally:
        dist.destroy_process_group()


def test_cpp_facade_demo_runs(cuda):
    subprocess.run(["make", "-s", "-C", str(ROOT / "examples")], check=True)
    r = subprocess.run([str(ROOT / "examples" / "cpp_facade_demo")], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "checksum" in r.stdout and "ConfigError as in the reference" in r.stdout


def test_learner_loop_example_runs(cuda, tmp_path):
    """examples/learner_loop.py: act -> replay insert -> update_k from replay -> PBT -> checkpoint
    on the device (the run_training learner loop)."""
    out = tmp_path / "policy.pbrl"
    r = subprocess.run([sys.executable, str(ROOT / "examples" / "learner_loop.py"), "--pop", "6",
                        "--envs", "4", "--iters", "8", "--pbt-interval", "4", "--out", str(out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "done:" in r.stdout and out.exists() and out.read_bytes()[:8] == b"PBRLNET1"
