"""N > 1 path on CPU: the sharded PBT exchange (paper_2206_08888_b200/dist.py) with world_size 2
over gloo.  Each rank holds half of an 8-member population in host memory; after
ShardedPBT.evolve the union of both shards must equal the single-process pbt_evolve_trainer
result (evolve.hpp:169-190): bitwise donor copies (including cross-rank ones), resets of exactly
the replaced members, identical hyper re-draws on both ranks, identical plans."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N_TOTAL, P = 8, 37
RETURNS = [3.0, -1.0, 7.5, 0.0, 2.0, 9.0, -4.0, 1.0]


class HostShard:
    def __init__(self, rank, world, hyper):
        self.n_local = N_TOTAL // world
        self.offset = rank * self.n_local
        self.params = {m: np.arange(P, dtype=np.float32) + 1000.0 * (self.offset + m)
                       for m in range(self.n_local)}
        self.reset = set()
        self.hyper = hyper

    def blob_size(self):
        return P

    def new_blob(self):
        return torch.empty(P, dtype=torch.float32)

    def export(self, m, blob):
        blob.copy_(torch.from_numpy(self.params[m]))

    def import_(self, m, blob):
        self.params[m] = blob.numpy().copy()

    def plan(self, fitness, trunc, rng):
        from paper_2206_08888_b200.pbrl import plan_from_fitness
        return plan_from_fitness(list(fitness), trunc, rng)

    def apply(self, replaced, donors):
        lo, hi = self.offset, self.offset + self.n_local
        for d, s in zip(replaced, donors):
            if lo <= d < hi:
                self.reset.add(d - lo)
                if lo <= s < hi:
                    self.params[d - lo] = self.params[s - lo].copy()

    def set_hyper(self, m, one):
        self.hyper.set_member(m, one)

    def fitness_tensor(self, values):
        return torch.as_tensor(values, dtype=torch.float64)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2206_08888_b200 as pb
    from paper_2206_08888_b200.dist import ShardedPBT
    hy = pb.Td3Hyper.defaults(N_TOTAL // world)
    shard = HostShard(rank, world, hy)
    pbt = pb.PBTState(shard.n_local)
    for m in range(shard.n_local):
        pbt.record_return(m, RETURNS[shard.offset + m])
    rng = pb.RngSequence(1, 2, "kDonorChoice")
    plan = ShardedPBT(shard, N_TOTAL).evolve(pbt, rng, pb.Td3Prior())
    q.put((rank, plan.replaced, plan.donors, {shard.offset + m: v for m, v in shard.params.items()},
           sorted(shard.offset + m for m in shard.reset),
           {f: list(getattr(hy, f)) for f in hy.FIELDS}, rng.next))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_pbt_equals_single_process():
    import paper_2206_08888_b200 as pb
    from paper_2206_08888_b200.pbrl import plan_from_fitness
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    # single-process reference semantics
    rng = pb.RngSequence(1, 2, "kDonorChoice")
    rep, don = plan_from_fitness(RETURNS, 0.3, rng)
    params = {m: np.arange(P, dtype=np.float32) + 1000.0 * m for m in range(N_TOTAL)}
    hy = pb.Td3Hyper.defaults(N_TOTAL)
    for d, s in zip(rep, don):
        params[d] = params[s].copy()
        hy.set_member(d, pb.Td3Prior().sample_member(rng))
    assert any((d // 4) != (s // 4) for d, s in zip(rep, don)), "want a cross-rank copy"
    merged, resets, hypers = {}, [], {f: [] for f in hy.FIELDS}
    for rank, r_rep, r_don, prm, rs, h, nxt in res:
        assert r_rep == rep and r_don == don and nxt == rng.next  # identical plans / rng state
        merged.update(prm)
        resets += rs
        for f in hy.FIELDS:
            hypers[f] += h[f]
    for m in range(N_TOTAL):
        assert np.array_equal(merged[m], params[m]), m
    assert sorted(resets) == sorted(rep)
    for f in hy.FIELDS:
        assert hypers[f] == list(getattr(hy, f)), f
