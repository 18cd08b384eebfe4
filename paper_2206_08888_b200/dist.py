"""Population sharding across GPUs: the PBT exchange step (evolve.hpp:169-213).

Product path: ``Comm`` + ``NativeShardedPBT`` -- the exchange runs inside libpbrl_b200.so
(``pbrl_pbt_evolve_sharded``) over NCCL (``Comm.nccl``, NVLink / NVSwitch) or over a host
transport the caller supplies (``Comm.host``: torch.distributed, e.g. gloo, for ranks that share
one GPU).  ``ShardedPBT`` below is the same protocol written with torch.distributed collectives
around the per-step C-ABI pieces (plan / apply / member blobs); the CPU tests use it with host
shards to pin the protocol without a GPU.

Each rank owns the contiguous member block [offset, offset + n_local) of an n_total population,
with RNG streams keyed by GLOBAL member id, so a shard computes exactly what the unsharded
population computes for those members and the update step needs no communication at all.  The
one exchange is PBT, every pbt_interval updates:

  1. all_gather of per-member fitness (mean of the last 10 returns, float64);
  2. every rank computes the identical plan (stable rank + donor draws from the shared
     RngSequence; on device via pbrl_pbt_plan);
  3. exploit copies: a replaced member whose donor lives on another rank receives the donor's
     full state blob (every network, plus log_alpha for SAC) with batched send/recv;
     same-rank pairs are copied on device;
  4. optimiser reset + delay reset on the owner (pbrl_pbt_apply) and the hyper re-draw: every
     rank draws the same 6-value prior sample per replaced member (keeping the RngSequence in
     lock-step) and applies the ones it owns.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .errors import NotReadyError, PbrlError
from .pbrl import (EvolvePlan, PBTState, RngSequence, member_blob_size, export_member,
                   import_member)


class DeviceShard:
    """Adapter binding ShardedPBT to a population resident on this rank's GPU."""

    def __init__(self, pop, hyper):
        import torch
        self.pop, self.hyper = pop, hyper
        self.n_local = pop.n
        self.offset = pop.member_offset
        self.device = torch.device("cuda", pop.device)

    def blob_size(self) -> int:
        return member_blob_size(self.pop)

    def new_blob(self):
        import torch
        return torch.empty(self.blob_size(), dtype=torch.float32, device=self.device)

    def export(self, m_local: int, blob) -> None:
        export_member(self.pop, m_local, blob.data_ptr())

    def import_(self, m_local: int, blob) -> None:
        import torch
        torch.cuda.synchronize(self.device)
        import_member(self.pop, m_local, blob.data_ptr())

    def plan(self, fitness: np.ndarray, trunc: float, rng: RngSequence) -> Tuple[list, list]:
        n = fitness.size
        fit = np.ascontiguousarray(fitness, np.float64)
        rep = np.zeros(n, np.uint64)
        don = np.zeros(n, np.uint64)
        nxt = C.c_uint64(rng.next)
        cnt = C.c_uint32()
        _lib.call("pbrl_pbt_plan", self.pop.handle, fit.ctypes.data_as(_lib.f64p), n, trunc,
                  rng.stream.key, C.byref(nxt), rep.ctypes.data_as(_lib.u64p),
                  don.ctypes.data_as(_lib.u64p), C.byref(cnt))
        rng.next = nxt.value
        c = cnt.value
        return [int(x) for x in rep[:c]], [int(x) for x in don[:c]]

    def apply(self, replaced: Sequence[int], donors: Sequence[int]) -> None:
        rep = np.asarray(replaced, np.uint64)
        don = np.asarray(donors, np.uint64)
        _lib.call("pbrl_pbt_apply", self.pop.handle, rep.ctypes.data_as(_lib.u64p),
                  don.ctypes.data_as(_lib.u64p), len(rep))

    def set_hyper(self, m_local: int, one) -> None:
        self.hyper.set_member(m_local, one)

    def fitness_tensor(self, values: np.ndarray):
        import torch
        return torch.as_tensor(values, dtype=torch.float64, device=self.device)


class ShardedPBT:
    """The PBT exchange for one rank of a sharded population."""

    def __init__(self, shard, n_total: int, group=None, truncation_fraction: float = 0.3):
        import torch.distributed as dist
        self.dist = dist
        self.shard = shard
        self.n_total = n_total
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.trunc = truncation_fraction
        if n_total % self.world:
            raise ValueError("population must split evenly over the ranks")
        self.per_rank = n_total // self.world

    def owner(self, member: int) -> int:
        return member // self.per_rank

    def gather_fitness(self, local: np.ndarray) -> np.ndarray:
        import torch
        t = self.shard.fitness_tensor(np.asarray(local, np.float64))
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return torch.cat(out).cpu().numpy()

    def evolve(self, pbt_local: PBTState, rng: RngSequence, prior) -> Optional[EvolvePlan]:
        """pbt_evolve_trainer for the sharded population.  pbt_local holds this rank's members'
        return rings (local indices); returns the global plan (identical on every rank)."""
        if self.n_total < 4:
            return None
        # readiness first, on every rank: a shard with an unscored member must not leave the
        # others blocked in the fitness all_gather -- every rank raises NotReadyError together
        ready = self.gather_fitness(np.asarray([1.0 if pbt_local.every_member_scored() else 0.0]))
        if not bool(np.all(ready > 0.0)):
            raise NotReadyError("pbt_rank: every member needs at least one recorded return "
                                f"(ranks not ready: {np.flatnonzero(ready <= 0.0).tolist()})")
        fitness = self.gather_fitness(pbt_local.fitness())
        replaced, donors = self.shard.plan(fitness, self.trunc, rng)
        lo = self.shard.offset
        # exploit copies across ranks (batched point-to-point, one blob per remote pair)
        ops, recv = [], []
        for dst, src in zip(replaced, donors):
            od, os_ = self.owner(dst), self.owner(src)
            if od == os_:
                continue
            if os_ == self.rank:
                blob = self.shard.new_blob()
                self.shard.export(src - lo, blob)
                ops.append(self.dist.P2POp(self.dist.isend, blob, od, self.group))
            elif od == self.rank:
                blob = self.shard.new_blob()
                recv.append((dst - lo, blob))
                ops.append(self.dist.P2POp(self.dist.irecv, blob, os_, self.group))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        for m_local, blob in recv:
            self.shard.import_(m_local, blob)
        # local copies + optimiser / delay reset of the local receivers
        self.shard.apply(replaced, donors)
        # hyper re-draw: every rank draws for every replaced member (RngSequence in lock-step)
        for dst in replaced:
            one = prior.sample_member(rng)
            if self.owner(dst) == self.rank:
                self.shard.set_hyper(dst - lo, one)
                pbt_local.returns[dst - lo].clear()
        pbt_local.steps_since_evolve = 0
        return EvolvePlan(list(replaced), list(donors))


# ---------------------------------------------------------------- native exchange (C ABI)
class Comm:
    """A pbrl_comm handle: the transport of pbrl_pbt_evolve_sharded."""

    def __init__(self, handle, rank: int, world: int, kind: str, keep=()):
        self.handle, self.rank, self.world, self.kind = handle, rank, world, kind
        self._keep = keep  # ctypes callbacks must outlive the handle

    @staticmethod
    def nccl(device: int, group=None) -> "Comm":
        """NCCL communicator over the ranks of `group` (torch.distributed distributes the id)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = [None]
        if rank == 0:
            buf = C.create_string_buffer(128)
            _lib.call("pbrl_nccl_unique_id", buf, 128)
            uid[0] = buf.raw
        dist.broadcast_object_list(uid, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        h = C.c_void_p()
        idb = C.create_string_buffer(uid[0], 128)
        _lib.call("pbrl_comm_create_nccl", idb, rank, world, device, C.byref(h))
        return Comm(h, rank, world, "nccl")

    @staticmethod
    def host(device: int, group=None) -> "Comm":
        """Host transport over torch.distributed (any backend with CPU tensors, e.g. gloo):
        the library stages the member blobs through host memory around these callbacks."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)

        def allgather(_ctx, send, count, recv):
            try:
                src = torch.from_numpy(np.ctypeslib.as_array(send, (count,)).copy())
                out = torch.from_numpy(np.ctypeslib.as_array(recv, (world * count,)))
                parts = list(out.view(world, count).unbind(0))
                gathered = [torch.empty_like(src) for _ in range(world)]
                dist.all_gather(gathered, src, group=group)
                for dst, g in zip(parts, gathered):
                    dst.copy_(g)
                return 0
            except Exception:  # pragma: no cover - reported as PBRL_E_NCCL
                return 1

        def exchange(_ctx, ops, n_ops):
            try:
                reqs = []
                for i in range(n_ops):
                    op = ops[i]
                    t = torch.from_numpy(np.ctypeslib.as_array(op.buf, (op.floats,)))
                    peer = dist.get_global_rank(group, op.peer) if group else op.peer
                    fn = dist.isend if op.is_send else dist.irecv
                    reqs.append(dist.P2POp(fn, t, peer, group))
                if reqs:
                    for r in dist.batch_isend_irecv(reqs):
                        r.wait()
                return 0
            except Exception:  # pragma: no cover
                return 1

        def allreduce(_ctx, buf, count):
            try:
                t = torch.from_numpy(np.ctypeslib.as_array(buf, (count,)))
                dist.all_reduce(t, group=group)  # in place, sum
                return 0
            except Exception:  # pragma: no cover
                return 1

        ag, ex = _lib.ALLGATHER_FN(allgather), _lib.EXCHANGE_FN(exchange)
        ar = _lib.ALLREDUCE_FN(allreduce)
        ops = _lib.CommOps(None, ag, ex, ar)
        h = C.c_void_p()
        _lib.call("pbrl_comm_create_host", C.byref(ops), rank, world, device, C.byref(h))
        return Comm(h, rank, world, "host", keep=(ag, ex, ar, ops))

    def close(self) -> None:
        if self.handle:
            _lib.lib().pbrl_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NativeShardedPBT:
    """pbt_evolve_trainer for one shard of a population, exchange inside the library
    (pbrl_pbt_evolve_sharded): fitness all-gather, identical device plan on every rank,
    cross-rank member blobs point-to-point, resets + lock-step hyper re-draws on the owner."""

    def __init__(self, pop, hyper, comm: Comm, truncation_fraction: float = 0.3):
        self.pop, self.hyper, self.comm = pop, hyper, comm
        self.trunc = truncation_fraction
        self.last_exchange_ms = None

    def evolve(self, pbt_local: PBTState, rng: RngSequence) -> Optional[EvolvePlan]:
        pop = self.pop
        n_total = pop.n * self.comm.world
        if n_total < 4:
            return None
        ready = pbt_local.every_member_scored()
        fit = np.ascontiguousarray(pbt_local.fitness() if ready else np.zeros(pop.n), np.float64)
        rep = np.zeros(n_total, np.uint64)
        don = np.zeros(n_total, np.uint64)
        nxt = C.c_uint64(rng.next)
        cnt = C.c_uint32()
        ms = np.zeros(3, np.float64)
        pop._sync_hyper(self.hyper)
        _lib.call("pbrl_pbt_evolve_sharded", pop.handle, self.comm.handle,
                  fit.ctypes.data_as(_lib.f64p), 1 if ready else 0, self.trunc, rng.stream.key,
                  C.byref(nxt), rep.ctypes.data_as(_lib.u64p), don.ctypes.data_as(_lib.u64p),
                  C.byref(cnt), ms.ctypes.data_as(_lib.f64p))
        rng.next = nxt.value
        self.last_exchange_ms = dict(fitness_allgather=ms[0], plan=ms[1], copies_and_resets=ms[2])
        c = cnt.value
        plan = EvolvePlan([int(x) for x in rep[:c]], [int(x) for x in don[:c]])
        # the re-drawn hypers live in the library: mirror them into the host object
        for f in pop.FIELDS:
            setattr(self.hyper, f, [float(v) for v in pop.get_hyper(f)])
        pop._hyper_cache = None
        lo = pop.member_offset
        for dst in plan.replaced:
            if lo <= dst < lo + pop.n:
                pbt_local.returns[dst - lo].clear()
        pbt_local.steps_since_evolve = 0
        return plan
