"""The reference's update benchmark harness on the device (bench.hpp:20-323, bench.cpp:11-74):
BenchConfig / BenchResult, bench_update in its three modes, summarize_bench (median / IQR),
bench_estimated_bytes with the memory-budget ResourceError, bench_cross_mode_audit and
time_k_step_batching.

Modes (BenchMode, bench.hpp:17):
  vectorized        one population of n members, one update per step over the whole batch;
  sequential        n populations of one (slice_member of the same initial state), stepped one
                    after another -- the per-agent loop the paper compares against;
  parallel_threads  the same n singletons, one host thread per member (run_member_threads: at
                    most hardware_concurrency lanes), each on its own CUDA stream.

Times are wall-clock per repetition like the reference (steady_clock around the K steps), with
the device synchronised before the clock stops; repetition 0 is the discarded warm-up.
"""
from __future__ import annotations

import os
import threading
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .errors import ConfigError, ResourceError
from .pbrl import (SacHyper, Td3Hyper, TransitionBatch, make_sac_state,
                   make_synthetic_batches, make_td3_state, sac_update_step, serialize_state,
                   set_member, slice_member, td3_update_step, update_k_steps)

BENCH_MODES = ("sequential", "vectorized", "parallel_threads")


def parse_bench_mode(name: str) -> str:
    """parse_bench_mode (bench.cpp:20-26)."""
    if name not in BENCH_MODES:
        raise ConfigError(f"unknown bench mode '{name}' (expected sequential, vectorized, or "
                          f"parallel_threads)")
    return name


@dataclass
class BenchConfig:
    """BenchConfig (bench.hpp:22-40); precision / device select the B200 arithmetic."""
    mode: str = "vectorized"
    algo: str = "td3"
    n: int = 1
    k: int = 50
    reps: int = 5
    batch: int = 64
    obs_dim: int = 17
    act_dim: int = 6
    hidden: List[int] = field(default_factory=lambda: [32, 32])
    seed: int = 7
    memory_budget_bytes: int = 4 << 30
    precision: str = "ffma32"
    device: int = 0

    def validate(self) -> None:
        parse_bench_mode(self.mode)
        if self.algo not in ("td3", "sac"):
            raise ConfigError(f"BenchConfig: unknown algorithm '{self.algo}'")
        if self.n < 1 or self.k < 1:
            raise ConfigError("BenchConfig: n and k must be >= 1")
        if self.reps < 3:
            raise ConfigError("BenchConfig: need at least 3 repetitions")


@dataclass
class BenchResult:
    """BenchResult (bench.hpp:42-58)."""
    mode: str = ""
    n: int = 0
    k: int = 0
    reps: int = 0
    times_ms: List[float] = field(default_factory=list)
    median_ms: float = 0.0
    iqr_ms: float = 0.0
    warmup_ms: float = 0.0
    kernel_launches: int = 0

    CSV_HEADER = "mode,n,k,reps,median_ms,iqr_ms,warmup_ms"

    def csv_row(self) -> str:
        return (f"{self.mode},{self.n},{self.k},{self.reps},{self.median_ms:g},{self.iqr_ms:g},"
                f"{self.warmup_ms:g}")

    def agent_updates_per_s(self) -> float:
        return self.n * self.k / (self.median_ms / 1e3)


def summarize_bench(r: BenchResult) -> None:
    """summarize_bench (bench.cpp:30-35): median = sorted[n/2], IQR = sorted[3n/4] - sorted[n/4]."""
    s = sorted(r.times_ms)
    r.median_ms = s[len(s) // 2]
    r.iqr_ms = s[(3 * len(s)) // 4] - s[len(s) // 4]


def _param_count(dims):
    return sum(dims[i] * dims[i + 1] + dims[i + 1] for i in range(len(dims) - 1))


def bench_estimated_bytes(cfg: BenchConfig, scalar_bytes: int = 4) -> int:
    """bench_estimated_bytes (bench.cpp:37-56), the reference's footprint estimate."""
    dims_in = cfg.obs_dim + cfg.act_dim
    pol = [cfg.obs_dim] + list(cfg.hidden) + [cfg.act_dim * (2 if cfg.algo == "sac" else 1)]
    q = [dims_in] + list(cfg.hidden) + [1]
    per_member = _param_count(pol) + 2 * _param_count(q)
    state = cfg.n * per_member * 4 * scalar_bytes
    batches = cfg.k * cfg.n * cfg.batch * (2 * cfg.obs_dim + cfg.act_dim + 2) * scalar_bytes
    widest = max([dims_in] + list(cfg.hidden))
    activations = 16 * cfg.n * cfg.batch * widest * scalar_bytes
    return state + batches + activations


def _make_state(cfg: BenchConfig):
    make = make_td3_state if cfg.algo == "td3" else make_sac_state
    return make(cfg.n, cfg.obs_dim, cfg.act_dim, cfg.hidden, 1.0, cfg.seed,
                precision=cfg.precision, device=cfg.device)


def _hyper(cfg: BenchConfig, n: int):
    return Td3Hyper.defaults(n) if cfg.algo == "td3" else SacHyper.defaults(n, cfg.act_dim)


def _step(cfg: BenchConfig):
    return td3_update_step if cfg.algo == "td3" else sac_update_step


def _slice_batch(b: TransitionBatch, m: int) -> TransitionBatch:
    """slice_member of a batch (bench.hpp:95-104)."""
    return TransitionBatch(*[x[m:m + 1].contiguous() for x in (b.s, b.a, b.r, b.s2, b.done)])


def run_member_threads(n: int, member_fn) -> None:
    """run_member_threads (bench.cpp:58-74): min(n, hardware threads) lanes pulling members."""
    lanes = min(n, max(1, os.cpu_count() or 1))
    nxt = [0]
    lock = threading.Lock()
    errors = []

    def lane():
        while True:
            with lock:
                m = nxt[0]
                nxt[0] += 1
            if m >= n:
                return
            try:
                member_fn(m)
            except BaseException as e:  # pragma: no cover - re-raised below
                errors.append(e)
                return

    ts = [threading.Thread(target=lane) for _ in range(lanes)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errors:
        raise errors[0]


def bench_update(cfg: BenchConfig, final_policy: Optional[list] = None) -> BenchResult:
    """bench_update (bench.hpp:137-227): reps + 1 runs of K update steps from the same initial
    state; run 0 is the warm-up.  final_policy (a list) receives the final policy parameters
    [n][P] of the last repetition."""
    cfg.validate()
    need = bench_estimated_bytes(cfg, 4)
    if need > cfg.memory_budget_bytes:
        raise ResourceError(f"bench_update: population of {cfg.n} needs an estimated {need} "
                            f"bytes, over the budget of {cfg.memory_budget_bytes}")
    import torch
    dev = torch.device("cuda", cfg.device)
    batches = make_synthetic_batches(cfg.k, cfg.n, cfg.batch, cfg.obs_dim, cfg.act_dim,
                                     cfg.seed, device=dev)
    step = _step(cfg)
    res = BenchResult(mode=cfg.mode, n=cfg.n, k=cfg.k, reps=cfg.reps)
    slices = None
    if cfg.mode != "vectorized":
        slices = [[_slice_batch(b, m) for b in batches] for m in range(cfg.n)]
    st = None
    for rep in range(cfg.reps + 1):
        st = _make_state(cfg)  # st = init (bench.hpp:186): same seed, same initial state
        hy = _hyper(cfg, cfg.n)
        members, hys = None, None
        if cfg.mode != "vectorized":
            members = [slice_member(st, m) for m in range(cfg.n)]
            hys = [hy.slice(m) for m in range(cfg.n)]
        torch.cuda.synchronize(dev)
        launches0 = st.launch_count()
        t0 = time.perf_counter()
        if cfg.mode == "vectorized":
            for b in batches:
                step(st, b, hy)
            st.synchronize()
        elif cfg.mode == "sequential":
            for m in range(cfg.n):
                for b in slices[m]:
                    step(members[m], b, hys[m])
            for one in members:
                one.synchronize()
        else:
            def member_fn(m):
                for b in slices[m]:
                    step(members[m], b, hys[m])
                members[m].synchronize()
            run_member_threads(cfg.n, member_fn)
        ms = (time.perf_counter() - t0) * 1e3
        if rep == 0:
            res.warmup_ms = ms
        else:
            res.times_ms.append(ms)
            res.kernel_launches = st.launch_count() - launches0
        if members is not None and rep == cfg.reps:
            for m, one in enumerate(members):
                set_member(st, m, one)
    if final_policy is not None:
        final_policy.clear()
        final_policy.append(st.params("policy"))
    summarize_bench(res)
    return res


def bench_cross_mode_audit(cfg: BenchConfig) -> float:
    """bench_cross_mode_audit (bench.hpp:229-250): the largest |difference| between the final
    policies of the three modes (0 in the FFMA32 check mode: members are independent)."""
    import copy
    finals = []
    for mode in ("sequential", "vectorized", "parallel_threads"):
        c = copy.copy(cfg)
        c.reps, c.mode = 3, mode
        out: list = []
        bench_update(c, out)
        finals.append(out[0].astype(np.float64))
    return float(max(np.max(np.abs(finals[0] - f)) for f in finals[1:]))


@dataclass
class KStepTiming:
    """KStepTiming (bench.hpp:252-256)."""
    batched_ms: float = 0.0  # one call carrying k steps + one export, median
    loop_ms: float = 0.0     # k calls, exporting after each, median
    bitwise_equal: bool = False


def time_k_step_batching(cfg: BenchConfig, reps: int = 5, scratch_dir: Optional[str] = None
                         ) -> KStepTiming:
    """time_k_step_batching (bench.hpp:258-323), TD3: update_k_steps with one serialize_state
    export against k single-step calls each followed by an export; the two final states must be
    byte-identical."""
    import tempfile
    import torch
    if cfg.algo != "td3":
        raise ConfigError("time_k_step_batching: TD3 only (as the reference)")
    dev = torch.device("cuda", cfg.device)
    batches = make_synthetic_batches(cfg.k, cfg.n, cfg.batch, cfg.obs_dim, cfg.act_dim,
                                     cfg.seed, device=dev)
    hyper = _hyper(cfg, cfg.n)
    d = scratch_dir or tempfile.mkdtemp(prefix="pbrl_kstep_")

    def run_batched(path):
        st = _make_state(cfg)
        it = iter(batches)
        t0 = time.perf_counter()
        update_k_steps(st, lambda: next(it, None), cfg.k, hyper)
        serialize_state(st, path)
        return (time.perf_counter() - t0) * 1e3

    def run_loop(path):
        st = _make_state(cfg)
        t0 = time.perf_counter()
        for b in batches:
            td3_update_step(st, b, hyper)
            serialize_state(st, path)
        return (time.perf_counter() - t0) * 1e3

    pb_, pl_ = os.path.join(d, "batched.bin"), os.path.join(d, "loop.bin")
    tb, tl = [], []
    for _ in range(reps):
        tb.append(run_batched(pb_))
        tl.append(run_loop(pl_))
    with open(pb_, "rb") as f1, open(pl_, "rb") as f2:
        equal = f1.read() == f2.read()
    return KStepTiming(sorted(tb)[len(tb) // 2], sorted(tl)[len(tl) // 2], equal)


__all__ = ["BENCH_MODES", "BenchConfig", "BenchResult", "KStepTiming", "bench_cross_mode_audit",
           "bench_estimated_bytes", "bench_update", "parse_bench_mode", "run_member_threads",
           "summarize_bench", "time_k_step_batching"]
