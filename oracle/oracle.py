"""TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.

ctypes front end for the two CPU checkers:

* ``Oracle``  — the C restatement in ``oracle/pbrl_oracle.c`` (``_build/libpbrl_oracle.so``);
* ``Ref``     — the unmodified reference library compiled from /root/reference sources
  (``_ref/libpbrl_ref.so``, built by ``oracle/Makefile``; absent when it could not be built).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline / reference arm import this
module.  Both classes expose the same small surface (``td3(...)``, ``sac(...)``, replay, PBT,
synthetic batches) so a test can run the same scenario through either and compare bits.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libpbrl_oracle.so"
REF_SO = HERE / "_ref" / "libpbrl_ref.so"

u64 = C.c_uint64
u32 = C.c_uint32
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
i64p = C.POINTER(C.c_int64)
vp = C.c_void_p

TD3_FIELDS = ("critic_lr", "policy_lr", "policy_delay_ratio", "explore_std", "target_std",
              "target_clip", "gamma", "tau")
SAC_FIELDS = ("policy_lr", "critic_lr", "alpha_lr", "target_entropy", "reward_scale", "gamma",
              "tau")
NETS = {"policy": 0, "policy_target": 1, "critic1": 2, "critic2": 3, "critic1_target": 4,
        "critic2_target": 5}


def build() -> None:
    """Build the restatement (always) and the reference shim (when sources are present)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def td3_defaults(n: int) -> dict:
    """Td3Hyper::defaults (algos.hpp:42-53)."""
    return dict(critic_lr=[3e-4] * n, policy_lr=[3e-4] * n, policy_delay_ratio=[0.5] * n,
                explore_std=[0.1] * n, target_std=[0.2] * n, target_clip=[0.5] * n,
                gamma=[0.99] * n, tau=[0.005] * n)


def sac_defaults(n: int, act_dim: int) -> dict:
    """SacHyper::defaults (algos.hpp:121-131)."""
    return dict(policy_lr=[3e-4] * n, critic_lr=[3e-4] * n, alpha_lr=[3e-4] * n,
                target_entropy=[-float(act_dim)] * n, reward_scale=[1.0] * n, gamma=[0.99] * n,
                tau=[0.005] * n)


def pack_hyper(h: dict, fields, n: int) -> np.ndarray:
    return np.ascontiguousarray(np.stack([np.asarray(h[f], dtype=np.float64) for f in fields]))


def unpack_hyper(a: np.ndarray, fields) -> dict:
    return {f: a[i].copy() for i, f in enumerate(fields)}


class OraDvd(C.Structure):
    """ora_dvd (pbrl_oracle.h)"""
    _fields_ = [("probe", C.POINTER(C.c_double)), ("m_states", C.c_uint64),
                ("length_scale", C.c_double), ("jitter", C.c_double), ("lam", C.c_double)]


class _Lib:
    prefix = ""

    def __init__(self, path: Path):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(str(path))
        self._declare()

    # ---- declarations -------------------------------------------------------------------
    def _fn(self, name, res, *args):
        f = getattr(self.lib, name)
        f.restype = res
        f.argtypes = list(args)
        return f

    def _declare(self):
        raise NotImplementedError

    # ---- DvD / CEM (evolve.hpp:221-525), same surface on both libraries ---------------------
    def dvd_lambda(self, step, start, end, horizon):
        return getattr(self.lib, f"{self.pfx}_dvd_lambda")(step, start, end, horizon)

    def dvd_loss(self, emb, length_scale, jitter, lam):
        """(loss, logdet, grad [n][dim]); raises FloatingPointError on a singular kernel."""
        emb = np.ascontiguousarray(emb, np.float64)
        n, dim = emb.shape
        loss, logdet = C.c_double(), C.c_double()
        grad = np.zeros_like(emb)
        rc = getattr(self.lib, f"{self.pfx}_dvd_loss")(_ptr(emb, f64p), n, dim, length_scale,
                                                         jitter, lam, C.byref(loss),
                                                         C.byref(logdet), _ptr(grad, f64p))
        if rc == -10:
            raise FloatingPointError("DegeneratePopulationError")
        if rc < 0:
            raise ValueError(f"dvd_loss: config error ({rc})")
        return loss.value, logdet.value, grad

    def median_pairwise_distance(self, emb):
        emb = np.ascontiguousarray(emb, np.float64)
        return getattr(self.lib, f"{self.pfx}_median_pairwise_distance")(_ptr(emb, f64p),
                                                                         *emb.shape)

    def cem_sample(self, mean, var, noise, count, key, next_):
        """candidates [count][dim] and the advanced RngSequence counter"""
        mean = np.ascontiguousarray(mean, np.float64)
        var = np.ascontiguousarray(var, np.float64)
        out = np.zeros((count, mean.size), np.float64)
        nx = C.c_uint64(next_)
        getattr(self.lib, f"{self.pfx}_cem_sample")(_ptr(mean, f64p), _ptr(var, f64p), noise,
                                                     mean.size, count, key, C.byref(nx),
                                                     _ptr(out, f64p))
        return out, nx.value

    def cem_update(self, mean, var, noise, cands, scores, noise_final=1e-3, noise_decay=0.999,
                   elite_fraction=0.5):
        """(mean, var, noise) after cem_update; ValueError on ConfigError"""
        mean = np.array(mean, np.float64)
        var = np.array(var, np.float64)
        cands = np.ascontiguousarray(cands, np.float64)
        scores = np.ascontiguousarray(scores, np.float64)
        nz = C.c_double(noise)
        rc = getattr(self.lib, f"{self.pfx}_cem_update")(
            _ptr(mean, f64p), _ptr(var, f64p), C.byref(nz), noise_final, noise_decay,
            elite_fraction, mean.size, _ptr(cands, f64p), _ptr(scores, f64p), cands.shape[0])
        if rc < 0:
            raise ValueError(f"cem_update: config error ({rc})")
        return mean, var, nz.value


class Oracle(_Lib):
    """The C restatement (oracle/pbrl_oracle.c)."""
    pfx = "ora"

    def __init__(self, path: Path = ORACLE_SO):
        super().__init__(path)

    def _declare(self):
        F = self._fn
        self.mix64 = F("ora_mix64", u64, u64)
        self.stream_key = F("ora_stream_key", u64, u64, u64, u64, u64)
        self.bits = F("ora_bits", u64, u64, u64)
        self.uniform = F("ora_uniform", C.c_double, u64, u64)
        self.normal_pair = F("ora_normal_pair", C.c_double, u64, u64)
        self.set_emulation = F("ora_set_emulation", None, C.c_int)
        for algo in ("td3", "sac"):
            F(f"ora_{algo}_create", vp, u64, u64, u64, u64p, u32, C.c_double, u64)
            F(f"ora_{algo}_destroy", None, vp)
            F(f"ora_{algo}_param_count", u64, vp, C.c_int)
            F(f"ora_{algo}_get_net", None, vp, C.c_int, u64, f32p)
            F(f"ora_{algo}_set_net", None, vp, C.c_int, u64, f32p)
            F(f"ora_{algo}_get_adam", None, vp, C.c_int, u64, f32p, f32p, i64p)
        for algo in ("td3", "sac"):
            F(f"ora_{algo}_create_mode", vp, u64, u64, u64, u64p, u32, C.c_double, u64, C.c_int)
        F("ora_td3_step_hook", C.c_int, vp, f32p, f32p, f32p, f32p, f32p, u64, f64p, C.c_char_p,
          f64p, C.POINTER(OraDvd))
        F("ora_dvd_lambda", C.c_double, u64, C.c_double, C.c_double, u64)
        F("ora_dvd_loss", C.c_int, f64p, u64, u64, C.c_double, C.c_double, C.c_double, f64p, f64p,
          f64p)
        F("ora_median_pairwise_distance", C.c_double, f64p, u64, u64)
        F("ora_td3_dvd_embed", None, vp, f64p, u64, f32p)
        F("ora_cem_sample", None, f64p, f64p, C.c_double, u64, u64, u64, u64p, f64p)
        F("ora_cem_update", C.c_int, f64p, f64p, f64p, C.c_double, C.c_double, C.c_double, u64,
          f64p, f64p, u64)
        F("ora_td3_get_counters", None, vp, f64p, u64p)
        F("ora_td3_target", None, vp, f32p, f32p, f32p, u64, f64p, f32p)
        F("ora_td3_step", C.c_int, vp, f32p, f32p, f32p, f32p, f32p, u64, f64p, C.c_char_p, f64p)
        F("ora_sac_get_alpha", None, vp, f32p, f32p, f32p, i64p, u64p)
        F("ora_sac_step", C.c_int, vp, f32p, f32p, f32p, f32p, f32p, u64, f64p, f64p)
        F("ora_td3_act", None, vp, f32p, u64, f64p, u64, u64p, C.c_int, f32p)
        F("ora_sac_act", None, vp, f32p, u64, u64, u64p, C.c_int, f32p)
        F("ora_synthetic_batches", None, u64, u64, u64, u64, u64, u64, f32p, f32p, f32p, f32p, f32p)
        F("ora_replay_create", vp, u64, u64, u64)
        F("ora_replay_destroy", None, vp)
        F("ora_replay_push", None, vp, f32p, f32p, C.c_float, f32p, C.c_float, u32)
        F("ora_replay_size", u64, vp)
        F("ora_sample_batch", C.c_int, C.POINTER(vp), u64, u64, C.c_int, u64, u64, u64p, u64, u64,
          f32p, f32p, f32p, f32p, f32p, u64p)
        F("ora_pbt_rank", C.c_int, f64p, u32p, u64, u64, u64p)
        F("ora_pbt_plan", C.c_int, f64p, u32p, u64, u64, C.c_double, u64, u64p, u64p, u64p)
        F("ora_td3_pbt_evolve", C.c_int, vp, f64p, u32p, u64, f64p, u64, u64p, u64p, u64p)
        F("ora_sac_pbt_evolve", C.c_int, vp, f64p, u32p, u64, f64p, C.c_double, u64, u64p, u64p,
          u64p)

    def td3(self, n, ds, da, hidden, bound, seed, shared=False):
        return _State(self, "ora_td3", n, ds, da, hidden, bound, seed, "td3", shared=shared)

    def sac(self, n, ds, da, hidden, bound, seed, shared=False):
        return _State(self, "ora_sac", n, ds, da, hidden, bound, seed, "sac", shared=shared)

    def synthetic_batches(self, count, n, b, ds, da, seed):
        s = np.zeros((count, n, b, ds), np.float32)
        a = np.zeros((count, n, b, da), np.float32)
        r = np.zeros((count, n, b), np.float32)
        s2 = np.zeros((count, n, b, ds), np.float32)
        d = np.zeros((count, n, b), np.float32)
        self.lib.ora_synthetic_batches(count, n, b, ds, da, seed, _ptr(s, f32p), _ptr(a, f32p),
                                       _ptr(r, f32p), _ptr(s2, f32p), _ptr(d, f32p))
        return s, a, r, s2, d

    def replay(self, cap, ds, da):
        return _Replay(self, "ora_replay", cap, ds, da)

    def sample_batch(self, bufs, b, mode, members, seed, streams, draw_id, min_size=1):
        ds, da = bufs[0].ds, bufs[0].da
        out = [np.zeros((members, b, ds), np.float32), np.zeros((members, b, da), np.float32),
               np.zeros((members, b), np.float32), np.zeros((members, b, ds), np.float32),
               np.zeros((members, b), np.float32)]
        slots = np.zeros((members, b), np.uint64)
        arr = (vp * len(bufs))(*[x.h for x in bufs])
        st = np.asarray(streams, np.uint64)
        rc = self.lib.ora_sample_batch(arr, len(bufs), b, mode, members, seed, _ptr(st, u64p),
                                       draw_id, min_size, *[_ptr(o, f32p) for o in out],
                                       _ptr(slots, u64p))
        if rc < 0:
            raise ValueError("sample_batch: config error")
        return (tuple(out) + (slots,)) if rc == 1 else None

    def pbt_rank(self, rings, counts):
        rings, counts = _rings(rings, counts)
        n = rings.shape[0]
        order = np.zeros(n, np.uint64)
        rc = self.lib.ora_pbt_rank(_ptr(rings, f64p), _ptr(counts, u32p), n, rings.shape[1],
                                   _ptr(order, u64p))
        if rc == -4:
            raise LookupError("pbt_rank: not every member has a recorded return")
        return order

    def pbt_plan(self, rings, counts, trunc, rng_key, rng_next):
        rings, counts = _rings(rings, counts)
        n = rings.shape[0]
        rep = np.zeros(n, np.uint64)
        don = np.zeros(n, np.uint64)
        nxt = u64(rng_next)
        rc = self.lib.ora_pbt_plan(_ptr(rings, f64p), _ptr(counts, u32p), n, rings.shape[1], trunc,
                                   rng_key, C.byref(nxt), _ptr(rep, u64p), _ptr(don, u64p))
        if rc == -4:
            raise LookupError("pbt_rank: not every member has a recorded return")
        return rep[:rc], don[:rc], nxt.value


class Ref(_Lib):
    """The unmodified reference (oracle/_ref/libpbrl_ref.so)."""
    pfx = "ref"

    def __init__(self, path: Path = REF_SO):
        super().__init__(path)

    def _declare(self):
        F = self._fn
        self.mix64 = F("ref_mix64", u64, u64)
        self.stream_key = F("ref_stream_key", u64, u64, u64, u64, u64)
        self.normal_pair = F("ref_normal_pair", C.c_double, u64, u64)
        self.uniform = F("ref_uniform", C.c_double, u64, u64)
        self.tanhf = F("ref_tanhf", C.c_float, C.c_float)
        F("ref_last_error", C.c_char_p)
        for algo in ("td3f", "td3d", "sacf", "sacd"):
            fp = f32p if algo.endswith("f") else f64p
            F(f"ref_{algo}_create", vp, u64, u64, u64, u64p, u32, C.c_double, u64)
            F(f"ref_{algo}_destroy", None, vp)
            F(f"ref_{algo}_param_count", u64, vp, C.c_int)
            F(f"ref_{algo}_get_net", None, vp, C.c_int, u64, fp)
            F(f"ref_{algo}_set_net", None, vp, C.c_int, u64, fp)
            F(f"ref_{algo}_get_adam", None, vp, C.c_int, u64, fp, fp, i64p)
            if algo.startswith("td3"):
                F(f"ref_{algo}_get_counters", None, vp, f64p, u64p)
                F(f"ref_{algo}_step", C.c_int, vp, fp, fp, fp, fp, fp, u64, f64p, C.c_char_p)
                F(f"ref_{algo}_losses", C.c_int, vp, fp, fp, fp, fp, fp, u64, f64p, f64p)
                F(f"ref_{algo}_target", C.c_int, vp, fp, fp, fp, fp, fp, u64, f64p, fp)
            else:
                F(f"ref_{algo}_get_alpha", None, vp, fp, fp, fp, i64p, u64p)
                F(f"ref_{algo}_step", C.c_int, vp, fp, fp, fp, fp, fp, u64, f64p)
                F(f"ref_{algo}_losses", C.c_int, vp, fp, fp, fp, fp, fp, u64, f64p, f64p)
        F("ref_synthetic_batches_f", None, u64, u64, u64, u64, u64, u64, f32p, f32p, f32p, f32p,
          f32p)
        F("ref_td3f_act", C.c_int, vp, f32p, u64, f64p, u64, u64p, C.c_int, f32p)
        F("ref_td3f_save_checkpoint", C.c_int, vp, C.c_int, C.c_char_p)
        F("ref_td3f_load_checkpoint", C.c_int, vp, C.c_int, C.c_char_p)
        F("ref_td3f_serialize_state", C.c_int, vp, C.c_char_p)
        F("ref_sacf_act", C.c_int, vp, f32p, u64, u64, u64p, C.c_int, f32p)
        F("ref_replay_create", vp, u64, u64, u64)
        F("ref_replay_destroy", None, vp)
        F("ref_replay_push", None, vp, f32p, f32p, C.c_float, f32p, C.c_float, u32)
        F("ref_replay_size", u64, vp)
        F("ref_replay_save_snapshot", C.c_int, vp, C.c_char_p)
        F("ref_replay_load_snapshot", vp, C.c_char_p)
        F("ref_sample_batch", C.c_int, C.POINTER(vp), u64, u64, C.c_int, u64, u64, u64p, u64, u64,
          f32p, f32p, f32p, f32p, f32p)
        F("ref_pbt_rank", C.c_int, f64p, u32p, u64, u64, u64p)
        F("ref_pbt_plan", C.c_int, f64p, u32p, u64, u64, C.c_double, u64, u64p, u64p, u64p)
        F("ref_td3f_pbt_evolve", C.c_int, vp, f64p, u32p, u64, f64p, u64, u64p, u64p, u64p)
        F("ref_sacf_pbt_evolve", C.c_int, vp, f64p, u32p, u64, f64p, C.c_double, u64, u64p, u64p,
          u64p)
        F("ref_bench_update", C.c_int, C.c_int, C.c_int, u64, u64, u64, u64, u64p, u32, u64, f64p,
          f64p, f64p, u64p)
        F("ref_kernel_invocations", u64)
        for algo in ("td3f", "td3d", "sacf", "sacd"):
            F(f"ref_{algo}_create_mode", vp, u64, u64, u64, u64p, u32, C.c_double, u64, C.c_int)
        for algo, fp in (("td3f", f32p), ("td3d", f64p)):
            F(f"ref_{algo}_step_dvd", C.c_int, vp, fp, fp, fp, fp, fp, u64, f64p, C.c_char_p, f64p,
              u64, C.c_double, C.c_double, C.c_double, C.c_double, u64, u64)
            F(f"ref_{algo}_dvd_embed", None, vp, f64p, u64, fp)
        F("ref_dvd_lambda", C.c_double, u64, C.c_double, C.c_double, u64)
        F("ref_dvd_loss", C.c_int, f64p, u64, u64, C.c_double, C.c_double, C.c_double, f64p, f64p,
          f64p)
        F("ref_median_pairwise_distance", C.c_double, f64p, u64, u64)
        F("ref_cem_sample", None, f64p, f64p, C.c_double, u64, u64, u64, u64p, f64p)
        F("ref_cem_update", C.c_int, f64p, f64p, f64p, C.c_double, C.c_double, C.c_double, u64,
          f64p, f64p, u64)

    def td3(self, n, ds, da, hidden, bound, seed, dtype=np.float32, shared=False):
        sfx = "td3f" if dtype == np.float32 else "td3d"
        return _State(self, f"ref_{sfx}", n, ds, da, hidden, bound, seed, "td3", dtype, shared)

    def sac(self, n, ds, da, hidden, bound, seed, dtype=np.float32, shared=False):
        sfx = "sacf" if dtype == np.float32 else "sacd"
        return _State(self, f"ref_{sfx}", n, ds, da, hidden, bound, seed, "sac", dtype, shared)

    def synthetic_batches(self, count, n, b, ds, da, seed):
        s = np.zeros((count, n, b, ds), np.float32)
        a = np.zeros((count, n, b, da), np.float32)
        r = np.zeros((count, n, b), np.float32)
        s2 = np.zeros((count, n, b, ds), np.float32)
        d = np.zeros((count, n, b), np.float32)
        self.lib.ref_synthetic_batches_f(count, n, b, ds, da, seed, _ptr(s, f32p), _ptr(a, f32p),
                                         _ptr(r, f32p), _ptr(s2, f32p), _ptr(d, f32p))
        return s, a, r, s2, d

    def replay(self, cap, ds, da):
        return _Replay(self, "ref_replay", cap, ds, da)

    def sample_batch(self, bufs, b, mode, members, seed, streams, draw_id, min_size=1):
        ds, da = bufs[0].ds, bufs[0].da
        out = [np.zeros((members, b, ds), np.float32), np.zeros((members, b, da), np.float32),
               np.zeros((members, b), np.float32), np.zeros((members, b, ds), np.float32),
               np.zeros((members, b), np.float32)]
        arr = (vp * len(bufs))(*[x.h for x in bufs])
        st = np.asarray(streams, np.uint64)
        rc = self.lib.ref_sample_batch(arr, len(bufs), b, mode, members, seed, _ptr(st, u64p),
                                       draw_id, min_size, *[_ptr(o, f32p) for o in out])
        if rc < 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return tuple(out) if rc == 1 else None

    def pbt_rank(self, rings, counts):
        rings, counts = _rings(rings, counts)
        n = rings.shape[0]
        order = np.zeros(n, np.uint64)
        rc = self.lib.ref_pbt_rank(_ptr(rings, f64p), _ptr(counts, u32p), n, rings.shape[1],
                                   _ptr(order, u64p))
        if rc == -4:
            raise LookupError(self.lib.ref_last_error().decode())
        return order

    def pbt_plan(self, rings, counts, trunc, rng_key, rng_next):
        rings, counts = _rings(rings, counts)
        n = rings.shape[0]
        rep = np.zeros(n, np.uint64)
        don = np.zeros(n, np.uint64)
        nxt = u64(rng_next)
        rc = self.lib.ref_pbt_plan(_ptr(rings, f64p), _ptr(counts, u32p), n, rings.shape[1], trunc,
                                   rng_key, C.byref(nxt), _ptr(rep, u64p), _ptr(don, u64p))
        if rc == -4:
            raise LookupError(self.lib.ref_last_error().decode())
        return rep[:rc], don[:rc], nxt.value

    def bench_update(self, mode, algo, n, k, reps, batch, hidden, budget=0):
        h = np.asarray(hidden, np.uint64)
        med, iqr, warm = C.c_double(), C.c_double(), C.c_double()
        launches = u64()
        rc = self.lib.ref_bench_update(mode, algo, n, k, reps, batch, _ptr(h, u64p), len(hidden),
                                       budget, C.byref(med), C.byref(iqr), C.byref(warm),
                                       C.byref(launches))
        if rc < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return dict(median_ms=med.value, iqr_ms=iqr.value, warmup_ms=warm.value,
                    kernel_launches=launches.value)


def _rings(rings, counts):
    rings = np.ascontiguousarray(rings, np.float64)
    counts = np.ascontiguousarray(counts, np.uint32)
    return rings, counts


class _State:
    """A TD3 or SAC population state living in one of the CPU libraries."""

    def __init__(self, owner, prefix, n, ds, da, hidden, bound, seed, algo, dtype=np.float32,
                 shared=False):
        self.o, self.p, self.algo, self.dtype = owner, prefix, algo, dtype
        self.n, self.ds, self.da = n, ds, da
        self.shared = bool(shared)
        self.nc = 1 if shared else n  # critic population (PopMode::kSharedCritic: 1)
        self.fp = f32p if dtype == np.float32 else f64p
        h = np.asarray(hidden, np.uint64)
        self.h = getattr(owner.lib, f"{prefix}_create_mode")(n, ds, da, _ptr(h, u64p),
                                                             len(hidden), bound, seed,
                                                             1 if shared else 0)
        self.fields = TD3_FIELDS if algo == "td3" else SAC_FIELDS

    def __del__(self):
        try:
            getattr(self.o.lib, f"{self.p}_destroy")(self.h)
        except Exception:
            pass

    def _f(self, name):
        return getattr(self.o.lib, f"{self.p}_{name}")

    def param_count(self, net):
        return int(self._f("param_count")(self.h, NETS.get(net, net)))

    def get_net(self, net, m=None):
        k = NETS.get(net, net)
        P = self.param_count(k)
        if m is None:
            cnt = self.n if k <= 1 else self.nc
            return np.stack([self.get_net(k, i) for i in range(cnt)])
        out = np.zeros(P, self.dtype)
        self._f("get_net")(self.h, k, m, _ptr(out, self.fp))
        return out

    def set_net(self, net, m, flat):
        k = NETS.get(net, net)
        flat = np.ascontiguousarray(flat, self.dtype)
        self._f("set_net")(self.h, k, m, _ptr(flat, self.fp))

    def get_adam(self, net, m):
        k = NETS.get(net, net)
        P = self.param_count(k)
        mo, vo = np.zeros(P, self.dtype), np.zeros(P, self.dtype)
        t = C.c_int64()
        self._f("get_adam")(self.h, k, m, _ptr(mo, self.fp), _ptr(vo, self.fp), C.byref(t))
        return mo, vo, t.value

    def counters(self):
        if self.algo == "td3":
            da = np.zeros(self.n, np.float64)
            st = np.zeros(self.n, np.uint64)
            self._f("get_counters")(self.h, _ptr(da, f64p), _ptr(st, u64p))
            return da, st
        la, am, av = (np.zeros(self.n, self.dtype) for _ in range(3))
        at = np.zeros(self.n, np.int64)
        st = np.zeros(self.n, np.uint64)
        self._f("get_alpha")(self.h, _ptr(la, self.fp), _ptr(am, self.fp), _ptr(av, self.fp),
                             _ptr(at, i64p), _ptr(st, u64p))
        return la, am, av, at, st

    def _batch(self, batch):
        s, a, r, s2, d = (np.ascontiguousarray(x, self.dtype) for x in batch)
        return s, a, r, s2, d, s.shape[1]

    def step(self, batch, hyper, policy_mask=None, want_losses=False, dvd=None):
        """One update step.  dvd (TD3): dict probe [M][ds] (double), length_scale, jitter and
        the LambdaSchedule lam_start / lam_end / horizon at `step` (dvd_policy_hook)."""
        s, a, r, s2, d, b = self._batch(batch)
        hy = pack_hyper(hyper, self.fields, self.n)
        args = [self.h] + [_ptr(x, self.fp) for x in (s, a, r, s2, d)] + [b, _ptr(hy, f64p)]
        losses = np.zeros((3, self.n), np.float64)
        if dvd is not None:
            probe = np.ascontiguousarray(dvd["probe"], np.float64)
            ms = probe.shape[0]
            mask = None if policy_mask is None else bytes(np.asarray(policy_mask, np.uint8))
            if isinstance(self.o, Oracle):
                lam = self.o.lib.ora_dvd_lambda(dvd.get("step", 0), dvd["lam_start"],
                                                dvd["lam_end"], dvd["horizon"])
                cfg = OraDvd(_ptr(probe, f64p), ms, dvd["length_scale"], dvd["jitter"], lam)
                rc = self.o.lib.ora_td3_step_hook(*args, mask, _ptr(losses, f64p), C.byref(cfg))
            else:
                rc = self._f("step_dvd")(*args, mask, _ptr(probe, f64p), ms, dvd["length_scale"],
                                         dvd["jitter"], dvd["lam_start"], dvd["lam_end"],
                                         dvd["horizon"], dvd.get("step", 0))
            if rc == -10:
                raise FloatingPointError("DegeneratePopulationError")
            if rc < 0:
                raise ValueError(f"step failed ({rc})")
            return losses
        if isinstance(self.o, Oracle):
            if self.algo == "td3":
                mask = None if policy_mask is None else bytes(np.asarray(policy_mask, np.uint8))
                rc = self._f("step")(*args, mask, _ptr(losses, f64p))
            else:
                rc = self._f("step")(*args, _ptr(losses, f64p))
        else:
            if want_losses:
                tot = np.zeros(3, np.float64)
                rc = self._f("losses")(*args, _ptr(tot, f64p))
                if rc < 0:
                    raise ValueError(self.o.lib.ref_last_error().decode())
                losses = tot
            if self.algo == "td3":
                mask = None if policy_mask is None else bytes(np.asarray(policy_mask, np.uint8))
                rc = self._f("step")(*args, mask)
            else:
                rc = self._f("step")(*args)
            if rc < 0:
                raise ValueError(self.o.lib.ref_last_error().decode())
        if rc == -2:
            raise ValueError("config error")
        return losses

    def dvd_embed(self, probe):
        """dvd_embed (evolve.hpp:314-339): [n][M*da] deterministic actions on the probes"""
        probe = np.ascontiguousarray(probe, np.float64)
        out = np.zeros((self.n, probe.shape[0] * self.da), self.dtype)
        self._f("dvd_embed")(self.h, _ptr(probe, f64p), probe.shape[0], _ptr(out, self.fp))
        return out

    def act(self, obs, seed, steps, noise_std=None, deterministic=False):
        """act / sac_act (algos.hpp:895-942): actions [n][rows][da] for obs [n][rows][ds]."""
        obs = np.ascontiguousarray(obs, np.float32)
        rows = obs.shape[1]
        steps = np.ascontiguousarray(steps, np.uint64)
        out = np.zeros((self.n, rows, self.da), np.float32)
        det = 1 if deterministic else 0
        if self.algo == "td3":
            ns = np.ascontiguousarray(noise_std if noise_std is not None else [0.0] * self.n,
                                      np.float64)
            rc = self._f("act")(self.h, _ptr(obs, f32p), rows, _ptr(ns, f64p), seed,
                                _ptr(steps, u64p), det, _ptr(out, f32p))
        else:
            rc = self._f("act")(self.h, _ptr(obs, f32p), rows, seed, _ptr(steps, u64p), det,
                                _ptr(out, f32p))
        if rc is not None and rc < 0:
            raise ValueError(self.o.lib.ref_last_error().decode())
        return out

    def target(self, batch, hyper):
        s, a, r, s2, d, b = self._batch(batch)
        hy = pack_hyper(hyper, self.fields, self.n)
        y = np.zeros((self.n, b), self.dtype)
        if isinstance(self.o, Oracle):
            self._f("target")(self.h, _ptr(s2, self.fp), _ptr(r, self.fp), _ptr(d, self.fp), b,
                              _ptr(hy, f64p), _ptr(y, self.fp))
        else:
            rc = self._f("target")(self.h, *[_ptr(x, self.fp) for x in (s, a, r, s2, d)], b,
                                   _ptr(hy, f64p), _ptr(y, self.fp))
            if rc < 0:
                raise ValueError(self.o.lib.ref_last_error().decode())
        return y

    def pbt_evolve(self, rings, counts, hyper, rng_key, rng_next, default_te=-1.0):
        rings, counts = _rings(rings, counts)
        hy = pack_hyper(hyper, self.fields, self.n)
        rep = np.zeros(self.n, np.uint64)
        don = np.zeros(self.n, np.uint64)
        nxt = u64(rng_next)
        pre = "ora" if isinstance(self.o, Oracle) else "ref"
        tag = self.algo if pre == "ora" else self.algo + "f"
        fn = getattr(self.o.lib, f"{pre}_{tag}_pbt_evolve")
        extra = [] if self.algo == "td3" else [default_te]
        rc = fn(self.h, _ptr(rings, f64p), _ptr(counts, u32p), rings.shape[1], _ptr(hy, f64p),
                *extra, rng_key, C.byref(nxt), _ptr(rep, u64p), _ptr(don, u64p))
        if rc < 0:
            raise LookupError("pbt_evolve failed")
        return rep[:rc], don[:rc], nxt.value, unpack_hyper(hy, self.fields)


class _Replay:
    def __init__(self, owner, prefix, cap, ds, da):
        self.o, self.p, self.ds, self.da = owner, prefix, ds, da
        self.h = getattr(owner.lib, f"{prefix}_create")(cap, ds, da)

    def __del__(self):
        try:
            getattr(self.o.lib, f"{self.p}_destroy")(self.h)
        except Exception:
            pass

    def push(self, s, a, r, s2, d, member=0):
        s = np.ascontiguousarray(s, np.float32)
        a = np.ascontiguousarray(a, np.float32)
        s2 = np.ascontiguousarray(s2, np.float32)
        getattr(self.o.lib, f"{self.p}_push")(self.h, _ptr(s, f32p), _ptr(a, f32p), float(r),
                                              _ptr(s2, f32p), float(d), member)

    def size(self):
        return int(getattr(self.o.lib, f"{self.p}_size")(self.h))


def have_ref() -> bool:
    return REF_SO.exists()


def load_oracle() -> Oracle:
    if not ORACLE_SO.exists():
        build()
    return Oracle()


def load_ref():
    return Ref() if REF_SO.exists() else None


__all__ = ["Oracle", "Ref", "build", "have_ref", "load_oracle", "load_ref", "td3_defaults",
           "sac_defaults", "pack_hyper", "unpack_hyper", "TD3_FIELDS", "SAC_FIELDS", "NETS"]

if os.environ.get("PBRL_ORACLE_AUTOBUILD") == "1" and not ORACLE_SO.exists():  # pragma: no cover
    build()
