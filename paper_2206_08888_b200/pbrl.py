"""Host mirror of the reference population-trainer API (proj/core, namespace pbrl).

Same names, argument meanings and error behaviour as the reference C++ templates, backed by
the B200 library through the C ABI (include/pbrl_b200.h):

    make_td3_state / Td3Hyper / td3_update_step / update_k_steps        algos.hpp:32-422, :948-983
    make_sac_state / SacHyper / sac_update_step                         algos.hpp:112-156, :470-837
    make_synthetic_batches                                              bench.hpp:69-93
    DeviceReplay (ReplayBuffer) / sample_batch                          replay.hpp:28-204
    RngSequence                                                         rng.hpp:74-95
    PBTState / pbt_rank / pbt_plan / pbt_evolve_trainer / priors        evolve.hpp:13-213

State lives in HBM; numpy arrays cross the boundary only when the caller asks for them
(flatten_member, counters, losses).  Batches may be numpy (host) or torch CUDA tensors (device).
"""
from __future__ import annotations

import ctypes as C
import math
from collections import deque
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .errors import (ConfigError, DataStarvationError, NotReadyError, ShapeError, UsageError)

PRECISIONS = {"ffma32": 0, "bf16": 1, "tf32": 2}
MODES = {"independent": 0, "kIndependent": 0, "shared_critic": 1, "kSharedCritic": 1,
         "shared": 1}
NETS = {"policy": 0, "policy_target": 1, "critic1": 2, "critic2": 3, "critic1_target": 4,
        "critic2_target": 5}
TD3_FIELDS = ("critic_lr", "policy_lr", "policy_delay_ratio", "explore_std", "target_std",
              "target_clip", "gamma", "tau")
SAC_FIELDS = ("policy_lr", "critic_lr", "alpha_lr", "target_entropy", "reward_scale", "gamma",
              "tau")
RNG_USE = dict(kInitWeight=1, kInitBias=2, kExploreNoise=3, kTargetNoise=4, kSacEps=5,
               kSacEpsTarget=6, kSample=7, kDonorChoice=8, kHyperDraw=9, kCemDraw=10,
               kEnvReset=11, kGeneric=12)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a, t):
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------------- RNG (rng.hpp)
M64 = (1 << 64) - 1


def mix64(x: int) -> int:
    """SplitMix64 finalizer (rng.hpp:13-18)."""
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


class RngStream:
    """RngStream (rng.hpp:36-71): every draw is a pure function of (key, counter)."""

    def __init__(self, key: int):
        self.key = key & M64

    @staticmethod
    def of(seed: int, stream_id: int, use, step: int = 0) -> "RngStream":
        use = RNG_USE[use] if isinstance(use, str) else int(use)
        k = mix64(seed & M64)
        k = mix64(k ^ (stream_id & M64))
        k = mix64(k ^ use)
        k = mix64(k ^ (step & M64))
        return RngStream(k)

    def bits(self, counter: int) -> int:
        return mix64(self.key ^ mix64(counter & M64))

    def uniform(self, counter: int, lo: float = None, hi: float = None) -> float:
        u = float(self.bits(counter) >> 11) * 2.0 ** -53
        return u if lo is None else lo + (hi - lo) * u


class RngSequence:
    """Stateful wrapper (rng.hpp:74-95); Python floats are IEEE doubles and math.exp/log are
    the same libm calls the reference makes, so draws are bit-identical."""

    def __init__(self, seed_or_stream, stream_id: int = 0, use="kGeneric", step: int = 0):
        if isinstance(seed_or_stream, RngStream):
            self.stream = seed_or_stream
        else:
            self.stream = RngStream.of(seed_or_stream, stream_id, use, step)
        self.next = 0

    def bits(self) -> int:
        b = self.stream.bits(self.next)
        self.next += 1
        return b

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        v = self.stream.uniform(self.next, lo, hi)
        self.next += 1
        return v

    def log_uniform(self, lo: float, hi: float) -> float:
        return math.exp(self.uniform(math.log(lo), math.log(hi)))

    def index(self, n: int) -> int:
        return self.bits() % n


# ---------------------------------------------------------------------- hyperparameters
@dataclass
class Td3Hyper:
    """Per-member TD3 hyperparameters (algos.hpp:32-109)."""
    critic_lr: List[float] = field(default_factory=list)
    policy_lr: List[float] = field(default_factory=list)
    policy_delay_ratio: List[float] = field(default_factory=list)
    explore_std: List[float] = field(default_factory=list)
    target_std: List[float] = field(default_factory=list)
    target_clip: List[float] = field(default_factory=list)
    gamma: List[float] = field(default_factory=list)
    tau: List[float] = field(default_factory=list)
    FIELDS = TD3_FIELDS

    @staticmethod
    def defaults(n: int) -> "Td3Hyper":
        return Td3Hyper([3e-4] * n, [3e-4] * n, [0.5] * n, [0.1] * n, [0.2] * n, [0.5] * n,
                        [0.99] * n, [0.005] * n)

    def members(self) -> int:
        return len(self.critic_lr)

    def slice(self, i: int) -> "Td3Hyper":
        return Td3Hyper(*[[getattr(self, f)[i]] for f in TD3_FIELDS])

    def set_member(self, i: int, one: "Td3Hyper") -> None:
        for f in TD3_FIELDS:
            getattr(self, f)[i] = getattr(one, f)[0]

    def validate(self, n: int) -> None:
        for f in TD3_FIELDS:
            if len(getattr(self, f)) != n:
                raise ConfigError(f"Td3Hyper: {f} length != N")
        for i in range(n):
            if not (self.critic_lr[i] > 0) or not (self.policy_lr[i] > 0):
                raise ConfigError("Td3Hyper: learning rates must be positive")
            if not (0 < self.policy_delay_ratio[i] <= 1.0):
                raise ConfigError("Td3Hyper: policy_delay_ratio must be in (0, 1]")
            if self.explore_std[i] < 0 or self.target_std[i] < 0 or self.target_clip[i] < 0:
                raise ConfigError("Td3Hyper: noise parameters must be >= 0")
            if not (0.9 <= self.gamma[i] <= 1.0) and self.gamma[i] != 0.0:
                raise ConfigError("Td3Hyper: discount must be in [0.9, 1] (or 0 in tests)")
            if not (0 < self.tau[i] <= 1.0):
                raise ConfigError("Td3Hyper: tau must be in (0, 1]")


@dataclass
class SacHyper:
    """Per-member SAC hyperparameters (algos.hpp:112-156)."""
    policy_lr: List[float] = field(default_factory=list)
    critic_lr: List[float] = field(default_factory=list)
    alpha_lr: List[float] = field(default_factory=list)
    target_entropy: List[float] = field(default_factory=list)
    reward_scale: List[float] = field(default_factory=list)
    gamma: List[float] = field(default_factory=list)
    tau: List[float] = field(default_factory=list)
    FIELDS = SAC_FIELDS

    @staticmethod
    def defaults(n: int, action_dim: int) -> "SacHyper":
        return SacHyper([3e-4] * n, [3e-4] * n, [3e-4] * n, [-float(action_dim)] * n, [1.0] * n,
                        [0.99] * n, [0.005] * n)

    def members(self) -> int:
        return len(self.policy_lr)

    def slice(self, i: int) -> "SacHyper":
        return SacHyper(*[[getattr(self, f)[i]] for f in SAC_FIELDS])

    def set_member(self, i: int, one: "SacHyper") -> None:
        for f in SAC_FIELDS:
            getattr(self, f)[i] = getattr(one, f)[0]

    def validate(self, n: int) -> None:
        for f in SAC_FIELDS:
            if len(getattr(self, f)) != n:
                raise ConfigError(f"SacHyper: {f} length != N")


# ---------------------------------------------------------------------- batches
@dataclass
class TransitionBatch:
    """Population batch (algos.hpp:14-24): s [N,B,ds], a [N,B,da], r [N,B,1], s2, done."""
    s: object
    a: object
    r: object
    s2: object
    done: object

    def members(self) -> int:
        return int(self.s.shape[0])

    def rows(self) -> int:
        return int(self.s.shape[1])

    def is_device(self) -> bool:
        return hasattr(self.s, "is_cuda") and bool(self.s.is_cuda)


def make_synthetic_batches(count: int, n: int, batch: int, obs_dim: int, act_dim: int,
                           seed: int, device=None) -> List[TransitionBatch]:
    """make_synthetic_batches (bench.hpp:69-93), generated on the GPU by the library.
    Returns torch CUDA tensors on `device` (default cuda:0)."""
    import torch
    dev = torch.device(device if device is not None else "cuda:0")
    shapes = [(count, n, batch, obs_dim), (count, n, batch, act_dim), (count, n, batch, 1),
              (count, n, batch, obs_dim), (count, n, batch, 1)]
    ts = [torch.empty(s, dtype=torch.float32, device=dev) for s in shapes]
    with torch.cuda.device(dev):
        _lib.call("pbrl_synthetic_batches_device", None, count, n, batch, obs_dim, act_dim, seed,
                  C.byref(_lib.Batch(*[t.data_ptr() for t in ts])))
        torch.cuda.synchronize(dev)
    return [TransitionBatch(*[t[i] for t in ts]) for i in range(count)]


def _check_batch_shapes(b: TransitionBatch, n: int, rows: int, ds: int, da: int) -> None:
    """TransitionBatch extents (algos.hpp:14-24): s, s2 [n, rows, ds], a [n, rows, da], r and done
    [n, rows, 1] (or [n, rows]).  The library copies n*rows*dim elements per field, so a wrong
    width must fail here (ShapeError, naming both shapes) instead of reading out of bounds."""
    for name, x, dim in (("s", b.s, ds), ("a", b.a, da), ("r", b.r, 1), ("s2", b.s2, ds),
                         ("done", b.done, 1)):
        shp = tuple(int(v) for v in x.shape)
        ok = len(shp) == 3 and shp == (n, rows, dim)
        if dim == 1 and len(shp) == 2:
            ok = shp == (n, rows)
        if not ok:
            raise ShapeError(f"TransitionBatch.{name}: shape {list(shp)} != "
                             f"[{n}, {rows}, {dim}]")


def _batch_struct(b: TransitionBatch, keep: list, device: int):
    if b.is_device():
        import torch
        arrs = []
        for x in (b.s, b.a, b.r, b.s2, b.done):
            if x.dtype != torch.float32:
                raise UsageError(f"device batch tensors must be float32 (got {x.dtype})")
            if x.device.index != device:
                raise UsageError(f"device batch on {x.device}, population on cuda:{device}")
            arrs.append(x.contiguous())
        keep.extend(arrs)
        return _lib.Batch(*[x.data_ptr() for x in arrs]), True
    arrs = [_f32(np.asarray(x)) for x in (b.s, b.a, b.r, b.s2, b.done)]
    keep.extend(arrs)
    return _lib.Batch(*[x.ctypes.data for x in arrs]), False


# ---------------------------------------------------------------------- population state
class _Population:
    algo = 0
    FIELDS: Sequence[str] = ()

    def __init__(self, n, obs_dim, act_dim, hidden, action_bound, seed, precision="ffma32",
                 device=0, member_offset=0, n_global=None, mode="independent"):
        if mode not in MODES:
            raise ConfigError(f"unknown population mode {mode!r}")
        # PopMode (algos.hpp:26): a shared-critic population has ONE critic pair whose batch is
        # the population folded into rows (CEM-RL / DvD)
        self.mode = "shared_critic" if MODES[mode] else "independent"
        self.shared = bool(MODES[mode])
        if precision not in PRECISIONS:
            raise ConfigError(f"unknown precision {precision!r}")
        self.n, self.obs_dim, self.act_dim = int(n), int(obs_dim), int(act_dim)
        self.hidden = [int(h) for h in hidden]
        self.seed = int(seed)
        self.precision = precision
        self.device = int(device)
        self.member_offset = int(member_offset)
        self.n_global = int(n_global or n)
        self._action_bound = float(action_bound)
        hid = (C.c_uint64 * max(1, len(self.hidden)))(*self.hidden)
        desc = _lib.PopDesc(self.algo, self.n, self.obs_dim, self.act_dim, len(self.hidden),
                            C.cast(hid, _lib.u64p), self._action_bound, self.seed,
                            PRECISIONS[precision], self.device, self.member_offset,
                            self.n_global, MODES[mode])
        h = C.c_void_p()
        _lib.call("pbrl_pop_create", C.byref(desc), C.byref(h))
        self._h = h
        self._hyper_cache = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().pbrl_pop_destroy(h)
            except Exception:
                pass
            self._h = None

    # -- reference accessors
    def members(self) -> int:
        return self.n

    @property
    def handle(self):
        return self._h

    def param_count(self, net) -> int:
        c = C.c_uint64()
        _lib.call("pbrl_param_count", self._h, NETS.get(net, net), C.byref(c))
        return c.value

    def flatten_member(self, net, i: int) -> np.ndarray:
        """flatten_member (net_pop.hpp:163-173) of one network."""
        out = np.empty(self.param_count(net), np.float32)
        _lib.call("pbrl_get_member", self._h, NETS.get(net, net), i, _ptr(out, _lib.f32p))
        return out

    def unflatten_member(self, net, i: int, vec) -> None:
        """unflatten_member (net_pop.hpp:176-189)."""
        vec = _f32(vec)
        if vec.size != self.param_count(net):
            raise ShapeError(f"unflatten_member: vector length {vec.size} != member parameter "
                             f"count {self.param_count(net)}")
        _lib.call("pbrl_set_member", self._h, NETS.get(net, net), i, _ptr(vec, _lib.f32p))

    def copy_member(self, net, src: int, dst: int) -> None:
        _lib.call("pbrl_copy_member", self._h, NETS.get(net, net), src, dst)

    def net_members(self, net) -> int:
        """members of one network: n, or 1 for the critics of a shared-critic population"""
        k = NETS.get(net, net)
        return self.n if (k <= 1 or not self.shared) else 1

    def params(self, net) -> np.ndarray:
        return np.stack([self.flatten_member(net, i) for i in range(self.net_members(net))])

    def adam(self, net, i: int):
        P = self.param_count(net)
        m, v = np.empty(P, np.float32), np.empty(P, np.float32)
        t = C.c_int64()
        _lib.call("pbrl_get_adam", self._h, NETS.get(net, net), i, _ptr(m, _lib.f32p),
                  _ptr(v, _lib.f32p), C.byref(t))
        return m, v, t.value

    @property
    def steps(self) -> np.ndarray:
        st = np.empty(self.n, np.uint64)
        _lib.call("pbrl_get_counters", self._h, None, _ptr(st, _lib.u64p))
        return st

    def last_losses(self):
        out = [np.empty(self.n, np.float64) for _ in range(3)]
        _lib.call("pbrl_last_losses", self._h, *[_ptr(o, _lib.f64p) for o in out])
        return tuple(out)

    def synchronize(self) -> None:
        _lib.call("pbrl_synchronize", self._h)

    def device_bytes(self) -> int:
        b = C.c_uint64()
        _lib.call("pbrl_device_bytes", self._h, C.byref(b))
        return b.value

    # -- hyper upload (cached: only re-sent when the host vectors change)
    def _sync_hyper(self, hyper) -> None:
        hyper.validate(self.n)
        snap = tuple(tuple(float(x) for x in getattr(hyper, f)) for f in self.FIELDS)
        if snap == self._hyper_cache:
            return
        for f, vals in zip(self.FIELDS, snap):
            arr = np.asarray(vals, np.float64)
            _lib.call("pbrl_set_hyper", self._h, f.encode(), _ptr(arr, _lib.f64p))
        self._hyper_cache = snap

    def get_hyper(self, f: str) -> np.ndarray:
        out = np.empty(self.n, np.float64)
        _lib.call("pbrl_get_hyper", self._h, f.encode(), _ptr(out, _lib.f64p))
        return out

    # -- updates
    def lib_stream(self):
        """The library's CUDA stream of this population as a torch ExternalStream."""
        if getattr(self, "_ext_stream", None) is None:
            import torch
            sp = C.c_void_p()
            _lib.call("pbrl_get_stream", self._h, C.byref(sp))
            self._ext_stream = torch.cuda.ExternalStream(sp.value,
                                                         device=torch.device("cuda", self.device))
        return self._ext_stream

    def _device_call_begin(self):
        """Device batches are written on torch's current stream: the library stream waits for
        that work before its first kernel reads them."""
        import torch
        ext = self.lib_stream()
        ext.wait_stream(torch.cuda.current_stream(torch.device("cuda", self.device)))
        return ext

    def _device_call_end(self, ext, keep):
        """The library runs asynchronously: tensors it reads (incl. .contiguous() temporaries)
        must not be reused by torch's caching allocator before the library stream is done.
        torch's current stream waits for the library stream, so any later reuse of that memory
        (allocations are ordered on the stream that freed them) comes after the library's reads.
        (record_stream on the library stream would tie the tensors' frees to a stream that dies
        with the population.)"""
        import torch
        if ext is not None:
            torch.cuda.current_stream(torch.device("cuda", self.device)).wait_stream(ext)
        del keep

    def _update(self, batches: Sequence[TransitionBatch], mask=None,
                return_losses: bool = False) -> Optional[np.ndarray]:
        if not batches:
            raise ConfigError("update_k_steps: k must be >= 1")
        keep = []
        structs, dev = [], None
        rows = batches[0].rows()
        for b in batches:
            if b.members() != self.n:
                raise ConfigError(f"update_step: batch population {b.members()} != state "
                                  f"population {self.n}")
            if b.rows() != rows:
                raise ShapeError("all batches of one call must have the same row count")
            _check_batch_shapes(b, self.n, rows, self.obs_dim, self.act_dim)
            s, d = _batch_struct(b, keep, self.device)
            if dev is None:
                dev = d
            elif dev != d:
                raise UsageError("mixing host and device batches in one call")
            structs.append(s)
        arr = (_lib.Batch * len(structs))(*structs)
        m = None
        if mask is not None:
            mk = np.ascontiguousarray(np.asarray(mask, dtype=bool).astype(np.uint8))
            if mk.shape != (self.n,):
                raise ShapeError(f"policy_member_mask: {mk.size} entries != population {self.n}")
            keep.append(mk)
            m = _ptr(mk, _lib.u8p)
        if return_losses and not dev:
            # every step's losses, H2D of batch i+1 overlapping step i (one host round trip)
            out = np.empty((len(structs), 3, self.n), np.float64)
            _lib.call("pbrl_update_batches_losses", self._h, arr, len(structs), rows, m,
                      _ptr(out, _lib.f64p))
            return out
        ext = self._device_call_begin() if dev else None
        try:
            if return_losses:  # device batches: step by step
                out = np.empty((len(structs), 3, self.n), np.float64)
                for i in range(len(structs)):
                    one = (_lib.Batch * 1)(structs[i])
                    _lib.call("pbrl_update_batches_device", self._h, one, 1, rows, m)
                    out[i] = np.stack(self.last_losses())
                return out
            fn = "pbrl_update_batches_device" if dev else "pbrl_update_batches"
            _lib.call(fn, self._h, arr, len(structs), rows, m)
            return None
        finally:
            if ext is not None:
                self._device_call_end(ext, keep)

    def attach_comm(self, comm) -> None:
        """Shared-critic population sharded over ranks: sum the critic gradients over `comm`
        (dist.Comm) every step before the critic Adam (pbrl_attach_comm); None detaches."""
        _lib.call("pbrl_attach_comm", self._h, None if comm is None else comm.handle)
        self._comm = comm

    def launch_count(self) -> int:
        c = C.c_uint64()
        _lib.call("pbrl_launch_count", self._h, C.byref(c))
        return c.value


class Td3State(_Population):
    """Td3State (algos.hpp:165-179) resident on one B200."""
    algo = 0
    FIELDS = TD3_FIELDS

    @property
    def action_bound(self) -> float:
        return float(np.float32(self._action_bound))

    @property
    def delay_acc(self) -> np.ndarray:
        d = np.empty(self.n, np.float64)
        _lib.call("pbrl_get_counters", self._h, _ptr(d, _lib.f64p), None)
        return d


class SacState(_Population):
    """SacState (algos.hpp:473-488) resident on one B200."""
    algo = 1
    FIELDS = SAC_FIELDS

    def alpha_state(self):
        la, m, v = (np.empty(self.n, np.float32) for _ in range(3))
        t = np.empty(self.n, np.int64)
        _lib.call("pbrl_get_alpha", self._h, _ptr(la, _lib.f32p), _ptr(m, _lib.f32p),
                  _ptr(v, _lib.f32p), _ptr(t, _lib.i64p))
        return la, m, v, t

    @property
    def log_alpha(self) -> np.ndarray:
        return self.alpha_state()[0]


def make_td3_state(n, obs_dim, act_dim, hidden, action_bound, seed, mode="independent",
                   precision="ffma32", device=0, member_offset=0, n_global=None) -> Td3State:
    """make_td3_state (algos.hpp:181-212)."""
    return Td3State(n, obs_dim, act_dim, hidden, action_bound, seed, precision, device,
                    member_offset, n_global, mode)


def make_sac_state(n, obs_dim, act_dim, hidden, action_bound, seed, mode="independent",
                   precision="ffma32", device=0, member_offset=0, n_global=None) -> SacState:
    """make_sac_state (algos.hpp:490-521)."""
    return SacState(n, obs_dim, act_dim, hidden, action_bound, seed, precision, device,
                    member_offset, n_global, mode)


def slice_member(st: _Population, i: int) -> _Population:
    """slice_member for states (algos.hpp:425-447, :839-865): member i as a population of one on
    the same device -- every network, Adam moments and counters, steps, stream id, delay_acc
    (TD3) or the temperature state (SAC), and the member's hypers."""
    if not 0 <= i < st.n:
        raise UsageError(f"slice_member: index {i} out of range for {st.n} members")
    one = type(st)(1, st.obs_dim, st.act_dim, st.hidden, st._action_bound, st.seed, st.precision,
                   st.device, st.member_offset + i, st.n_global)
    _lib.call("pbrl_copy_member_state", one.handle, 0, st.handle, i)
    return one


def set_member(st: _Population, i: int, sub: _Population) -> None:
    """set_member for states (algos.hpp:449-464, :867-886): member 0 of `sub` into member i."""
    if sub.n != 1:
        raise UsageError("set_member: the source must be a population of one")
    _lib.call("pbrl_copy_member_state", st.handle, i, sub.handle, 0)
    st._hyper_cache = None


def td3_update_step(st: Td3State, batch: TransitionBatch, hyper: Td3Hyper, hook=None,
                    policy_member_mask=None) -> None:
    """td3_update_step (algos.hpp:351-422).  hook: a DvdHook from dvd_policy_hook (the only
    PolicyGradHook the reference builds, evolve.hpp:507-525), applied on the device."""
    st._sync_hyper(hyper)
    with _hooked(st, hook):
        st._update([batch], policy_member_mask)


class _hooked:
    """Installs a DvD hook on the population for the duration of one update call."""

    def __init__(self, st, hook):
        self.st, self.hook = st, hook

    def __enter__(self):
        if self.hook is not None:
            if not isinstance(self.hook, DvdHook):
                raise ConfigError("td3_update_step: hook must come from dvd_policy_hook")
            self.hook._install(self.st)

    def __exit__(self, *exc):
        if self.hook is not None:
            _lib.call("pbrl_set_dvd", self.st.handle, None, 0, 1.0, 0.0, 0.0)
        return False


def sac_update_step(st: SacState, batch: TransitionBatch, hyper: SacHyper) -> None:
    """sac_update_step (algos.hpp:781-837)."""
    st._sync_hyper(hyper)
    st._update([batch])


def update_k_steps(st, sampler: Callable[[], Optional[TransitionBatch]], k: int, hyper,
                   hook=None, return_losses: bool = False) -> Optional[np.ndarray]:
    """update_k_steps (algos.hpp:953-983): k chained steps, no export in between; the device
    runs them back to back.  An exhausted sampler raises DataStarvationError.  return_losses:
    the k steps' critic1 / critic2 / policy losses as a [k, 3, n] array (with host batches the
    H2D copy of batch i+1 overlaps step i)."""
    if k < 1:
        raise ConfigError("update_k_steps: k must be >= 1")
    batches = []
    for i in range(k):
        b = sampler()
        if b is None:
            raise DataStarvationError(f"update_k_steps: sampler exhausted after {i} of {k} steps")
        batches.append(b)
    st._sync_hyper(hyper)
    with _hooked(st, hook):
        return st._update(batches, return_losses=return_losses)


# ---------------------------------------------------------------------- DvD (evolve.hpp:304-525)
@dataclass
class LambdaSchedule:
    """Linear ramp from start to end over horizon steps, clamped afterwards (evolve.hpp:304-309)."""
    start: float = 0.0
    end: float = 0.5
    horizon: int = 1


def dvd_lambda(step: int, s: LambdaSchedule) -> float:
    """dvd_lambda (evolve.hpp:310-314)."""
    out = C.c_double()
    _lib.call("pbrl_dvd_lambda", int(step), float(s.start), float(s.end), int(s.horizon),
              C.byref(out))
    return out.value


@dataclass
class DvDConfig:
    """DvDConfig (evolve.hpp:489-503): probe states (row-major M x ds), kernel and schedule."""
    probe_states: Sequence[float] = field(default_factory=list)
    m_states: int = 0
    length_scale: float = 1.0
    jitter: float = 1e-6
    schedule: LambdaSchedule = field(default_factory=LambdaSchedule)

    def validate(self, population: int) -> None:
        if self.m_states < population:
            raise ConfigError("DvDConfig: need at least as many probe states as members")
        if not self.length_scale > 0:
            raise ConfigError("DvDConfig: length scale must be positive")
        if self.jitter < 0:
            raise ConfigError("DvDConfig: jitter must be >= 0")


class DvdHook:
    """dvd_policy_hook(cfg, step) (evolve.hpp:507-525): the diversity gradient of
    -lambda * logdet(K + jitter I) over the policies' probe-state embeddings, added to the policy
    gradients inside the device update step."""

    def __init__(self, cfg: DvDConfig, lam: float):
        self.cfg, self.lam = cfg, float(lam)

    def _install(self, st) -> None:
        probe = np.ascontiguousarray(np.asarray(self.cfg.probe_states, np.float64).ravel())
        if probe.size != self.cfg.m_states * st.obs_dim:
            raise ShapeError("dvd_embed: probe matrix size != M * observation_dim")
        _lib.call("pbrl_set_dvd", st.handle, _ptr(probe, _lib.f64p), self.cfg.m_states,
                  float(self.cfg.length_scale), float(self.cfg.jitter), self.lam)


def dvd_policy_hook(cfg: DvDConfig, step: int) -> DvdHook:
    return DvdHook(cfg, dvd_lambda(step, cfg.schedule))


def dvd_embed(policies: "Td3State", probe_states, m_states: int) -> np.ndarray:
    """dvd_embed (evolve.hpp:337-340): [n, m_states * da] deterministic actions on the probes."""
    probe = np.ascontiguousarray(np.asarray(probe_states, np.float64).ravel())
    if probe.size != m_states * policies.obs_dim:
        raise ShapeError("dvd_embed: probe matrix size != M * observation_dim")
    out = np.empty((policies.n, m_states * policies.act_dim), np.float32)
    _lib.call("pbrl_dvd_embed", policies.handle, _ptr(probe, _lib.f64p), m_states,
              _ptr(out, _lib.f32p))
    return out


@dataclass
class DvdLossOut:
    loss: float
    logdet: float
    grad: np.ndarray  # [n, E]


def dvd_loss(embeddings, length_scale: float, jitter: float, lam: float) -> DvdLossOut:
    """dvd_loss (evolve.hpp:411-465) on host embeddings (double)."""
    e = np.ascontiguousarray(embeddings, np.float64)
    if e.ndim != 2 or e.shape[0] < 2:
        raise ConfigError("dvd_loss: need at least two embedding rows")
    loss, logdet = C.c_double(), C.c_double()
    grad = np.zeros_like(e)
    _lib.call("pbrl_dvd_loss", _ptr(e, _lib.f64p), e.shape[0], e.shape[1], float(length_scale),
              float(jitter), float(lam), C.byref(loss), C.byref(logdet), _ptr(grad, _lib.f64p))
    return DvdLossOut(loss.value, logdet.value, grad)


def median_pairwise_distance(embeddings) -> float:
    """median_pairwise_distance (evolve.hpp:469-486)."""
    e = np.ascontiguousarray(embeddings, np.float64)
    out = C.c_double()
    _lib.call("pbrl_median_pairwise_distance", _ptr(e, _lib.f64p), e.shape[0],
              int(np.prod(e.shape[1:])) if e.ndim > 1 else 1, C.byref(out))
    return out.value


# ---------------------------------------------------------------------- CEM (evolve.hpp:221-297)
class CEMState:
    """CEMState (evolve.hpp:224-233) over the flat policy vectors of a TD3 population, resident
    on its device: mean / var (double [P]), the noise schedule and the last candidates."""

    def __init__(self, policies: "Td3State", mean=None, init_var: float = 0.0):
        self.pop = policies
        m = None if mean is None else np.ascontiguousarray(mean, np.float64)
        if m is not None and m.size != policies.param_count("policy"):
            raise ShapeError("cem_init: mean length != policy parameter count")
        h = C.c_void_p()
        _lib.call("pbrl_cem_create", policies.handle,
                  None if m is None else _ptr(m, _lib.f64p), float(init_var), C.byref(h))
        self._h = h
        self._keep = m
        self.noise_init, self.noise_final, self.noise_decay = 1e-2, 1e-3, 0.999
        self.elite_fraction = 0.5
        self._noise = 1e-2

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().pbrl_cem_destroy(h)
            except Exception:
                pass
            self._h = None

    def _push(self):
        _lib.call("pbrl_cem_set_params", self._h, self._noise, self.noise_final,
                  self.noise_decay, self.elite_fraction)

    @property
    def noise(self) -> float:
        return self._noise

    @noise.setter
    def noise(self, v: float) -> None:
        self._noise = float(v)

    def _get(self):
        P = self.pop.param_count("policy")
        mean, var = np.empty(P, np.float64), np.empty(P, np.float64)
        nz = C.c_double()
        _lib.call("pbrl_cem_get", self._h, _ptr(mean, _lib.f64p), _ptr(var, _lib.f64p),
                  C.byref(nz))
        return mean, var, nz.value

    @property
    def mean(self) -> np.ndarray:
        return self._get()[0]

    @property
    def var(self) -> np.ndarray:
        return self._get()[1]

    def candidates(self) -> np.ndarray:
        out = np.empty((self.pop.n, self.pop.param_count("policy")), np.float64)
        _lib.call("pbrl_cem_candidates", self._h, _ptr(out, _lib.f64p))
        return out


def cem_init(policies: "Td3State", mean=None, init_var: float = 0.0) -> CEMState:
    """cem_init (evolve.hpp:231-237); mean None = flatten_member(policy, 0) (pipeline_run.hpp:159)."""
    return CEMState(policies, mean, init_var)


def cem_resample(cem: CEMState, rng: RngSequence) -> np.ndarray:
    """cem_resample (pipeline_run.hpp:148-158): cem_sample(cem, n, rng) on the device, each
    candidate written into its member's policy, targets = policies, policy Adam reset.  Returns
    the candidates [n, P] (double)."""
    cem._push()
    nx = C.c_uint64(rng.next)
    _lib.call("pbrl_cem_resample", cem._h, rng.stream.key, C.byref(nx))
    rng.next = nx.value
    return cem.candidates()


def cem_update(cem: CEMState, scores) -> None:
    """cem_update (evolve.hpp:255-297) against the candidates of the last cem_resample."""
    sc = np.ascontiguousarray(scores, np.float64)
    cem._push()
    _lib.call("pbrl_cem_update", cem._h, _ptr(sc, _lib.f64p), sc.size)
    cem._noise = max(cem.noise_final, cem._noise * cem.noise_decay)


# ---------------------------------------------------------------------- checkpoints
def save_checkpoint(st, net, path) -> None:
    """save_checkpoint (net_pop.hpp:245-261): one network of the population as a PBRLNET1 file
    (fp32), readable by the reference's load_checkpoint."""
    _lib.call("pbrl_save_checkpoint", st._h, NETS.get(net, net), str(path).encode())


def load_checkpoint(st, net, path) -> None:
    """load_checkpoint (net_pop.hpp:264-296) into network `net` of an existing population (the
    file's population size, extents, activation and scale must match)."""
    _lib.call("pbrl_load_checkpoint", st._h, NETS.get(net, net), str(path).encode())


def serialize_state(st, path) -> None:
    """serialize_state (algos.hpp:989-1015): the TD3 state export, byte-identical layout."""
    _lib.call("pbrl_serialize_state", st._h, str(path).encode())


def deserialize_state(st, path) -> None:
    """Full-trainer resume from a serialize_state file (the inverse the reference lacks)."""
    _lib.call("pbrl_deserialize_state", st.handle, str(path).encode())


# ---------------------------------------------------------------------- action selection
def _act(st, obs, noise_std, seed, steps, deterministic):
    obs = np.ascontiguousarray(obs, np.float32)
    if obs.ndim != 3 or obs.shape[0] != st.n or obs.shape[2] != st.obs_dim:
        raise ShapeError(f"act: observations {list(obs.shape)} do not match "
                         f"[{st.n}, rows, {st.obs_dim}]")
    steps = np.ascontiguousarray(steps, np.uint64)
    if steps.shape != (st.n,):
        raise ShapeError("act: one step counter per member")
    ns = None
    if noise_std is not None:
        ns = np.ascontiguousarray(noise_std, np.float64)
        if ns.shape != (st.n,):
            raise ShapeError("act: one noise_std per member")
    out = np.empty((st.n, obs.shape[1], st.act_dim), np.float32)
    _lib.call("pbrl_act", st._h, _ptr(obs, _lib.f32p), obs.shape[1],
              _ptr(ns, _lib.f64p) if ns is not None else None, seed, _ptr(steps, _lib.u64p),
              1 if deterministic else 0, _ptr(out, _lib.f32p))
    return out


def act(st: "Td3State", obs, noise_std, seed: int, steps, deterministic: bool = False):
    """act (algos.hpp:895-915): tanh policy output plus clipped Gaussian exploration noise for
    every member, obs [n, rows, obs_dim] -> actions [n, rows, act_dim]; noise keyed by
    (seed, the state's member streams, kExploreNoise, steps[m])."""
    return _act(st, obs, noise_std, seed, steps, deterministic)


def sac_act(st: "SacState", obs, seed: int, steps, deterministic: bool = False):
    """sac_act (algos.hpp:918-942): bound * tanh(mu + sigma * eps), or the mode."""
    return _act(st, obs, None, seed, steps, deterministic)


# ---------------------------------------------------------------------- replay
@dataclass
class SnapshotMailbox:
    """SnapshotMailbox (pipeline.hpp:53-83), device-resident: the learner publishes its policy
    population (+ explore_std) into a device slot; actors adopt it with actor_refresh."""

    def __init__(self, learner: _Population):
        h = C.c_void_p()
        _lib.call("pbrl_mailbox_create", learner.handle, C.byref(h))
        self._h, self.n = h, learner.n

    def publish(self, learner: _Population, explore_std=None) -> int:
        v = C.c_uint64()
        ex = None if explore_std is None else np.ascontiguousarray(explore_std, np.float64)
        if ex is not None and ex.size != self.n:
            raise ShapeError(f"publish: explore_std has {ex.size} entries, population {self.n}")
        _lib.call("pbrl_mailbox_publish", self._h, learner.handle,
                  None if ex is None else _ptr(ex, _lib.f64p), C.byref(v))
        return v.value

    def version(self) -> int:
        v = C.c_uint64()
        _lib.call("pbrl_mailbox_version", self._h, C.byref(v))
        return v.value

    def checksum(self):
        """(version, ActorSnapshot::compute_checksum) of the newest snapshot."""
        v, c = C.c_uint64(), C.c_uint64()
        _lib.call("pbrl_mailbox_checksum", self._h, C.byref(v), C.byref(c))
        return v.value, c.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().pbrl_mailbox_destroy(h)
            except Exception:
                pass
            self._h = None


def actor_refresh(actor: _Population, mailbox: SnapshotMailbox):
    """actor_loop's refresh() (pipeline.hpp:270-279): adopt the newest snapshot into the
    actor's own population if its version changed.  Returns (version held, explore_std)."""
    v = C.c_uint64()
    ex = np.zeros(actor.n, np.float64)
    _lib.call("pbrl_actor_refresh", actor.handle, mailbox._h, C.byref(v), _ptr(ex, _lib.f64p))
    return v.value, ex


class Transition:
    """Transition (replay.hpp:17-24)."""
    s: Sequence[float]
    a: Sequence[float]
    s2: Sequence[float]
    r: float = 0.0
    done: float = 0.0
    member: int = 0
    seq: int = 0


class DeviceReplay:
    """ReplayBuffer (replay.hpp:28-173) for a whole population, resident in HBM.  Per-agent
    mode keeps one ring per member (buffer m feeds member m); shared mode keeps one ring."""

    def __init__(self, st: _Population, capacity: int, mode: str = "per_agent"):
        self.st = st
        self.capacity = int(capacity)
        self.mode = mode
        _lib.call("pbrl_replay_create", st.handle, self.capacity,
                  0 if mode in ("per_agent", "kPerAgent") else 1)

    def push(self, t: Transition) -> None:
        if len(t.s) != self.st.obs_dim or len(t.s2) != self.st.obs_dim or \
                len(t.a) != self.st.act_dim:
            raise UsageError("ReplayBuffer::push: transition dims do not match buffer dims")
        self.insert(np.asarray([t.s]), np.asarray([t.a]), np.asarray([t.r]),
                    np.asarray([t.s2]), np.asarray([t.done]), np.asarray([t.member]))

    def insert(self, s, a, r, s2, done, member) -> None:
        """Batched push: rows in order, each to the ring of its member (per-agent mode)."""
        s, a, r, s2, done = (_f32(x) for x in (s, a, r, s2, done))
        member = np.ascontiguousarray(member, dtype=np.uint32)
        cnt = member.size
        if s.size != cnt * self.st.obs_dim or a.size != cnt * self.st.act_dim:
            raise UsageError("ReplayBuffer::push: transition dims do not match buffer dims")
        _lib.call("pbrl_replay_insert", self.st.handle, _ptr(s, _lib.f32p), _ptr(a, _lib.f32p),
                  _ptr(r, _lib.f32p), _ptr(s2, _lib.f32p), _ptr(done, _lib.f32p),
                  _ptr(member, _lib.u32p), cnt)

    def size(self, buffer: int = 0) -> int:
        c = C.c_uint64()
        _lib.call("pbrl_replay_size", self.st.handle, buffer, C.byref(c))
        return c.value

    def save_snapshot(self, path, buffer: int = 0) -> None:
        """ReplayBuffer::save_snapshot (replay.hpp:113-139) of one ring, PBRLBUF1 format."""
        _lib.call("pbrl_replay_save_snapshot", self.st.handle, buffer, str(path).encode())

    def load_snapshot(self, path, buffer: int = 0) -> None:
        """ReplayBuffer::load_snapshot (replay.hpp:141-165) into one ring (same capacity / dims)."""
        _lib.call("pbrl_replay_load_snapshot", self.st.handle, buffer, str(path).encode())


def sample_batch(replay: DeviceReplay, batch_size: int, seed: int, draw_id: int,
                 min_size: int = 1) -> Optional[TransitionBatch]:
    """sample_batch (replay.hpp:181-204) gathered on device and returned to the host;
    None when a source ring holds fewer than max(min_size, 1) transitions."""
    st = replay.st
    n, ds, da = st.n, st.obs_dim, st.act_dim
    out = [np.empty((n, batch_size, ds), np.float32), np.empty((n, batch_size, da), np.float32),
           np.empty((n, batch_size, 1), np.float32), np.empty((n, batch_size, ds), np.float32),
           np.empty((n, batch_size, 1), np.float32)]
    ready = C.c_int()
    _lib.call("pbrl_sample_batch", st.handle, seed, draw_id, batch_size, min_size,
              *[_ptr(o, _lib.f32p) for o in out], C.byref(ready))
    return TransitionBatch(*out) if ready.value else None


def update_k_from_replay(st, replay: DeviceReplay, k: int, hyper, batch_size: int, seed: int,
                         first_draw_id: int, min_size: int = 1) -> bool:
    """The prefetch + learner loop of run_training (pipeline_run.hpp:230-355) fused on device:
    k x (sample_batch(draw_id = first + i) -> update step).  Returns False (nothing ran) when
    the replay is not ready."""
    st._sync_hyper(hyper)
    ready = C.c_int()
    _lib.call("pbrl_update_k", st.handle, k, seed, first_draw_id, batch_size, min_size,
              C.byref(ready))
    return bool(ready.value)


# ---------------------------------------------------------------------- PBT (evolve.hpp)
@dataclass
class HyperRange:
    """HyperRange (evolve.hpp:18-26)."""
    log_scale: bool = False
    lo: float = 0.0
    hi: float = 1.0

    def sample(self, rng: RngSequence) -> float:
        return rng.log_uniform(self.lo, self.hi) if self.log_scale else rng.uniform(self.lo, self.hi)

    def contains(self, v: float) -> bool:
        return self.lo <= v <= self.hi


@dataclass
class Td3Prior:
    """Td3Prior (evolve.hpp:31-49)."""
    critic_lr: HyperRange = field(default_factory=lambda: HyperRange(True, 3e-5, 3e-3))
    policy_lr: HyperRange = field(default_factory=lambda: HyperRange(True, 3e-5, 3e-3))
    policy_delay_ratio: HyperRange = field(default_factory=lambda: HyperRange(False, 0.2, 1.0))
    explore_std: HyperRange = field(default_factory=lambda: HyperRange(False, 0.0, 1.0))
    target_std: HyperRange = field(default_factory=lambda: HyperRange(False, 0.0, 1.0))
    discount: HyperRange = field(default_factory=lambda: HyperRange(False, 0.9, 1.0))

    def sample_member(self, rng: RngSequence) -> Td3Hyper:
        h = Td3Hyper.defaults(1)
        h.critic_lr[0] = self.critic_lr.sample(rng)
        h.policy_lr[0] = self.policy_lr.sample(rng)
        h.policy_delay_ratio[0] = self.policy_delay_ratio.sample(rng)
        h.explore_std[0] = self.explore_std.sample(rng)
        h.target_std[0] = self.target_std.sample(rng)
        h.gamma[0] = self.discount.sample(rng)
        return h


@dataclass
class SacPrior:
    """SacPrior (evolve.hpp:54-73)."""
    policy_lr: HyperRange = field(default_factory=lambda: HyperRange(True, 3e-5, 3e-3))
    critic_lr: HyperRange = field(default_factory=lambda: HyperRange(True, 3e-5, 3e-3))
    alpha_lr: HyperRange = field(default_factory=lambda: HyperRange(True, 3e-5, 3e-3))
    entropy_scale: HyperRange = field(default_factory=lambda: HyperRange(False, 0.2, 2.0))
    reward_scale: HyperRange = field(default_factory=lambda: HyperRange(False, 0.1, 10.0))
    discount: HyperRange = field(default_factory=lambda: HyperRange(False, 0.9, 1.0))
    default_target_entropy: float = -1.0

    def sample_member(self, rng: RngSequence) -> SacHyper:
        h = SacHyper.defaults(1, 1)
        h.policy_lr[0] = self.policy_lr.sample(rng)
        h.critic_lr[0] = self.critic_lr.sample(rng)
        h.alpha_lr[0] = self.alpha_lr.sample(rng)
        h.target_entropy[0] = self.entropy_scale.sample(rng) * self.default_target_entropy
        h.reward_scale[0] = self.reward_scale.sample(rng)
        h.gamma[0] = self.discount.sample(rng)
        return h


class PBTState:
    """PBTState (evolve.hpp:80-108): rolling returns per member + evolution cadence."""

    def __init__(self, n: int = 0):
        self.returns = [deque() for _ in range(n)]
        self.ring_capacity = 10
        self.steps_since_evolve = 0
        self.evolve_interval = 100000
        self.truncation_fraction = 0.3

    def members(self) -> int:
        return len(self.returns)

    def record_return(self, member: int, ep_return: float) -> None:
        ring = self.returns[member]
        ring.append(float(ep_return))
        while len(ring) > self.ring_capacity:
            ring.popleft()

    def every_member_scored(self) -> bool:
        return bool(self.returns) and all(len(r) for r in self.returns)

    def mean_return(self, member: int) -> float:
        acc = 0.0
        for v in self.returns[member]:  # std::accumulate, left to right
            acc += v
        return acc / float(len(self.returns[member]))

    def fitness(self) -> np.ndarray:
        if not self.every_member_scored():
            raise NotReadyError("pbt_rank: every member needs at least one recorded return")
        return np.asarray([self.mean_return(m) for m in range(self.members())], np.float64)


@dataclass
class EvolvePlan:
    """EvolvePlan (evolve.hpp:125-128): replaced[i] copies from donors[i]."""
    replaced: List[int]
    donors: List[int]


def _rank_key(f: float) -> float:
    """Sort key of a fitness value: NaN (a diverged member) ranks as -inf, i.e. last, so the
    ranking is a total order (the reference's comparator is undefined for NaN)."""
    return -math.inf if math.isnan(f) else f


def pbt_rank(st: PBTState) -> List[int]:
    """pbt_rank (evolve.hpp:112-122): best first, ties toward the lower index."""
    f = st.fitness()
    return sorted(range(len(f)), key=lambda i: (-_rank_key(f[i]), i))


def pbt_plan(st: PBTState, rng: RngSequence, pop: _Population) -> Optional[EvolvePlan]:
    """pbt_plan (evolve.hpp:133-145), ranked and drawn on the device of `pop`."""
    n = st.members()
    if n < 4:
        return None
    fit = st.fitness()
    rep = np.zeros(n, np.uint64)
    don = np.zeros(n, np.uint64)
    nxt = C.c_uint64(rng.next)
    cnt = C.c_uint32()
    _lib.call("pbrl_pbt_plan", pop.handle, _ptr(fit, _lib.f64p), n, st.truncation_fraction,
              rng.stream.key, C.byref(nxt), _ptr(rep, _lib.u64p), _ptr(don, _lib.u64p),
              C.byref(cnt))
    rng.next = nxt.value
    c = cnt.value
    return EvolvePlan([int(x) for x in rep[:c]], [int(x) for x in don[:c]])


def pbt_apply_returns_reset(st: PBTState, plan: EvolvePlan) -> None:
    """pbt_apply_returns_reset (evolve.hpp:149-152)."""
    for m in plan.replaced:
        st.returns[m].clear()
    st.steps_since_evolve = 0


def pbt_evolve_trainer(st: PBTState, trainer: _Population, hyper, prior, rng: RngSequence
                       ) -> Optional[EvolvePlan]:
    """pbt_evolve_trainer (evolve.hpp:169-213): device ranking + donor draw, device copies of
    every network and optimiser reset, hyper re-draw on the host (bit-exact libm)."""
    plan = pbt_plan(st, rng, trainer)
    if plan is None:
        return None
    apply_plan(trainer, plan)
    for dst in plan.replaced:
        hyper.set_member(dst - trainer.member_offset, prior.sample_member(rng))
    pbt_apply_returns_reset(st, plan)
    return plan


def apply_plan(trainer: _Population, plan: EvolvePlan) -> None:
    k = len(plan.replaced)
    rep = np.asarray(plan.replaced, np.uint64)
    don = np.asarray(plan.donors, np.uint64)
    _lib.call("pbrl_pbt_apply", trainer.handle, _ptr(rep, _lib.u64p), _ptr(don, _lib.u64p), k)


def member_blob_size(pop: _Population) -> int:
    c = C.c_uint64()
    _lib.call("pbrl_member_blob_size", pop.handle, C.byref(c))
    return c.value


def export_member(pop: _Population, member: int, dev_ptr: int) -> None:
    _lib.call("pbrl_export_member", pop.handle, member, C.c_void_p(dev_ptr))


def import_member(pop: _Population, member: int, dev_ptr: int) -> None:
    _lib.call("pbrl_import_member", pop.handle, member, C.c_void_p(dev_ptr))


def plan_from_fitness(fitness: Sequence[float], trunc: float, rng: RngSequence
                      ) -> Tuple[List[int], List[int]]:
    """pbt_plan (evolve.hpp:133-145) on the host from per-member fitness: stable rank (best
    first, ties toward the lower index), bottom ceil(trunc*N) replaced by donors drawn uniformly
    from the top ceil(trunc*N).  Same semantics as the device kernel behind pbrl_pbt_plan."""
    n = len(fitness)
    if n < 4:
        return [], []
    order = sorted(range(n), key=lambda i: (-_rank_key(float(fitness[i])), i))
    cut = int(math.ceil(trunc * n))
    replaced, donors = [], []
    for i in range(cut):
        replaced.append(order[n - 1 - i])
        donors.append(order[rng.index(cut)])
    return replaced, donors
