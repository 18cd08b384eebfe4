"""ctypes binding of the C ABI in include/pbrl_b200.h (libpbrl_b200.so, built in-tree).

There is no fallback: if the CUDA library is missing or fails to load, importing the
population API raises.  This is the binding a reference-side maintainer would add (see
INTEGRATION.md); the rest of the package only uses the symbols declared here.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import raise_for

LIB_PATH = Path(__file__).resolve().parent / "libpbrl_b200.so"

u64 = C.c_uint64
u32 = C.c_uint32
i64 = C.c_int64
dbl = C.c_double
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
u8p = C.POINTER(C.c_uint8)
i64p = C.POINTER(C.c_int64)
intp = C.POINTER(C.c_int)
vp = C.c_void_p


class PopDesc(C.Structure):
    _fields_ = [("algo", C.c_int), ("n", u64), ("obs_dim", u64), ("act_dim", u64),
                ("n_hidden", u32), ("hidden", u64p), ("action_bound", dbl), ("seed", u64),
                ("precision", C.c_int), ("device", C.c_int), ("member_offset", u64),
                ("n_global", u64), ("mode", C.c_int)]


class Batch(C.Structure):
    _fields_ = [("s", vp), ("a", vp), ("r", vp), ("s2", vp), ("done", vp)]


class P2POp(C.Structure):
    _fields_ = [("peer", C.c_int), ("is_send", C.c_int), ("buf", f32p), ("floats", u64)]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, vp, f64p, u64, f64p)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, vp, C.POINTER(P2POp), u32)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, vp, f32p, u64)


class CommOps(C.Structure):
    _fields_ = [("ctx", vp), ("allgather_f64", ALLGATHER_FN), ("exchange", EXCHANGE_FN),
                ("allreduce_f32", ALLREDUCE_FN)]


# name -> (restype, argtypes); every function returns an int status
SIGNATURES = {
    "pbrl_attach_comm": [vp, vp],
    "pbrl_update_k_masked": [vp, u32, u64, u64, u64, u64, u8p, intp],
    "pbrl_set_dvd": [vp, f64p, u64, dbl, dbl, dbl],
    "pbrl_dvd_embed": [vp, f64p, u64, f32p],
    "pbrl_dvd_loss": [f64p, u64, u64, dbl, dbl, dbl, f64p, f64p, f64p],
    "pbrl_median_pairwise_distance": [f64p, u64, u64, f64p],
    "pbrl_dvd_lambda": [u64, dbl, dbl, u64, f64p],
    "pbrl_cem_create": [vp, f64p, dbl, C.POINTER(vp)],
    "pbrl_cem_destroy": [vp],
    "pbrl_cem_set_params": [vp, dbl, dbl, dbl, dbl],
    "pbrl_cem_get": [vp, f64p, f64p, f64p],
    "pbrl_cem_resample": [vp, u64, C.POINTER(u64)],
    "pbrl_cem_candidates": [vp, f64p],
    "pbrl_cem_update": [vp, f64p, u64],
    "pbrl_pop_create": [C.POINTER(PopDesc), C.POINTER(vp)],
    "pbrl_pop_destroy": [vp],
    "pbrl_last_error": [C.c_char_p, C.c_size_t],
    "pbrl_version": [intp, intp],
    "pbrl_set_hyper": [vp, C.c_char_p, f64p],
    "pbrl_get_hyper": [vp, C.c_char_p, f64p],
    "pbrl_param_count": [vp, C.c_int, u64p],
    "pbrl_get_member": [vp, C.c_int, u64, f32p],
    "pbrl_set_member": [vp, C.c_int, u64, f32p],
    "pbrl_copy_member": [vp, C.c_int, u64, u64],
    "pbrl_get_adam": [vp, C.c_int, u64, f32p, f32p, i64p],
    "pbrl_get_counters": [vp, f64p, u64p],
    "pbrl_get_alpha": [vp, f32p, f32p, f32p, i64p],
    "pbrl_update_batches": [vp, C.POINTER(Batch), u32, u64, u8p],
    "pbrl_update_batches_device": [vp, C.POINTER(Batch), u32, u64, u8p],
    "pbrl_update_batches_losses": [vp, C.POINTER(Batch), u32, u64, u8p, f64p],
    "pbrl_act": [vp, f32p, u64, f64p, u64, u64p, C.c_int, f32p],
    "pbrl_save_checkpoint": [vp, C.c_int, C.c_char_p],
    "pbrl_load_checkpoint": [vp, C.c_int, C.c_char_p],
    "pbrl_serialize_state": [vp, C.c_char_p],
    "pbrl_deserialize_state": [vp, C.c_char_p],
    "pbrl_replay_save_snapshot": [vp, u64, C.c_char_p],
    "pbrl_replay_load_snapshot": [vp, u64, C.c_char_p],
    "pbrl_update_k": [vp, u32, u64, u64, u64, u64, intp],
    "pbrl_last_losses": [vp, f64p, f64p, f64p],
    "pbrl_replay_create": [vp, u64, C.c_int],
    "pbrl_replay_insert": [vp, f32p, f32p, f32p, f32p, f32p, u32p, u64],
    "pbrl_replay_size": [vp, u64, u64p],
    "pbrl_sample_batch": [vp, u64, u64, u64, u64, f32p, f32p, f32p, f32p, f32p, intp],
    "pbrl_pbt_plan": [vp, f64p, u64, dbl, u64, u64p, u64p, u64p, u32p],
    "pbrl_pbt_apply": [vp, u64p, u64p, u32],
    "pbrl_pbt_evolve": [vp, f64p, u64, u64p, u64p, u64p, u32p],
    "pbrl_member_blob_size": [vp, u64p],
    "pbrl_export_member": [vp, u64, vp],
    "pbrl_import_member": [vp, u64, vp],
    "pbrl_launch_count": [vp, u64p],
    "pbrl_debug_tc_trace": [u64p, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int)],
    "pbrl_synchronize": [vp],
    "pbrl_get_stream": [vp, C.POINTER(vp)],
    "pbrl_profile_begin": [vp],
    "pbrl_profile_end": [vp, C.c_char_p, C.c_size_t],
    "pbrl_device_bytes": [vp, u64p],
    "pbrl_selftest_libm": [C.c_int, vp, vp, u64],
    "pbrl_selftest_tc_gemm": [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp,
                              C.c_longlong, C.c_longlong, vp, C.c_longlong, C.c_longlong, vp,
                              C.c_longlong, C.c_longlong],
    "pbrl_selftest_tc_gemm_bf16": [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp,
                                   C.c_longlong, C.c_longlong, vp, C.c_longlong, C.c_longlong,
                                   vp, C.c_longlong, C.c_longlong],
    "pbrl_synthetic_batches_device": [vp, u64, u64, u64, u64, u64, u64, C.POINTER(Batch)],
    "pbrl_copy_member_state": [vp, u64, vp, u64],
    "pbrl_mailbox_create": [vp, C.POINTER(vp)],
    "pbrl_mailbox_destroy": [vp],
    "pbrl_mailbox_publish": [vp, vp, f64p, u64p],
    "pbrl_mailbox_version": [vp, u64p],
    "pbrl_actor_refresh": [vp, vp, u64p, f64p],
    "pbrl_mailbox_checksum": [vp, u64p, u64p],
    "pbrl_nccl_unique_id": [vp, C.c_size_t],
    "pbrl_comm_create_nccl": [vp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)],
    "pbrl_comm_create_host": [C.POINTER(CommOps), C.c_int, C.c_int, C.c_int, C.POINTER(vp)],
    "pbrl_comm_destroy": [vp],
    "pbrl_pbt_evolve_sharded": [vp, vp, f64p, C.c_int, dbl, u64, u64p, u64p, u64p, u32p, f64p],
}

_lib = None


def lib():
    """Load libpbrl_b200.so once; raises if the CUDA extension is absent (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() or "
                              f"`make -C paper_2206_08888_b200`")
        L = C.CDLL(str(LIB_PATH))
        for name, args in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = C.c_int
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    buf = C.create_string_buffer(4096)
    lib().pbrl_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def call(name: str, *args) -> None:
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise_for(rc, f"{name}: {last_error()}")
