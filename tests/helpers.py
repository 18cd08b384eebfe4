"""Shared helpers for the parity tests."""
from __future__ import annotations

import numpy as np

TD3_NETS = ("policy", "policy_target", "critic1", "critic2", "critic1_target", "critic2_target")
SAC_NETS = ("policy", "critic1", "critic2", "critic1_target", "critic2_target")


def bits_equal(a, b) -> bool:
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def to_batch(pb, raw, k=None):
    """Oracle-layout batch (s, a, r[N,B], s2, d[N,B]) -> package TransitionBatch (host)."""
    s, a, r, s2, d = raw if k is None else (x[k] for x in raw)
    return pb.TransitionBatch(s, a, r[..., None], s2, d[..., None])


def raw_at(raw, k):
    return tuple(x[k] for x in raw)


def rel_delta_err(w_dev, w_ref, w0):
    """||(w_dev - w0) - (w_ref - w0)|| / ||w_ref - w0|| (SURVEY.md Appendix A tolerance metric)."""
    dref = np.asarray(w_ref, np.float64) - np.asarray(w0, np.float64)
    ddev = np.asarray(w_dev, np.float64) - np.asarray(w0, np.float64)
    den = np.linalg.norm(dref)
    return float(np.linalg.norm(ddev - dref) / den) if den > 0 else float(np.linalg.norm(ddev))
