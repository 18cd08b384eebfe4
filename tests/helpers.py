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


# ---------------------------------------------------------------- derived TF32 / BF16 tolerances
# tests/golden/tolerances.json is written by oracle/derive_tolerances.py: per parity case, the
# error of a CPU run whose tensor-core operands are rounded to TF32 / BF16 against the exact fp32
# oracle, times a safety factor (see that script's docstring).  The GPU run must stay inside it.
_TOL = None


def tolerances():
    global _TOL
    if _TOL is None:
        import json
        from pathlib import Path
        _TOL = json.loads((Path(__file__).parent / "golden" / "tolerances.json").read_text())
    return _TOL


def parity_case(pb, ora, name, precision, device=0):
    """Runs derived-tolerance case `name` on the GPU in `precision` and on the exact fp32 oracle,
    same batches and hypers.  Returns (loss error per step, {net: weight-delta error}) with the
    metrics of oracle/derive_tolerances.py."""
    c = tolerances()["cases"][name]
    algo, n, hidden, B, K, seed = c["algo"], c["n"], c["hidden"], c["batch"], c["K"], c["seed"]
    ds, da, ratio = c["ds"], c["da"], c["ratio"]
    shared = bool(c.get("shared", False))
    make = pb.make_td3_state if algo == "td3" else pb.make_sac_state
    st = make(n, ds, da, hidden, 1.0, seed, precision=precision, device=device,
              mode="shared_critic" if shared else "independent")
    ora.set_emulation(0)
    ref = (ora.td3 if algo == "td3" else ora.sac)(n, ds, da, hidden, 1.0, seed, shared=shared)
    hy = pb.Td3Hyper.defaults(n) if algo == "td3" else pb.SacHyper.defaults(n, da)
    if algo == "td3" and ratio is not None:
        hy.policy_delay_ratio = [ratio] * n
    oh = {f: list(getattr(hy, f)) for f in hy.FIELDS}
    nets = TD3_NETS if algo == "td3" else SAC_NETS
    w0 = {net: ref.get_net(net).astype(np.float64) for net in nets}
    raw = ora.synthetic_batches(K, n, B, ds, da, seed)
    upd = pb.td3_update_step if algo == "td3" else pb.sac_update_step
    dcfg, hook = None, None
    if c.get("dvd"):
        d = c["dvd"]
        probe = np.random.default_rng(d["seed"]).uniform(-1.0, 1.0, (d["ms"], ds))
        dcfg = {"probe": probe, "length_scale": d["length_scale"], "jitter": 1e-6,
                "lam_start": d["lam"], "lam_end": d["lam"], "horizon": 1, "step": 0}
        cfg = pb.DvDConfig(probe.ravel(), d["ms"], d["length_scale"], 1e-6,
                           pb.LambdaSchedule(d["lam"], d["lam"], 1))
        hook = pb.dvd_policy_hook(cfg, 0)
    lerr = []
    for k in range(K):
        if hook is not None:
            upd(st, to_batch(pb, raw, k), hy, hook=hook)
        else:
            upd(st, to_batch(pb, raw, k), hy)
        dl = np.stack(st.last_losses()).astype(np.float64)
        rl = ref.step(raw_at(raw, k), oh) if dcfg is None else ref.step(raw_at(raw, k), oh,
                                                                         dvd=dcfg)
        lerr.append(float(np.max(np.abs(dl - rl) / np.maximum(np.abs(rl), 1e-3))))
    werr = {net: rel_delta_err(st.params(net), ref.get_net(net), w0[net]) for net in nets}
    return np.asarray(lerr), werr


def check_parity(pb, ora, name, precision):
    lerr, werr = parity_case(pb, ora, name, precision)
    tol = tolerances()["cases"][name]["tol"][precision]
    emu = tolerances()["cases"][name]["emulated"][precision]
    print(f"\n{name} {precision}: loss err {lerr.max():.2e} (tol {tol['loss']:.2e}, "
          f"CPU emulation {max(emu['loss_per_step']):.2e}); delta err "
          + ", ".join(f"{k} {v:.4f}/{tol['delta'][k]:.4f}" for k, v in werr.items()))
    assert lerr.max() <= tol["loss"], (lerr.tolist(), tol["loss"])
    for net, e in werr.items():
        assert e <= tol["delta"][net], (net, e, tol["delta"][net])
