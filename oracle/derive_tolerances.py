"""TEST INFRASTRUCTURE: derives the TF32 / BF16 parity tolerances on the CPU, from the
restatement oracle and the reference, instead of calibrating them on the GPU.

For every parity case (the configurations the GPU tests run, incl. SURVEY.md §8(d) configs A, C,
D and E) three CPU runs of the same K update steps on the same synthetic batches are compared:

1. fp32 truth: the C restatement (oracle/pbrl_oracle.c), bit-identical to the unmodified
   reference ``Td3State<float>`` / ``SacState<float>`` (tests/test_oracle_vs_ref.py);
2. fp64: the unmodified reference instantiated for ``double`` (algos.hpp:181-212, :490-521),
   when oracle/_ref is built -- SURVEY.md Appendix A's "oracle's own fp32-vs-fp64 discrepancy",
   recorded to show that the fp32 truth is far inside every tolerance below;
3. precision-p emulation: the restatement with both operands of every tensor-core product
   (hidden-layer forward, dX and dW; ``ora_set_emulation``) rounded to p -- TF32: the low 13
   mantissa bits dropped, BF16: round-to-nearest-even to 8 significant bits -- and everything
   the library keeps in fp32 (output layers, biases, losses, TD target, Adam, Polyak) exact.

The metrics are the ones the GPU tests evaluate:

  loss error    per step, max over members of |L_p - L| / max(|L|, 1e-3)   (critic1, critic2,
                policy losses)
  delta error   per network, ||(w_p,K - w0) - (w_K - w0)|| / ||w_K - w0||

and a case's tolerance for precision p is ``SAFETY x`` the emulated run's error (the GPU run is
another realisation of the same rounding, with a different accumulation order inside the
tensor core), never below FLOOR.  The scaling rule of Appendix A (fp32-vs-fp64 drift times
u_p/u_fp32) is recorded next to it for comparison: with Adam's sign-driven first steps the
weight-delta error grows like sqrt(u) rather than u, so that rule over- or under-shoots by
orders of magnitude depending on the metric; the emulation measures the effect directly.

    python oracle/derive_tolerances.py [case ...]   # rewrites tests/golden/tolerances.json
"""
from __future__ import annotations

import json
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Oracle, load_ref, sac_defaults, td3_defaults  # noqa: E402

OUT = ROOT / "tests" / "golden" / "tolerances.json"
TD3_NETS = ("policy", "policy_target", "critic1", "critic2", "critic1_target", "critic2_target")
SAC_NETS = ("policy", "critic1", "critic2", "critic1_target", "critic2_target")

U = {"fp32": 2.0 ** -24, "tf32": 2.0 ** -11, "bf16": 2.0 ** -9}
EMUL = {"tf32": 1, "bf16": 2}
SAFETY = 3.0
FLOOR = {"loss": 2e-3, "delta": 5e-3}

# name -> dict(algo, n, hidden, batch, K, seed, ds, da, ratio); ratio = TD3 policy_delay_ratio
# (None: the default 0.5, i.e. fire and non-fire steps).  The GPU parity tests run exactly these.
CASES = {
    # SURVEY.md §8(d) config A shape (policy firing every step)
    "A_td3_pop4": dict(algo="td3", n=4, hidden=[256, 256], batch=256, K=6, seed=7, ratio=1.0),
    "A_sac_pop4": dict(algo="sac", n=4, hidden=[256, 256], batch=256, K=6, seed=7),
    # fused output widths outside 1 / 6 / 12
    "W_td3_da3": dict(algo="td3", n=3, hidden=[256, 256], batch=128, K=4, seed=11, ds=11, da=3,
                      ratio=1.0),
    "W_sac_da8": dict(algo="sac", n=3, hidden=[256, 256], batch=128, K=4, seed=11, ds=9, da=8),
    # fused-forward hidden shapes
    "H_td3_128x96": dict(algo="td3", n=3, hidden=[128, 96], batch=128, K=4, seed=5, ratio=1.0),
    "H_sac_128x128": dict(algo="sac", n=3, hidden=[128, 128], batch=128, K=4, seed=5),
    "H_td3_256x64": dict(algo="td3", n=3, hidden=[256, 64], batch=128, K=4, seed=5, ratio=1.0),
    "H_td3_3x512": dict(algo="td3", n=2, hidden=[512, 512, 512], batch=256, K=3, seed=3,
                        ratio=1.0),
    # config D shape at pop 40 / 80: > 148 tiles per grouped GEMM, several tiles per CTA
    "D_td3_pop40": dict(algo="td3", n=40, hidden=[256, 256], batch=256, K=4, seed=7),
    "D_td3_pop80": dict(algo="td3", n=80, hidden=[256, 256], batch=256, K=4, seed=7),
    # config C: SAC pop 32
    "C_sac_pop32": dict(algo="sac", n=32, hidden=[256, 256], batch=256, K=4, seed=7),
    # config E: 3 x 512, batch 1024, pop 8
    "E_td3_pop8": dict(algo="td3", n=8, hidden=[512, 512, 512], batch=1024, K=2, seed=7),
    # shared-critic mode: one critic pair on the folded batch
    "S_td3_shared_pop8": dict(algo="td3", n=8, hidden=[256, 256], batch=256, K=4, seed=7,
                              shared=True),
    "S_td3_shared_pop80": dict(algo="td3", n=80, hidden=[256, 256], batch=256, K=3, seed=7,
                               shared=True),
    "S_sac_shared_pop8": dict(algo="sac", n=8, hidden=[256, 256], batch=256, K=4, seed=7,
                              shared=True),
    # shared critic + the DvD policy-gradient hook (10 probe states, lambda 0.5)
    "S_td3_dvd_pop8": dict(algo="td3", n=8, hidden=[256, 256], batch=256, K=4, seed=7,
                           shared=True, dvd=dict(ms=10, length_scale=0.7, lam=0.5, seed=3)),
}


def dvd_cfg(d, ds):
    """the DvD hook of a parity case: probe states U[-1, 1) from numpy's PCG64(seed)"""
    if not d:
        return None
    probe = np.random.default_rng(d["seed"]).uniform(-1.0, 1.0, (d["ms"], ds))
    return {"probe": probe, "length_scale": d["length_scale"], "jitter": 1e-6,
            "lam_start": d["lam"], "lam_end": d["lam"], "horizon": 1, "step": 0}


def case_args(c):
    return dict(algo=c["algo"], n=c["n"], hidden=list(c["hidden"]), batch=c["batch"], K=c["K"],
                seed=c["seed"], ds=c.get("ds", 17), da=c.get("da", 6), ratio=c.get("ratio"),
                shared=bool(c.get("shared", False)), dvd=c.get("dvd"))


def hyper_for(algo, n, da, ratio):
    hy = td3_defaults(n) if algo == "td3" else sac_defaults(n, da)
    if algo == "td3" and ratio is not None:
        hy["policy_delay_ratio"] = [ratio] * n
    return hy


def run(lib, algo, n, hidden, batch, K, seed, ds, da, ratio, dtype=np.float32, raw=None,
        shared=False, dvd=None):
    """K steps on `lib` (Oracle or Ref); returns (losses [K][3][n] or [K][3], w0, wK)."""
    nets = TD3_NETS if algo == "td3" else SAC_NETS
    make = lib.td3 if algo == "td3" else lib.sac
    st = make(n, ds, da, hidden, 1.0, seed, shared=shared) if isinstance(lib, Oracle) else \
        make(n, ds, da, hidden, 1.0, seed, dtype=dtype, shared=shared)
    hy = hyper_for(algo, n, da, ratio)
    w0 = {net: st.get_net(net).astype(np.float64) for net in nets}
    losses = []
    for k in range(K):
        b = tuple(x[k] for x in raw)
        if dvd:
            lk = st.step(b, hy, dvd=dvd_cfg(dvd, ds))
            losses.append(lk if isinstance(lib, Oracle) else np.zeros(3))
            continue
        losses.append(st.step(b, hy) if isinstance(lib, Oracle) or shared
                      else st.step(b, hy, want_losses=True))
    wk = {net: st.get_net(net).astype(np.float64) for net in nets}
    return np.asarray(losses), w0, wk


def loss_err(l, lt):
    """per step: max over members and losses of |l - lt| / max(|lt|, 1e-3)"""
    return np.max(np.abs(l - lt) / np.maximum(np.abs(lt), 1e-3), axis=tuple(range(1, lt.ndim)))


def delta_err(w, wt, w0):
    dt, d = wt - w0, w - w0
    den = np.linalg.norm(dt)
    return float(np.linalg.norm(d - dt) / den) if den > 0 else float(np.linalg.norm(d))


def derive(ora: Oracle, ref, c):
    a = case_args(c)
    raw = ora.synthetic_batches(a["K"], a["n"], a["batch"], a["ds"], a["da"], a["seed"])
    ora.set_emulation(0)
    lt, w0, wt = run(ora, raw=raw, **a)
    out = {"emulated": {}, "tol": {}}
    for p, mode in EMUL.items():
        ora.set_emulation(mode)
        try:
            lp, _, wp = run(ora, raw=raw, **a)
        finally:
            ora.set_emulation(0)
        le = loss_err(lp, lt)
        de = {net: delta_err(wp[net], wt[net], w0[net]) for net in wt}
        out["emulated"][p] = {"loss_per_step": le.tolist(), "delta": de}
        out["tol"][p] = {"loss": max(FLOOR["loss"], SAFETY * float(le.max())),
                         "delta": {net: max(FLOOR["delta"], SAFETY * v) for net, v in de.items()}}
    if ref is not None:
        l32, w032, w32 = run(ref, raw=raw, dtype=np.float32, **a)
        l64, w064, w64 = run(ref, raw=raw, dtype=np.float64, **a)
        # the reference reports member-summed losses: relative to the largest |L| of the run
        dl = float(np.max(np.abs(l32 - l64)) / np.max(np.abs(l64)))
        dn = {net: delta_err(w32[net] - w032[net] + w064[net], w64[net], w064[net])
              for net in w32}
        out["fp32_vs_fp64"] = {"loss": dl, "delta": dn}
        out["appendix_a_rule"] = {
            p: {"loss": dl * U[p] / U["fp32"],
                "delta": {net: v * U[p] / U["fp32"] for net, v in dn.items()}}
            for p in EMUL}
    return out


def load():
    return json.loads(OUT.read_text()) if OUT.exists() else {"cases": {}}


def main(names=None):
    ora = Oracle()
    ref = load_ref()
    doc = load()
    doc.update({"_doc": "generated by oracle/derive_tolerances.py (see its docstring)",
                "u": U, "safety": SAFETY, "floor": FLOOR})
    for name, c in CASES.items():
        if names and name not in names:
            continue
        t0 = time.time()
        res = derive(ora, ref, c)
        doc["cases"][name] = {**case_args(c), **res}
        em = res["emulated"]
        print(f"{name}: tf32 loss {max(em['tf32']['loss_per_step']):.2e} "
              f"delta {max(em['tf32']['delta'].values()):.3f} | bf16 loss "
              f"{max(em['bf16']['loss_per_step']):.2e} delta "
              f"{max(em['bf16']['delta'].values()):.3f} | fp64 drift "
              f"{res.get('fp32_vs_fp64', {}).get('loss', math.nan):.1e} "
              f"({time.time() - t0:.0f} s)", flush=True)
        OUT.write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:] or None)
