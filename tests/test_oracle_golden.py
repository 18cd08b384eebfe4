"""The C restatement oracle against golden vectors produced by the unmodified reference build
(tests/golden/, written by oracle/make_golden.py).  Runs without /root/reference and without a
GPU, so the checker used by the GPU parity tests is pinned on every machine."""
from pathlib import Path

import numpy as np
import pytest

from helpers import SAC_NETS, TD3_NETS, bits_equal, raw_at

GOLD = Path(__file__).resolve().parent / "golden"


def _load(name):
    p = GOLD / f"{name}.npz"
    if not p.exists():
        pytest.skip(f"{p} missing (python oracle/make_golden.py)")
    return np.load(p)


@pytest.mark.parametrize("name", ["td3_small", "td3_halfcheetah"])
def test_td3_golden(ora, name):
    g = _load(name)
    n, ds, da, B, K = (int(g[k]) for k in ("n", "ds", "da", "B", "K"))
    st = ora.td3(n, ds, da, [int(h) for h in g["hidden"]], float(g["bound"]), int(g["seed"]))
    for k in TD3_NETS:
        assert bits_equal(st.get_net(k), g[f"init_{k}"]), k
    hy = {f[len("hyper_"):]: list(g[f]) for f in g.files if f.startswith("hyper_")}
    raw = ora.synthetic_batches(K, n, B, ds, da, int(g["bseed"]))
    for k in range(K):
        lo = st.step(raw_at(raw, k), hy)
        assert lo[0].sum() == pytest.approx(g["losses"][k][0], rel=1e-12)
        assert lo[1].sum() == pytest.approx(g["losses"][k][1], rel=1e-12)
    for k in TD3_NETS:
        assert bits_equal(st.get_net(k), g[f"final_{k}"]), k
    for k in ("policy", "critic1", "critic2"):
        for m in range(n):
            mo, vo, t = st.get_adam(k, m)
            assert bits_equal(mo, g[f"adam_m_{k}"][m]) and bits_equal(vo, g[f"adam_v_{k}"][m])
            assert t == g[f"adam_t_{k}"][m]
    da_, steps = st.counters()
    assert np.array_equal(da_, g["delay_acc"]) and np.array_equal(steps, g["steps"])


def test_sac_golden(ora):
    g = _load("sac_small")
    n, ds, da, B, K = (int(g[k]) for k in ("n", "ds", "da", "B", "K"))
    st = ora.sac(n, ds, da, [int(h) for h in g["hidden"]], 1.0, int(g["seed"]))
    from oracle.oracle import sac_defaults
    hy = sac_defaults(n, da)
    raw = ora.synthetic_batches(K, n, B, ds, da, int(g["bseed"]))
    for k in range(K):
        st.step(raw_at(raw, k), hy)
    for k in SAC_NETS:
        assert bits_equal(st.get_net(k), g[f"final_{k}"]), k
    la, am, av, at, steps = st.counters()
    assert bits_equal(la, g["log_alpha"]) and bits_equal(am, g["alpha_m"])
    assert np.array_equal(at, g["alpha_t"]) and np.array_equal(steps, g["steps"])


def test_rng_golden(ora):
    g = _load("rng")
    for row, uni, nrm in zip(g["keys"], g["uniform"], g["normal"]):
        seed, stream, use, step, key = (int(x) for x in row)
        assert ora.stream_key(seed, stream, use, step) == key
        assert [ora.uniform(key, c) for c in range(16)] == list(uni)
        assert [ora.normal_pair(key, 2 * c) for c in range(16)] == list(nrm)


def test_replay_golden(ora):
    g = _load("replay")
    n, cap, B = 3, int(g["cap"]), int(g["B"])
    bufs = [ora.replay(cap, 4, 2) for _ in range(n)]
    for i, m in enumerate(g["member"]):
        bufs[m].push(g["s"][i], g["a"][i], g["r"][i], g["s2"][i], g["d"][i], int(m))
    for draw in (0, 3):
        got = ora.sample_batch(bufs, B, 0, n, 77, [0, 1, 2], draw)
        for x, k in zip(got[:5], ("s", "a", "r", "s2", "d")):
            assert bits_equal(x, g[f"draw{draw}_{k}"])


def test_pbt_golden(ora):
    g = _load("pbt")
    for n in (4, 10, 33, 80):
        rings, counts = g[f"n{n}_rings"], g[f"n{n}_counts"]
        assert np.array_equal(ora.pbt_rank(rings, counts), g[f"n{n}_order"])
        rep, don, nxt = ora.pbt_plan(rings, counts, 0.3, int(g[f"n{n}_key"]), 7)
        assert np.array_equal(rep, g[f"n{n}_replaced"]) and np.array_equal(don, g[f"n{n}_donors"])
        assert nxt == int(g[f"n{n}_next"])


def test_tanhf_golden():
    """The libm tanhf the reference calls (glibc fdlibm) == the fixture; the device port of the
    same algorithm is checked on the GPU in test_gpu_numerics.py."""
    import ctypes as C
    g = _load("tanhf")
    libm = C.CDLL("libm.so.6")
    libm.tanhf.restype = C.c_float
    libm.tanhf.argtypes = [C.c_float]
    got = np.asarray([libm.tanhf(float(v)) for v in g["x"]], np.float32)
    assert bits_equal(got, g["y"])


def test_act_golden(ora):
    """act / sac_act of the restatement vs the reference's outputs (algos.hpp:895-942)."""
    g = _load("act")
    for algo in ("td3", "sac"):
        st = (ora.td3 if algo == "td3" else ora.sac)(int(g["n"]), int(g["ds"]), int(g["da"]),
                                                     [int(h) for h in g["hidden"]], 1.0,
                                                     int(g["state_seed"]))
        for det in (0, 1):
            got = st.act(g["obs"], int(g["seed"]), g["steps"], g["noise"], bool(det))
            assert bits_equal(got, g[f"{algo}_det{det}"]), (algo, det)


def test_f4_golden(ora):
    """shared-critic TD3 (+ member mask, DvD hook) / SAC, dvd_loss, median, CEM: the oracle
    against the reference's outputs (oracle/make_golden.py f4)"""
    g = _load("f4")
    n, ds, da, B, K = (int(g[k]) for k in ("n", "ds", "da", "B", "K"))
    hidden = [int(h) for h in g["hidden"]]
    raw = ora.synthetic_batches(K, n, B, ds, da, 34)
    from oracle.oracle import sac_defaults, td3_defaults
    st = ora.td3(n, ds, da, hidden, 1.0, 33, shared=True)
    for k in range(K):
        dvd = {"probe": g["probe"], "length_scale": 0.7, "jitter": 1e-6, "lam_start": 0.1,
               "lam_end": 0.7, "horizon": 4, "step": k}
        mask = [1, 1, 0, 0] if k == 1 else None
        if k == 3:
            st.step(raw_at(raw, k), td3_defaults(n), policy_mask=mask)
        else:
            st.step(raw_at(raw, k), td3_defaults(n), policy_mask=mask, dvd=dvd)
    for k in TD3_NETS:
        assert bits_equal(st.get_net(k), g[f"td3_{k}"]), k
    ss = ora.sac(n, ds, da, hidden, 1.0, 41, shared=True)
    for k in range(K):
        ss.step(raw_at(raw, k), sac_defaults(n, da))
    for k in SAC_NETS:
        assert bits_equal(ss.get_net(k), g[f"sac_{k}"]), k
    loss, logdet, grad = ora.dvd_loss(g["dvd_emb"], 0.9, 1e-8, 1.3)
    assert loss == g["dvd_loss"] and logdet == g["dvd_logdet"]
    assert np.array_equal(grad, g["dvd_grad"])
    assert ora.median_pairwise_distance(g["dvd_emb"]) == g["median"]
    cand, nxt = ora.cem_sample(g["cem_mean"], g["cem_var"], 1e-2, 6, int(g["cem_key"]), 4)
    assert nxt == int(g["cem_next"]) and np.array_equal(cand, g["cem_cand"])
    m2, v2, nz = ora.cem_update(g["cem_mean"], g["cem_var"], 1e-2, g["cem_cand"], g["cem_scores"])
    assert np.array_equal(m2, g["cem_mean2"]) and np.array_equal(v2, g["cem_var2"])
    assert nz == g["cem_noise2"]
