"""Pins the C restatement's shared-critic TD3 / SAC, DvD and CEM to
the unmodified reference build (oracle/_ref/libpbrl_ref.so), bit for bit:
  shared-critic mode      algos.hpp:181-233, :351-422, :781-837
  DvD                     evolve.hpp:304-525 (dvd_lambda, dvd_embed, dvd_loss, median, hook)
  CEM                     evolve.hpp:221-297 (cem_sample, cem_update)
The reference tests these come from: test_algos_td3.cpp:120-146, :250-274, test_evolve.cpp:144-320.
"""
import numpy as np
import pytest

from helpers import SAC_NETS, TD3_NETS, bits_equal, raw_at
from oracle.oracle import sac_defaults, td3_defaults


def _same_td3(so, sr, n, nets=TD3_NETS):
    for net in nets:
        assert bits_equal(so.get_net(net), sr.get_net(net)), net
    for net in ("policy", "critic1", "critic2"):
        cnt = n if net == "policy" else so.nc
        for m in range(cnt):
            a, b = so.get_adam(net, m), sr.get_adam(net, m)
            assert bits_equal(a[0], b[0]) and bits_equal(a[1], b[1]) and a[2] == b[2], (net, m)


@pytest.mark.parametrize("hidden,n,ds,da,B,K", [([8, 8], 3, 4, 2, 8, 6), ([6], 4, 3, 1, 4, 5)])
def test_td3_shared_critic_bitexact(ora, ref, hidden, n, ds, da, B, K):
    so = ora.td3(n, ds, da, hidden, 1.0, 28, shared=True)
    sr = ref.td3(n, ds, da, hidden, 1.0, 28, shared=True)
    assert so.get_net("critic1").shape[0] == 1  # test_algos_td3.cpp:253
    hy = td3_defaults(n)
    hy["critic_lr"] = list(np.linspace(3e-4, 1e-3, n))  # only critic_lr[0] is used
    hy["tau"] = list(np.linspace(0.005, 0.05, n))
    raw = ora.synthetic_batches(K, n, B, ds, da, 29)
    p0 = so.get_net("policy", 0)
    for k in range(K):
        mask = [1, 1] + [0] * (n - 2) if k % 2 else None  # test_algos_td3.cpp:263-274
        so.step(raw_at(raw, k), hy, policy_mask=mask)
        sr.step(raw_at(raw, k), hy, policy_mask=mask)
    assert not np.array_equal(so.get_net("policy", 0), p0)  # no delay in shared mode
    _same_td3(so, sr, n)
    for x, y in zip(so.counters(), sr.counters()):
        assert np.array_equal(x, y)


def test_td3_shared_mask_freezes_members(ora):
    n, ds, da, B = 4, 3, 1, 4
    so = ora.td3(n, ds, da, [6], 1.0, 30, shared=True)
    raw = raw_at(ora.synthetic_batches(1, n, B, ds, da, 31), 0)
    frozen = so.get_net("policy", 2)
    so.step(raw, td3_defaults(n), policy_mask=[1, 1, 0, 0])
    assert not np.array_equal(so.get_net("policy", 0), so.get_net("policy", 2))
    assert np.array_equal(so.get_net("policy", 2), frozen)


@pytest.mark.parametrize("hidden,n,ds,da,B,K", [([8, 8], 3, 4, 2, 8, 4)])
def test_sac_shared_critic_bitexact(ora, ref, hidden, n, ds, da, B, K):
    so = ora.sac(n, ds, da, hidden, 1.0, 41, shared=True)
    sr = ref.sac(n, ds, da, hidden, 1.0, 41, shared=True)
    hy = sac_defaults(n, da)
    hy["tau"] = list(np.linspace(0.005, 0.05, n))
    raw = ora.synthetic_batches(K, n, B, ds, da, 42)
    for k in range(K):
        so.step(raw_at(raw, k), hy)
        sr.step(raw_at(raw, k), hy)
    for net in SAC_NETS:
        assert bits_equal(so.get_net(net), sr.get_net(net)), net
    for x, y in zip(so.counters(), sr.counters()):
        assert np.array_equal(x, y)


def _dvd_cfg(ora, n, ds, ms=None, seed=5, ls=0.7, lam=(0.1, 0.7, 10), step=4):
    ms = ms or n + 2
    rng = np.random.default_rng(seed)
    return {"probe": rng.uniform(-1, 1, (ms, ds)), "length_scale": ls, "jitter": 1e-6,
            "lam_start": lam[0], "lam_end": lam[1], "horizon": lam[2], "step": step}


@pytest.mark.parametrize("shared", [True, False])
def test_td3_dvd_hook_step_bitexact(ora, ref, shared):
    n, ds, da, B, K = 4, 5, 2, 6, 4
    so = ora.td3(n, ds, da, [8, 8], 1.0, 33, shared=shared)
    sr = ref.td3(n, ds, da, [8, 8], 1.0, 33, shared=shared)
    hy = td3_defaults(n)
    raw = ora.synthetic_batches(K, n, B, ds, da, 34)
    cfg = _dvd_cfg(ora, n, ds)
    assert bits_equal(so.dvd_embed(cfg["probe"]), sr.dvd_embed(cfg["probe"]))
    for k in range(K):
        c = dict(cfg, step=k)
        so.step(raw_at(raw, k), hy, dvd=c, policy_mask=[1, 0, 1, 1] if k == 2 else None)
        sr.step(raw_at(raw, k), hy, dvd=c, policy_mask=[1, 0, 1, 1] if k == 2 else None)
    _same_td3(so, sr, n)
    # lambda = 0 adds nothing (test_evolve.cpp:295-319)
    s0 = ora.td3(n, ds, da, [8, 8], 1.0, 33, shared=True)
    s1 = ora.td3(n, ds, da, [8, 8], 1.0, 33, shared=True)
    s0.step(raw_at(raw, 0), hy, dvd=dict(cfg, lam_start=0.0, step=0))
    s1.step(raw_at(raw, 0), hy)
    assert bits_equal(s0.get_net("policy"), s1.get_net("policy"))


def test_dvd_loss_and_helpers_bitexact(ora, ref):
    rng = np.random.default_rng(9)
    for n, dim in ((2, 3), (5, 8), (12, 30)):
        e = rng.normal(size=(n, dim))
        for ls, jit, lam in ((0.9, 1e-8, 1.3), (2.0, 0.0, 0.5)):
            a = ora.dvd_loss(e, ls, jit, lam)
            b = ref.dvd_loss(e, ls, jit, lam)
            assert a[0] == b[0] and a[1] == b[1] and bits_equal(a[2], b[2])
        assert ora.median_pairwise_distance(e) == ref.median_pairwise_distance(e)
    # 2x2 oracle with kernel value one half (test_evolve.cpp:244-253)
    ell = 1.0
    e = np.array([[0.0], [np.sqrt(2 * np.log(2.0))]])
    loss, logdet, _ = ora.dvd_loss(e, ell, 0.0, 2.0)
    assert logdet == pytest.approx(np.log(0.75), rel=1e-12)
    assert loss == pytest.approx(-2.0 * np.log(0.75), rel=1e-12)
    # identical rows: singular without jitter (test_evolve.cpp:255-265)
    same = np.ones((3, 4))
    with pytest.raises(FloatingPointError):
        ora.dvd_loss(same, 1.0, 0.0, 1.0)
    with pytest.raises(FloatingPointError):
        ref.dvd_loss(same, 1.0, 0.0, 1.0)
    with pytest.raises(ValueError):
        ora.dvd_loss(same[:1], 1.0, 0.0, 1.0)
    assert ora.median_pairwise_distance(same) == 1.0 == ref.median_pairwise_distance(same)
    for t in (0, 3, 50, 99, 100, 10**6):
        assert ora.dvd_lambda(t, 0.1, 0.7, 100) == ref.dvd_lambda(t, 0.1, 0.7, 100)
    assert ora.dvd_lambda(5, 0.1, 0.7, 0) == 0.7


def test_cem_bitexact(ora, ref):
    rng = np.random.default_rng(3)
    dim, count = 37, 6
    mean = rng.normal(size=dim)
    var = rng.uniform(0, 0.1, dim)
    key = ora.stream_key(7, 2, 11, 0)
    a, na = ora.cem_sample(mean, var, 1e-2, count, key, 4)
    b, nb = ref.cem_sample(mean, var, 1e-2, count, key, 4)
    assert na == nb == 4 + 2 * dim * count
    assert bits_equal(a, b)
    scores = rng.normal(size=count)
    scores[1] = scores[4]  # a tie: stable order
    x = ora.cem_update(mean, var, 1e-2, a, scores)
    y = ref.cem_update(mean, var, 1e-2, a, scores)
    assert bits_equal(x[0], y[0]) and bits_equal(x[1], y[1]) and x[2] == y[2]
    # hand-computed elites (test_evolve.cpp:168-191)
    m, v, nz = ora.cem_update([0.0], [0.0], 1e-2, [[2.0], [2.0], [9.0], [9.0]], [5, 5, 0, 0])
    assert m[0] == 2.0 and v[0] == 0.0 and nz == pytest.approx(1e-2 * 0.999)
    for bad in (([[0.0]], [1]), ([[0.0], [1.0], [2.0]], [1, 2, 3]), ([[0.0], [1.0]], [np.nan, 1])):
        with pytest.raises(ValueError):
            ora.cem_update([0.0], [0.0], 1e-2, *bad)
        with pytest.raises(ValueError):
            ref.cem_update([0.0], [0.0], 1e-2, *bad)
    # degenerate distribution: every sample is the mean (test_evolve.cpp:144-150)
    s, _ = ora.cem_sample([1.0, -2.0], [0.0, 0.0], 0.0, 4, key, 0)
    assert (s == np.array([1.0, -2.0])).all()
