"""Pins the C restatement (oracle/pbrl_oracle.c) to the unmodified reference build
(oracle/_ref/libpbrl_ref.so, compiled from /root/reference sources by oracle/Makefile).
Everything here must be bit-identical; the GPU parity tests then only need the oracle."""
import numpy as np
import pytest

from helpers import SAC_NETS, TD3_NETS, bits_equal, raw_at
from oracle.oracle import sac_defaults, td3_defaults


def test_rng_streams(ora, ref):
    for seed, stream, use, step in [(0, 0, 1, 0), (7, 3, 4, 99), (2**63 + 5, 12345, 12, 2**40)]:
        k1, k2 = ora.stream_key(seed, stream, use, step), ref.stream_key(seed, stream, use, step)
        assert k1 == k2
        for c in (0, 1, 2, 1000, 2**50):
            assert ora.uniform(k1, c) == ref.uniform(k2, c)
            assert ora.normal_pair(k1, c) == ref.normal_pair(k2, c)


def test_synthetic_batches(ora, ref):
    a = ora.synthetic_batches(3, 4, 16, 17, 6, 7)
    b = ref.synthetic_batches(3, 4, 16, 17, 6, 7)
    for x, y in zip(a, b):
        assert bits_equal(x, y)


@pytest.mark.parametrize("hidden,n,ds,da,B,K,bound", [
    ([8, 8], 3, 4, 2, 8, 20, 1.0),
    ([7], 2, 5, 3, 13, 8, 2.0),
    ([33, 17, 9], 3, 3, 1, 10, 6, 0.5),
])
def test_td3_steps_bitexact(ora, ref, hidden, n, ds, da, B, K, bound):
    so, sr = ora.td3(n, ds, da, hidden, bound, 11), ref.td3(n, ds, da, hidden, bound, 11)
    hy = td3_defaults(n)
    hy["policy_delay_ratio"] = list(np.linspace(0.3, 1.0, n))
    hy["critic_lr"] = list(np.linspace(3e-4, 1e-3, n))
    raw = ora.synthetic_batches(K, n, B, ds, da, 12)
    for k in range(K):
        mask = None if k % 3 else [1] * (n - 1) + [0]
        lo = so.step(raw_at(raw, k), hy, policy_mask=mask)
        lr = sr.step(raw_at(raw, k), hy, policy_mask=mask, want_losses=True)
        assert lo[0].sum() == pytest.approx(lr[0], rel=1e-12)
        assert lo[1].sum() == pytest.approx(lr[1], rel=1e-12)
    for net in TD3_NETS:
        assert bits_equal(so.get_net(net), sr.get_net(net)), net
    for net in ("policy", "critic1", "critic2"):
        for m in range(n):
            a, b = so.get_adam(net, m), sr.get_adam(net, m)
            assert bits_equal(a[0], b[0]) and bits_equal(a[1], b[1]) and a[2] == b[2]
    for x, y in zip(so.counters(), sr.counters()):
        assert np.array_equal(x, y)


def test_td3_target(ora, ref):
    n, ds, da, B = 3, 5, 2, 9
    so, sr = ora.td3(n, ds, da, [6], 1.0, 3), ref.td3(n, ds, da, [6], 1.0, 3)
    raw = raw_at(ora.synthetic_batches(1, n, B, ds, da, 4), 0)
    hy = td3_defaults(n)
    hy["gamma"] = [0.0, 0.95, 1.0]
    assert bits_equal(so.target(raw, hy), sr.target(raw, hy))
    # gamma = 0 reduces to the reward (test_algos_td3.cpp:29-46)
    assert bits_equal(so.target(raw, hy)[0], raw[2][0])


@pytest.mark.parametrize("hidden,n,ds,da,B,K", [([8, 8], 3, 4, 2, 8, 10), ([16], 2, 3, 3, 12, 5)])
def test_sac_steps_bitexact(ora, ref, hidden, n, ds, da, B, K):
    so, sr = ora.sac(n, ds, da, hidden, 1.0, 21), ref.sac(n, ds, da, hidden, 1.0, 21)
    hy = sac_defaults(n, da)
    hy["reward_scale"] = list(np.linspace(0.5, 2.0, n))
    raw = ora.synthetic_batches(K, n, B, ds, da, 22)
    for k in range(K):
        lo = so.step(raw_at(raw, k), hy)
        lr = sr.step(raw_at(raw, k), hy, want_losses=True)
        assert lo[2].sum() == pytest.approx(lr[2], rel=1e-9, abs=1e-12)
    for net in SAC_NETS:
        assert bits_equal(so.get_net(net), sr.get_net(net)), net
    for x, y in zip(so.counters(), sr.counters()):
        assert np.array_equal(x, y)


def _fill(lib, cap, ds, da, count, seed, member=0):
    rb = lib.replay(cap, ds, da)
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(count):
        t = (rng.standard_normal(ds), rng.standard_normal(da), float(rng.standard_normal()),
             rng.standard_normal(ds), float(i % 7 == 0))
        rb.push(t[0], t[1], t[2], t[3], t[4], member)
        rows.append(t)
    return rb, rows


@pytest.mark.parametrize("mode", [0, 1])
def test_replay_sample(ora, ref, mode):
    n, ds, da, B = 3, 4, 2, 37
    nb = n if mode == 0 else 1
    bo = [_fill(ora, 50, ds, da, 30 + 20 * m, m, m)[0] for m in range(nb)]
    br = [_fill(ref, 50, ds, da, 30 + 20 * m, m, m)[0] for m in range(nb)]
    streams = [5, 9, 2]
    for draw in (0, 1, 17):
        a = ora.sample_batch(bo, B, mode, n, 77, streams, draw)
        b = ref.sample_batch(br, B, mode, n, 77, streams, draw)
        for x, y in zip(a[:5], b):
            assert bits_equal(x, y)
    # min_size gating returns "not ready" (nullopt)
    assert ora.sample_batch(bo, B, mode, n, 77, streams, 0, min_size=1000) is None
    assert ref.sample_batch(br, B, mode, n, 77, streams, 0, min_size=1000) is None


def test_pbt_rank_and_plan(ora, ref):
    rng = np.random.default_rng(0)
    for n in (4, 5, 10, 33, 80):
        rings = rng.standard_normal((n, 10)).round(1)  # rounding creates ties
        counts = rng.integers(1, 11, n).astype(np.uint32)
        assert np.array_equal(ora.pbt_rank(rings, counts), ref.pbt_rank(rings, counts))
        key = ref.stream_key(1, 0, 8, 0)
        a = ora.pbt_plan(rings, counts, 0.3, key, 5)
        b = ref.pbt_plan(rings, counts, 0.3, key, 5)
        assert all(np.array_equal(x, y) for x, y in zip(a[:2], b[:2])) and a[2] == b[2]
    # evolve.hpp test: ranks [5,1,9] -> [2,0,1]
    assert list(ora.pbt_rank(np.array([[5.0], [1.0], [9.0]]), [1, 1, 1])) == [2, 0, 1]


def test_pbt_evolve_trainer(ora, ref):
    n, ds, da = 10, 3, 2
    so, sr = ora.td3(n, ds, da, [4], 1.0, 60), ref.td3(n, ds, da, [4], 1.0, 60)
    raw = ora.synthetic_batches(2, n, 6, ds, da, 1)
    hy = td3_defaults(n)
    for k in range(2):
        so.step(raw_at(raw, k), hy)
        sr.step(raw_at(raw, k), hy)
    rings = np.arange(n, dtype=np.float64)[:, None] * np.ones((1, 3))
    counts = np.full(n, 3, np.uint32)
    key = ref.stream_key(1, 2, 8, 0)
    a = so.pbt_evolve(rings, counts, hy, key, 0)
    b = sr.pbt_evolve(rings, counts, hy, key, 0)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    assert sorted(a[0].tolist()) == [0, 1, 2] and all(d >= 7 for d in a[1])
    for f in a[3]:
        assert np.array_equal(a[3][f], b[3][f]), f
    for net in TD3_NETS:
        assert bits_equal(so.get_net(net), sr.get_net(net))
    ss, rs = ora.sac(n, ds, da, [4], 1.0, 61), ref.sac(n, ds, da, [4], 1.0, 61)
    hs = sac_defaults(n, da)
    a = ss.pbt_evolve(rings, counts, hs, key, 3, -2.0)
    b = rs.pbt_evolve(rings, counts, hs, key, 3, -2.0)
    assert np.array_equal(a[0], b[0]) and a[2] == b[2]
    for f in a[3]:
        assert np.array_equal(a[3][f], b[3][f]), f


@pytest.mark.parametrize("algo", ["td3", "sac"])
def test_act_bitexact(ora, ref, algo):
    """act / sac_act (algos.hpp:895-942): restatement == reference, several row counts."""
    rng = np.random.default_rng(3)
    for rows, hidden in ((1, [16, 16]), (7, [32, 32])):
        o = (ora.td3 if algo == "td3" else ora.sac)(4, 11, 3, hidden, 2.0, 9)
        r = (ref.td3 if algo == "td3" else ref.sac)(4, 11, 3, hidden, 2.0, 9)
        obs = rng.uniform(-1, 1, (4, rows, 11)).astype(np.float32)
        steps = np.asarray([0, 5, 17, 2], np.uint64)
        noise = [0.1, 0.0, 0.5, 0.2]
        for det in (False, True):
            a = o.act(obs, 123, steps, noise, det)
            b = r.act(obs, 123, steps, noise, det)
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (rows, det)
