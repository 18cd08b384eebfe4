"""Device replay (ReplayBuffer / sample_batch, replay.hpp) and PBT (evolve.hpp) vs the oracle.

Sampled indices and gathered rows, PBT rankings, donor draws, member copies, optimiser resets
and hyper re-draws are all required to be bit-exact (north_star)."""
import numpy as np
import pytest

from helpers import TD3_NETS, SAC_NETS, bits_equal, raw_at, to_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb(cuda):
    import paper_2206_08888_b200 as pb
    return pb


def _transitions(n_rows, ds, da, seed, members):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((n_rows, ds)).astype(np.float32),
            rng.standard_normal((n_rows, da)).astype(np.float32),
            rng.standard_normal(n_rows).astype(np.float32),
            rng.standard_normal((n_rows, ds)).astype(np.float32),
            (rng.random(n_rows) < 0.1).astype(np.float32), members)


@pytest.mark.parametrize("mode", ["per_agent", "shared"])
def test_replay_sample_bitexact_with_wraparound(pb, ora, mode):
    n, ds, da, cap, B = 4, 17, 6, 64, 256
    st = pb.make_td3_state(n, ds, da, [8], 1.0, 3)
    rep = pb.DeviceReplay(st, cap, mode)
    nb = n if mode == "per_agent" else 1
    obufs = [ora.replay(cap, ds, da) for _ in range(nb)]
    # uneven fill, including wrap-around past capacity (FIFO eviction, replay.hpp:56-69)
    fills = [40, 64, 150, 9] if mode == "per_agent" else [70]
    for chunk in range(3):
        mem = np.concatenate([np.full(f // 3 + (chunk < f % 3), m, np.uint32)
                              for m, f in enumerate(fills)])
        np.random.default_rng(chunk).shuffle(mem)
        s, a, r, s2, d, _ = _transitions(mem.size, ds, da, 10 + chunk, mem)
        rep.insert(s, a, r, s2, d, mem)
        for i in range(mem.size):
            ob = obufs[mem[i]] if mode == "per_agent" else obufs[0]
            ob.push(s[i], a[i], r[i], s2[i], d[i], int(mem[i]))
    for b in range(nb):
        assert rep.size(b) == obufs[b].size()
    streams = list(range(n))
    for draw in (0, 1, 99):
        got = pb.sample_batch(rep, B, seed=77, draw_id=draw)
        want = ora.sample_batch(obufs, B, 0 if mode == "per_agent" else 1, n, 77, streams, draw)
        for g, w in zip((got.s, got.a, got.r[..., 0], got.s2, got.done[..., 0]), want[:5]):
            assert bits_equal(g, w)
    assert pb.sample_batch(rep, B, seed=77, draw_id=0, min_size=1000) is None


def test_update_from_replay_equals_host_batches(pb, ora):
    """pbrl_update_k (device sample + update) == sample_batch on host + td3_update_step."""
    n, ds, da, cap, B, K = 3, 17, 6, 500, 64, 4
    a = pb.make_td3_state(n, ds, da, [32, 32], 1.0, 8)
    b = pb.make_td3_state(n, ds, da, [32, 32], 1.0, 8)
    rep = pb.DeviceReplay(a, cap)
    rep_b = pb.DeviceReplay(b, cap)
    mem = np.repeat(np.arange(n, dtype=np.uint32), 200)
    s, aa, r, s2, d, _ = _transitions(mem.size, ds, da, 4, mem)
    rep.insert(s, aa, r, s2, d, mem)
    rep_b.insert(s, aa, r, s2, d, mem)
    hy = pb.Td3Hyper.defaults(n)
    assert pb.update_k_from_replay(a, rep, K, hy, B, seed=5, first_draw_id=10)
    for i in range(K):
        bt = pb.sample_batch(rep_b, B, seed=5, draw_id=10 + i)
        pb.td3_update_step(b, bt, hy)
    for net in TD3_NETS:
        assert bits_equal(a.params(net), b.params(net)), net
    assert not pb.update_k_from_replay(a, rep, 1, hy, B, seed=5, first_draw_id=0, min_size=10 ** 6)


def test_pbt_evolve_td3_matches_oracle(pb, ora):
    n, ds, da = 10, 5, 2
    st = pb.make_td3_state(n, ds, da, [16, 16], 1.0, 60)
    ref = ora.td3(n, ds, da, [16, 16], 1.0, 60)
    hy = pb.Td3Hyper.defaults(n)
    oh = {f: list(getattr(hy, f)) for f in pb.Td3Hyper.FIELDS}
    raw = ora.synthetic_batches(3, n, 8, ds, da, 2)
    for k in range(3):
        pb.td3_update_step(st, to_batch(pb, raw, k), hy)
        ref.step(raw_at(raw, k), oh)
    pbt = pb.PBTState(n)
    rng = np.random.default_rng(3)
    rings = np.zeros((n, 10))
    counts = np.zeros(n, np.uint32)
    for m in range(n):
        for j in range(int(rng.integers(1, 13))):
            v = float(np.round(rng.standard_normal(), 1))
            pbt.record_return(m, v)
        vals = list(pbt.returns[m])
        rings[m, :len(vals)] = vals
        counts[m] = len(vals)
    prng = pb.RngSequence(1, 2, "kDonorChoice")
    plan = pb.pbt_evolve_trainer(pbt, st, hy, pb.Td3Prior(), prng)
    rep_, don_, nxt, ohy = ref.pbt_evolve(rings, counts, oh, prng.stream.key, 0)
    assert plan.replaced == [int(x) for x in rep_] and plan.donors == [int(x) for x in don_]
    assert prng.next == nxt
    for f in pb.Td3Hyper.FIELDS:
        assert np.array_equal(np.asarray(getattr(hy, f)), ohy[f]), f
    for net in TD3_NETS:
        assert bits_equal(st.params(net), ref.get_net(net)), net
    for net in ("policy", "critic1", "critic2"):
        for m in plan.replaced:
            a, b = st.adam(net, m), ref.get_adam(net, m)
            assert bits_equal(a[0], b[0]) and a[2] == b[2] == 0
    assert np.array_equal(st.delay_acc, ref.counters()[0])
    assert all(len(pbt.returns[m]) == 0 for m in plan.replaced)
    # training continues identically after the exploit step (new hypers reach the device)
    raw2 = ora.synthetic_batches(2, n, 8, ds, da, 9)
    for k in range(2):
        pb.td3_update_step(st, to_batch(pb, raw2, k), hy)
        ref.step(raw_at(raw2, k), {f: list(getattr(hy, f)) for f in pb.Td3Hyper.FIELDS})
    for net in TD3_NETS:
        assert bits_equal(st.params(net), ref.get_net(net)), net


def test_pbt_evolve_sac_matches_oracle(pb, ora):
    n, ds, da = 8, 4, 2
    st = pb.make_sac_state(n, ds, da, [12], 1.0, 61)
    ref = ora.sac(n, ds, da, [12], 1.0, 61)
    hy = pb.SacHyper.defaults(n, da)
    oh = {f: list(getattr(hy, f)) for f in pb.SacHyper.FIELDS}
    raw = ora.synthetic_batches(2, n, 8, ds, da, 5)
    for k in range(2):
        pb.sac_update_step(st, to_batch(pb, raw, k), hy)
        ref.step(raw_at(raw, k), oh)
    pbt = pb.PBTState(n)
    for m in range(n):
        pbt.record_return(m, float((m * 7) % 5))
    rings = np.array([[float((m * 7) % 5)] for m in range(n)])
    counts = np.ones(n, np.uint32)
    prng = pb.RngSequence(4, 0, "kDonorChoice")
    prior = pb.SacPrior(default_target_entropy=-2.0)
    plan = pb.pbt_evolve_trainer(pbt, st, hy, prior, prng)
    rep_, don_, nxt, ohy = ref.pbt_evolve(rings, counts, oh, prng.stream.key, 0, -2.0)
    assert plan.replaced == [int(x) for x in rep_] and plan.donors == [int(x) for x in don_]
    for f in pb.SacHyper.FIELDS:
        assert np.array_equal(np.asarray(getattr(hy, f)), ohy[f]), f
    for net in SAC_NETS:
        assert bits_equal(st.params(net), ref.get_net(net)), net
    assert bits_equal(st.log_alpha, ref.counters()[0])


def test_pbt_small_population_and_not_ready(pb):
    st = pb.make_td3_state(3, 3, 1, [4], 1.0, 1)
    pbt = pb.PBTState(3)
    for m in range(3):
        pbt.record_return(m, m)
    assert pb.pbt_evolve_trainer(pbt, st, pb.Td3Hyper.defaults(3), pb.Td3Prior(),
                                 pb.RngSequence(1)) is None  # N < 4 is left alone
    st5 = pb.make_td3_state(5, 3, 1, [4], 1.0, 1)
    pbt5 = pb.PBTState(5)
    pbt5.record_return(0, 1.0)
    with pytest.raises(pb.NotReadyError):
        pb.pbt_plan(pbt5, pb.RngSequence(1), st5)
