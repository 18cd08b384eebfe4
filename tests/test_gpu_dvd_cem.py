"""DvD and CEM on the B200 vs the CPU oracle.

DvD (evolve.hpp:304-525): dvd_embed, and td3_update_step with dvd_policy_hook -- the hook's
forward on the probe states and its backward run on the device, the log-determinant loss on the
host -- bit-exact in FFMA32 (shared and independent critics, member masks, a lambda schedule),
within the derived tolerance in TF32 / BF16 (case S_td3_dvd_pop8).
CEM (evolve.hpp:221-297, cem_resample pipeline_run.hpp:148-158): device draws vs cem_sample, the
policy arena / targets / Adam reset, and cem_update's elite refit vs the oracle on the same
candidates.
"""
import numpy as np
import pytest

from helpers import TD3_NETS, bits_equal, check_parity, raw_at, to_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb(cuda):
    import paper_2206_08888_b200 as pb
    return pb


def _cfgs(pb, ds, ms, step, seed=5, sched=(0.1, 0.7, 4)):
    probe = np.random.default_rng(seed).uniform(-1, 1, (ms, ds))
    dev = pb.DvDConfig(probe.ravel(), ms, 0.7, 1e-6, pb.LambdaSchedule(*sched))
    ora = {"probe": probe, "length_scale": 0.7, "jitter": 1e-6, "lam_start": sched[0],
           "lam_end": sched[1], "horizon": sched[2], "step": step}
    return dev, ora


def test_dvd_embed_bitexact(pb, ora):
    n, ds, da, ms = 5, 17, 6, 9
    st = pb.make_td3_state(n, ds, da, [64, 64], 1.0, 3)
    ref = ora.td3(n, ds, da, [64, 64], 1.0, 3)
    probe = np.random.default_rng(1).uniform(-1, 1, (ms, ds))
    assert bits_equal(pb.dvd_embed(st, probe, ms), ref.dvd_embed(probe))


@pytest.mark.parametrize("mode", ["shared_critic", "independent"])
def test_td3_dvd_hook_bitexact(pb, ora, mode):
    n, ds, da, B, K, ms = 4, 17, 6, 16, 5, 6
    shared = mode == "shared_critic"
    st = pb.make_td3_state(n, ds, da, [32, 32], 1.0, 33, mode=mode)
    ref = ora.td3(n, ds, da, [32, 32], 1.0, 33, shared=shared)
    hy = pb.Td3Hyper.defaults(n)
    if not shared:
        hy.policy_delay_ratio = [1.0, 0.5, 1.0, 0.5]
    oh = {f: list(getattr(hy, f)) for f in pb.Td3Hyper.FIELDS}
    raw = ora.synthetic_batches(K, n, B, ds, da, 34)
    for k in range(K):  # lambda ramps 0.1 -> 0.7 over 4 steps, then clamps
        cfg, ocfg = _cfgs(pb, ds, ms, k)
        mask = [1, 0, 1, 1] if k == 2 else None
        pb.td3_update_step(st, to_batch(pb, raw, k), hy, hook=pb.dvd_policy_hook(cfg, k),
                           policy_member_mask=mask)
        ref.step(raw_at(raw, k), oh, policy_mask=mask, dvd=ocfg)
    for net in TD3_NETS:
        assert bits_equal(st.params(net), ref.get_net(net)), net
    for m in range(n):
        a, b = st.adam("policy", m), ref.get_adam("policy", m)
        assert bits_equal(a[0], b[0]) and bits_equal(a[1], b[1]) and a[2] == b[2]
    # the hook is per call: a plain step afterwards adds nothing
    cfg, _ = _cfgs(pb, ds, ms, 0)
    pb.td3_update_step(st, to_batch(pb, raw, 0), hy)
    ref.step(raw_at(raw, 0), oh)
    assert bits_equal(st.params("policy"), ref.get_net("policy"))


def test_dvd_k_steps_through_graph(pb, ora):
    """update_k_steps with the hook: the step graph carries the gradient add, the pre-pass runs
    eagerly before every replay."""
    n, ds, da, B, K, ms = 6, 17, 6, 32, 4, 8
    st = pb.make_td3_state(n, ds, da, [32, 32], 1.0, 8, mode="shared_critic")
    ref = ora.td3(n, ds, da, [32, 32], 1.0, 8, shared=True)
    hy = pb.Td3Hyper.defaults(n)
    oh = {f: list(getattr(hy, f)) for f in pb.Td3Hyper.FIELDS}
    raw = ora.synthetic_batches(K, n, B, ds, da, 9)
    cfg, ocfg = _cfgs(pb, ds, ms, 2)
    it = iter(range(K))
    pb.update_k_steps(st, lambda: to_batch(pb, raw, next(it)), K, hy,
                      hook=pb.dvd_policy_hook(cfg, 2))
    for k in range(K):
        ref.step(raw_at(raw, k), oh, dvd=ocfg)
    for net in TD3_NETS:
        assert bits_equal(st.params(net), ref.get_net(net)), net


def test_dvd_degenerate_population_raises(pb, ora):
    n, ds, da = 3, 5, 2
    st = pb.make_td3_state(n, ds, da, [16], 1.0, 1, mode="shared_critic")
    for m in range(1, n):  # identical policies -> identical embeddings
        st.unflatten_member("policy", m, st.flatten_member("policy", 0))
    probe = np.zeros((4, ds))
    cfg = pb.DvDConfig(probe.ravel(), 4, 1.0, 0.0, pb.LambdaSchedule(1.0, 1.0, 1))
    b = pb.make_synthetic_batches(1, n, 8, ds, da, 2)[0]
    with pytest.raises(pb.DegeneratePopulationError):
        pb.td3_update_step(st, b, pb.Td3Hyper.defaults(n), hook=pb.dvd_policy_hook(cfg, 0))


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
def test_dvd_tensor_core_within_derived_tolerance(pb, ora, precision):
    check_parity(pb, ora, "S_td3_dvd_pop8", precision)


def test_cem_resample_and_update(pb, ora):
    n, ds, da = 6, 17, 6
    st = pb.make_td3_state(n, ds, da, [64, 64], 1.0, 12, mode="shared_critic")
    P = st.param_count("policy")
    p0 = st.flatten_member("policy", 0).astype(np.float64)
    cem = pb.cem_init(st, None, 0.05)
    assert np.array_equal(cem.mean, p0) and (cem.var == 0.05).all()
    rng = pb.RngSequence(7, 2, "kCemDraw", 0)
    # advance the policies first so the resample visibly resets their Adam state
    b = pb.make_synthetic_batches(2, n, 16, ds, da, 3)
    pb.td3_update_step(st, b[0], pb.Td3Hyper.defaults(n))
    cand = pb.cem_resample(cem, rng)
    want, nxt = ora.cem_sample(p0, np.full(P, 0.05), 1e-2, n, rng.stream.key, 0)
    assert rng.next == nxt == 2 * n * P
    # device double log / cos may differ from glibc in the last bit: the candidates agree to a
    # few double ulp and the float policies bit for bit (but for a rare rounding-boundary case)
    assert np.max(np.abs(cand - want)) < 1e-14
    pol = st.params("policy")
    assert np.mean(pol == want.astype(np.float32)) > 1 - 1e-5
    assert bits_equal(pol, cand.astype(np.float32))
    assert bits_equal(st.params("policy_target"), pol)
    for m in range(n):
        mo, vo, t = st.adam("policy", m)
        assert t == 0 and not mo.any() and not vo.any()
    # cem_update on the device candidates == the oracle's on the same candidates
    scores = np.array([3.0, 1.0, 5.0, 1.0, -2.0, 4.0])
    pb.cem_update(cem, scores)
    m2, v2, nz = ora.cem_update(p0, np.full(P, 0.05), 1e-2, cand, scores)
    assert np.array_equal(cem.mean, m2) and np.array_equal(cem.var, v2)
    assert cem.noise == nz
    with pytest.raises(pb.ConfigError):
        pb.cem_update(cem, scores[:5])
    with pytest.raises(pb.ConfigError):
        pb.cem_update(cem, np.r_[scores[:5], np.nan])
    # the next generation samples around the refit mean
    cand2 = pb.cem_resample(cem, rng)
    want2, _ = ora.cem_sample(m2, v2, nz, n, rng.stream.key, 2 * n * P)
    assert np.max(np.abs(cand2 - want2)) < 1e-14
