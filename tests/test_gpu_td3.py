"""TD3 population update on the B200 vs the CPU oracle (FFMA32 check mode: bit-exact).

Mirrors the reference's own TD3 tests (proj/tests/test_algos_td3.cpp) with the device path
as the system under test and the C restatement (pinned to the reference in
test_oracle_vs_ref.py) as the checker.
"""
import numpy as np
import pytest

from helpers import TD3_NETS, bits_equal, raw_at, to_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb(cuda):
    import paper_2206_08888_b200 as pb
    return pb


def _run_pair(pb, ora, n, ds, da, hidden, B, K, seed=11, bseed=12, hyper=None, masks=None,
              bound=1.0):
    st = pb.make_td3_state(n, ds, da, hidden, bound, seed)
    ref = ora.td3(n, ds, da, hidden, bound, seed)
    hy = pb.Td3Hyper.defaults(n)
    for k, v in (hyper or {}).items():
        setattr(hy, k, list(v))
    oh = {f: list(getattr(hy, f)) for f in pb.Td3Hyper.FIELDS}
    raw = ora.synthetic_batches(K, n, B, ds, da, bseed)
    dev_losses, ref_losses = [], []
    for k in range(K):
        mask = None if masks is None else masks[k]
        pb.td3_update_step(st, to_batch(pb, raw, k), hy, policy_member_mask=mask)
        dev_losses.append(np.stack(st.last_losses()))
        ref_losses.append(ref.step(raw_at(raw, k), oh, policy_mask=mask))
    return st, ref, np.stack(dev_losses), np.stack(ref_losses)


def _assert_state_equal(st, ref, n):
    for net in TD3_NETS:
        assert bits_equal(st.params(net), ref.get_net(net)), net
    for net in ("policy", "critic1", "critic2"):
        for m in range(n):
            m1, v1, t1 = st.adam(net, m)
            m2, v2, t2 = ref.get_adam(net, m)
            assert bits_equal(m1, m2) and bits_equal(v1, v2) and t1 == t2, (net, m)
    da, steps = ref.counters()
    assert np.array_equal(st.delay_acc, da)
    assert np.array_equal(st.steps, steps)


def test_init_matches_reference_init(pb, ora):
    """make_td3_state on device == init_pop_mlp on the CPU, bitwise (net_pop.hpp:69-100)."""
    st = pb.make_td3_state(5, 17, 6, [256, 256], 1.0, 7)
    ref = ora.td3(5, 17, 6, [256, 256], 1.0, 7)
    for net in TD3_NETS:
        assert bits_equal(st.params(net), ref.get_net(net)), net


def test_vectorized_equals_oracle_distinct_members(pb, ora):
    """test_algos_td3.cpp:90-118 scenario: N=3, 20 steps, distinct delays and lrs."""
    hy = dict(policy_delay_ratio=[0.5, 1.0, 0.3], critic_lr=[3e-4, 1e-3, 3e-4])
    st, ref, dl, rl = _run_pair(pb, ora, 3, 4, 2, [8, 8], 8, 20, hyper=hy)
    _assert_state_equal(st, ref, 3)
    assert np.array_equal(dl, rl)


def test_halfcheetah_shape_bitexact(pb, ora):
    """Config A shape (obs 17, act 6, 2x256, B=256), pop 4, 4 steps: bit-exact."""
    st, ref, dl, rl = _run_pair(pb, ora, 4, 17, 6, [256, 256], 256, 4, seed=7, bseed=7)
    _assert_state_equal(st, ref, 4)
    assert np.array_equal(dl, rl)


def test_depth_and_ragged_dims(pb, ora):
    """One and three hidden layers, widths not multiples of any tile, action bound != 1."""
    st, ref, dl, rl = _run_pair(pb, ora, 2, 5, 3, [7], 13, 6, bound=2.0,
                                hyper=dict(policy_delay_ratio=[1.0, 0.7]))
    _assert_state_equal(st, ref, 2)
    st, ref, dl, rl = _run_pair(pb, ora, 3, 3, 1, [33, 17, 65], 70, 5,
                                hyper=dict(policy_delay_ratio=[1.0, 0.5, 0.25]))
    _assert_state_equal(st, ref, 3)
    assert np.array_equal(dl, rl)


def test_policy_member_mask(pb, ora):
    """policy_member_mask vetoes fired members: their policy stays bitwise (algos.hpp:391)."""
    masks = [[1, 0, 1, 1], [0, 1, 1, 0], None, [1, 1, 0, 1]]
    st, ref, dl, rl = _run_pair(pb, ora, 4, 4, 2, [16], 8, 4, masks=masks,
                                hyper=dict(policy_delay_ratio=[1.0] * 4))
    _assert_state_equal(st, ref, 4)


def test_gamma_zero_and_extreme_hypers(pb, ora):
    hy = dict(gamma=[0.0, 1.0, 0.9], tau=[1.0, 0.5, 1e-3], target_std=[0.0, 3.0, 0.2],
              target_clip=[0.0, 0.1, 10.0], policy_delay_ratio=[1.0, 1.0, 1.0])
    st, ref, dl, rl = _run_pair(pb, ora, 3, 4, 2, [12, 12], 16, 6, hyper=hy)
    _assert_state_equal(st, ref, 3)


def test_config_error_on_bad_hyper(pb):
    st = pb.make_td3_state(2, 3, 1, [4], 1.0, 1)
    hy = pb.Td3Hyper.defaults(2)
    hy.tau = [0.5, 1.5]
    b = pb.TransitionBatch(np.zeros((2, 4, 3)), np.zeros((2, 4, 1)), np.zeros((2, 4, 1)),
                           np.zeros((2, 4, 3)), np.zeros((2, 4, 1)))
    with pytest.raises(pb.ConfigError):
        pb.td3_update_step(st, b, hy)
    b2 = pb.TransitionBatch(*[np.zeros((3,) + x.shape[1:]) for x in (b.s, b.a, b.r, b.s2, b.done)])
    with pytest.raises(pb.ConfigError):
        pb.td3_update_step(st, b2, pb.Td3Hyper.defaults(2))


def test_k_steps_equals_chained_steps(pb, ora):
    """update_k_steps == k single calls, bitwise (test_algos_td3.cpp:227-248)."""
    n, ds, da, B, K = 3, 4, 2, 8, 6
    raw = ora.synthetic_batches(K, n, B, ds, da, 3)
    a = pb.make_td3_state(n, ds, da, [16, 16], 1.0, 5)
    b = pb.make_td3_state(n, ds, da, [16, 16], 1.0, 5)
    hy = pb.Td3Hyper.defaults(n)
    it = iter(range(K))
    pb.update_k_steps(a, lambda: to_batch(pb, raw, next(it)), K, hy)
    for k in range(K):
        pb.td3_update_step(b, to_batch(pb, raw, k), hy)
    for net in TD3_NETS:
        assert bits_equal(a.params(net), b.params(net))
    calls = iter([to_batch(pb, raw, 0), to_batch(pb, raw, 1)])
    with pytest.raises(pb.DataStarvationError):
        pb.update_k_steps(a, lambda: next(calls, None), 5, hy)


def test_device_batches_equal_host_batches(pb, ora, cuda):
    import torch
    n, ds, da, B = 3, 17, 6, 32
    dev = pb.make_synthetic_batches(3, n, B, ds, da, 7)
    raw = ora.synthetic_batches(3, n, B, ds, da, 7)
    for k in range(3):
        for x, y in zip((dev[k].s, dev[k].a, dev[k].r[..., 0], dev[k].s2, dev[k].done[..., 0]),
                        raw_at(raw, k)):
            assert bits_equal(x.cpu().numpy(), y)
    a = pb.make_td3_state(n, ds, da, [32, 32], 1.0, 5)
    b = pb.make_td3_state(n, ds, da, [32, 32], 1.0, 5)
    hy = pb.Td3Hyper.defaults(n)
    for k in range(3):
        pb.td3_update_step(a, dev[k], hy)
        pb.td3_update_step(b, to_batch(pb, raw, k), hy)
    for net in TD3_NETS:
        assert bits_equal(a.params(net), b.params(net))


def test_launch_count_independent_of_population(pb, ora):
    """Vectorized launch count does not grow with N (test_bench.cpp:40-53)."""
    counts = []
    for n in (1, 8, 32):
        st = pb.make_td3_state(n, 17, 6, [32, 32], 1.0, 1)
        raw = ora.synthetic_batches(2, n, 16, 17, 6, 1)
        hy = pb.Td3Hyper.defaults(n)
        before = st.launch_count()
        for k in range(2):
            pb.td3_update_step(st, to_batch(pb, raw, k), hy)
        counts.append(st.launch_count() - before)
    assert counts[0] == counts[1] == counts[2]


@pytest.mark.parametrize("precision,K", [("ffma32", 5), ("bf16", 5), ("bf16", 70)])
def test_update_k_steps_with_losses_matches_single_steps(pb, ora, precision, K):
    """pbrl_update_batches_losses (k host batches, overlapped H2D staging, every step's losses)
    leaves the same state and reports the same per-step losses as k single-step calls (K = 70:
    the device-side loss history is read back in blocks of 64 steps)."""
    n, B = 3, 128
    raw = ora.synthetic_batches(K, n, B, 17, 6, 13)
    hy = pb.Td3Hyper.defaults(n)
    a = pb.make_td3_state(n, 17, 6, [64, 64] if precision == "ffma32" else [256, 256], 1.0, 13,
                          precision=precision)
    b = pb.make_td3_state(n, 17, 6, [64, 64] if precision == "ffma32" else [256, 256], 1.0, 13,
                          precision=precision)
    batches = [to_batch(pb, raw, k) for k in range(K)]
    it = iter(batches)
    la = pb.update_k_steps(a, lambda: next(it), K, hy, return_losses=True)
    lb = []
    for k in range(K):
        pb.td3_update_step(b, batches[k], hy)
        lb.append(np.stack(b.last_losses()))
    assert la.shape == (K, 3, n)
    assert np.array_equal(la, np.stack(lb))
    for net in ("policy", "policy_target", "critic1", "critic2", "critic1_target",
                "critic2_target"):
        assert np.array_equal(a.params(net), b.params(net)), net


@pytest.mark.parametrize("precision,n", [("bf16", 80), ("ffma32", 6)])
def test_pack_overlap_device_batches_equal_single_steps(pb, ora, precision, n):
    """Inside one update call the pack of batch i+1 runs on its own stream beside step i's last
    Adam (after the step graph's ev_stage_free record node).  K device batches in one call at the
    config-D shape (80 members, B = 256, both step graphs, policy delays mixed so some steps fire
    for a few members only, some for none) leave the same state, bit for bit, as K single-step
    calls, whose packs run in member-stream order."""
    import torch
    B, K = 256, 12
    hidden = [256, 256] if precision == "bf16" else [64, 64]
    hy = pb.Td3Hyper.defaults(n)
    hy.policy_delay_ratio = [[0.5, 0.25, 0.34, 0.2, 0.5][m % 5] for m in range(n)]
    gb = pb.make_synthetic_batches(K, n, B, 17, 6, 31, device=torch.device("cuda", 0))
    a = pb.make_td3_state(n, 17, 6, hidden, 1.0, 31, precision=precision)
    b = pb.make_td3_state(n, 17, 6, hidden, 1.0, 31, precision=precision)
    it = iter(gb)
    pb.update_k_steps(a, lambda: next(it), K, hy)
    for k in range(K):
        pb.td3_update_step(b, gb[k], hy)
    for net in TD3_NETS:
        assert bits_equal(a.params(net), b.params(net)), net
    assert np.array_equal(a.steps, b.steps) and np.array_equal(a.delay_acc, b.delay_acc)


def test_graph_launch_count_equals_eager(pb, monkeypatch):
    """The launch counter (bench.py's gpu_launches) counts the kernels a replayed step graph
    runs -- not its event-record or conditional nodes -- so K graph-mode steps (fire and
    non-fire graphs, packs beside the previous Adam) count what K eager steps launch."""
    import torch
    n, B, K = 8, 256, 6
    hy = pb.Td3Hyper.defaults(n)
    hy.policy_delay_ratio = [0.5] * n
    gb = pb.make_synthetic_batches(K + 2, n, B, 17, 6, 41, device=torch.device("cuda", 0))
    g = pb.make_td3_state(n, 17, 6, [256, 256], 1.0, 41, precision="bf16")
    monkeypatch.setenv("PBRL_NO_GRAPH", "1")
    e = pb.make_td3_state(n, 17, 6, [256, 256], 1.0, 41, precision="bf16")
    monkeypatch.delenv("PBRL_NO_GRAPH")
    counts = []
    for st in (g, e):
        for k in range(2):  # warm-up: the graphs are captured here
            pb.td3_update_step(st, gb[k], hy)
        before = st.launch_count()
        it = iter(gb[2:])
        pb.update_k_steps(st, lambda: next(it), K, hy)
        counts.append(st.launch_count() - before)
    assert counts[0] == counts[1], counts


@pytest.mark.parametrize("precision", ["bf16", "ffma32"])
def test_pack_overlap_sac_device_batches_equal_single_steps(pb, ora, precision):
    """The same for the SAC step graph (config C shape: 32 members, B = 256), whose policy
    backward is the last reader of the packed batch."""
    import torch
    from helpers import SAC_NETS
    n, B, K = 32, 256, 8
    hidden = [256, 256] if precision == "bf16" else [64, 64]
    hy = pb.SacHyper.defaults(n, 6)
    gb = pb.make_synthetic_batches(K, n, B, 17, 6, 37, device=torch.device("cuda", 0))
    a = pb.make_sac_state(n, 17, 6, hidden, 1.0, 37, precision=precision)
    b = pb.make_sac_state(n, 17, 6, hidden, 1.0, 37, precision=precision)
    it = iter(gb)
    pb.update_k_steps(a, lambda: next(it), K, hy)
    for k in range(K):
        pb.sac_update_step(b, gb[k], hy)
    for net in SAC_NETS:
        assert bits_equal(a.params(net), b.params(net)), net


@pytest.mark.parametrize("precision", ["ffma32", "bf16"])
def test_fire_and_nonfire_step_graphs_equal_eager(pb, ora, precision, monkeypatch):
    """Graph mode replays one of two step graphs per step (the host mirror of the delay
    accumulators picks the fire-step graph, the other keeps the device-decided IF node).  With
    per-member delays that make some steps fire for a few members only, some for all and some
    for none, the graph replay equals the eager launch sequence bit for bit (and, in FFMA32, the
    oracle)."""
    n, ds, da, B, K = 5, 17, 6, 64, 9
    hidden = [64, 64] if precision == "ffma32" else [256, 256]
    hy = pb.Td3Hyper.defaults(n)
    hy.policy_delay_ratio = [1.0, 0.5, 0.25, 0.34, 0.2]
    raw = ora.synthetic_batches(K, n, B, ds, da, 21)
    batches = [to_batch(pb, raw, k) for k in range(K)]
    g = pb.make_td3_state(n, ds, da, hidden, 1.0, 21, precision=precision)
    monkeypatch.setenv("PBRL_NO_GRAPH", "1")
    e = pb.make_td3_state(n, ds, da, hidden, 1.0, 21, precision=precision)
    monkeypatch.delenv("PBRL_NO_GRAPH")
    it = iter(batches)
    pb.update_k_steps(g, lambda: next(it), K, hy)
    for k in range(K):
        pb.td3_update_step(e, batches[k], hy)
    for net in TD3_NETS:
        assert bits_equal(g.params(net), e.params(net)), net
    assert np.array_equal(g.steps, e.steps) and np.array_equal(g.delay_acc, e.delay_acc)
    if precision == "ffma32":
        ref = ora.td3(n, ds, da, hidden, 1.0, 21)
        oh = {f: list(getattr(hy, f)) for f in pb.Td3Hyper.FIELDS}
        for k in range(K):
            ref.step(raw_at(raw, k), oh)
        _assert_state_equal(g, ref, n)
