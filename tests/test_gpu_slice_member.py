"""State-level slice_member / set_member (algos.hpp:425-464, :839-886) and the reference's
central equivalence: a vectorized population equals its members run as separate populations of
one (test_algos_td3.cpp:90-118, test_algos_sac.cpp:110-136) -- bit for bit in the FFMA32 check
mode, here on the device."""
import numpy as np
import pytest

from helpers import SAC_NETS, TD3_NETS, bits_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb(cuda):
    import paper_2206_08888_b200 as pb
    return pb


def _slice_batch(pb, b, m):
    return pb.TransitionBatch(*[x[m:m + 1].contiguous() for x in (b.s, b.a, b.r, b.s2, b.done)])


@pytest.mark.parametrize("precision", ["ffma32", "bf16"])
def test_td3_vectorized_equals_singletons(pb, precision):
    n, ds, da, b = 3, 4, 2, 32
    st = pb.make_td3_state(n, ds, da, [32, 32], 1.0, 11, precision=precision)
    hy = pb.Td3Hyper.defaults(n)
    hy.policy_delay_ratio = [0.5, 1.0, 0.3]  # distinct delays per member
    hy.critic_lr = [3e-4, 1e-3, 3e-4]
    singles = [pb.slice_member(st, m) for m in range(n)]
    hys = [hy.slice(m) for m in range(n)]
    for batch in pb.make_synthetic_batches(20, n, b, ds, da, 12):
        pb.td3_update_step(st, batch, hy)
        for m in range(n):
            pb.td3_update_step(singles[m], _slice_batch(pb, batch, m), hys[m])
    for m in range(n):
        for net in TD3_NETS:
            assert bits_equal(st.flatten_member(net, m), singles[m].flatten_member(net, 0)), (m, net)
        assert st.delay_acc[m] == singles[m].delay_acc[0]
        for net in ("policy", "critic1", "critic2"):
            a, s1 = st.adam(net, m), singles[m].adam(net, 0)
            assert bits_equal(a[0], s1[0]) and bits_equal(a[1], s1[1]) and a[2] == s1[2]
    assert np.array_equal(st.steps, np.concatenate([s.steps for s in singles]))


def test_sac_vectorized_equals_singletons(pb):
    n, ds, da, b = 3, 4, 2, 8
    st = pb.make_sac_state(n, ds, da, [8, 8], 1.0, 21)
    hy = pb.SacHyper.defaults(n, da)
    hy.alpha_lr = [3e-4, 1e-3, 3e-3]
    singles = [pb.slice_member(st, m) for m in range(n)]
    hys = [hy.slice(m) for m in range(n)]
    for batch in pb.make_synthetic_batches(12, n, b, ds, da, 22):
        pb.sac_update_step(st, batch, hy)
        for m in range(n):
            pb.sac_update_step(singles[m], _slice_batch(pb, batch, m), hys[m])
    la = st.alpha_state()
    for m in range(n):
        for net in SAC_NETS:
            assert bits_equal(st.flatten_member(net, m), singles[m].flatten_member(net, 0)), (m, net)
        sa = singles[m].alpha_state()
        for x, y in zip(la, sa):
            assert x[m] == y[0]


def test_set_member_round_trip_moves_the_whole_state(pb):
    """set_member(dst, i, slice_member(src, j)): member i of dst becomes member j of src, incl.
    its stream id and step count (the target noise is keyed by them and by the state seed, which
    is state-level: both states share it), so the next updates agree bit for bit."""
    n, ds, da, b = 4, 5, 2, 16
    src = pb.make_td3_state(n, ds, da, [16, 16], 1.0, 31)
    dst = pb.make_td3_state(n, ds, da, [16, 16], 1.0, 31)
    hy = pb.Td3Hyper.defaults(n)
    batches = pb.make_synthetic_batches(6, n, b, ds, da, 33)
    for bt in batches[:3]:
        pb.td3_update_step(src, bt, hy)
    pb.td3_update_step(dst, pb.make_synthetic_batches(1, n, b, ds, da, 34)[0], hy)
    pb.set_member(dst, 1, pb.slice_member(src, 2))
    for net in TD3_NETS:
        assert bits_equal(dst.flatten_member(net, 1), src.flatten_member(net, 2)), net
    assert dst.adam("critic1", 1)[2] == src.adam("critic1", 2)[2] == 3
    # same rows for member 1 of dst and member 2 of src from here on
    for bt in batches[3:]:
        pb.td3_update_step(src, bt, hy)
        rows = [x.clone() for x in (bt.s, bt.a, bt.r, bt.s2, bt.done)]
        for x, y in zip(rows, (bt.s, bt.a, bt.r, bt.s2, bt.done)):
            x[1] = y[2]
        pb.td3_update_step(dst, pb.TransitionBatch(*rows), hy)
    for net in TD3_NETS:
        assert bits_equal(dst.flatten_member(net, 1), src.flatten_member(net, 2)), net


def test_slice_member_index_out_of_range_is_a_usage_error(pb):
    st = pb.make_td3_state(2, 3, 1, [4], 1.0, 1)
    with pytest.raises(pb.UsageError):
        pb.slice_member(st, 2)
