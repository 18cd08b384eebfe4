"""Shared-critic TD3 / SAC (PopMode::kSharedCritic) on the B200 vs the
CPU oracle.  One critic pair serves the whole population; its batch is the population folded
into rows (critic_forward, algos.hpp:219-233), its loss is the mean over all n*B rows, every
policy updates every step and the critic target tracks when some member fires
(td3_update_step, algos.hpp:351-422; sac_update_step :781-837).

FFMA32: bit-exact (params, targets, Adam moments and step counts, counters, losses).
TF32 / BF16: within the tolerances oracle/derive_tolerances.py derives on the CPU
(cases S_*), incl. config-D shape (pop 80, B 256: one critic group of 20,480 rows).
Reference tests mirrored: test_algos_td3.cpp:250-274 (one critic, no delay, member mask).
"""
import numpy as np
import pytest

from helpers import SAC_NETS, TD3_NETS, bits_equal, check_parity, raw_at, to_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb(cuda):
    import paper_2206_08888_b200 as pb
    return pb


def _state_equal(st, ref, nets, n):
    for net in nets:
        assert bits_equal(st.params(net), ref.get_net(net)), net
    for net in ("policy", "critic1", "critic2"):
        for m in range(n if net == "policy" else 1):
            a, b = st.adam(net, m), ref.get_adam(net, m)
            assert bits_equal(a[0], b[0]) and bits_equal(a[1], b[1]) and a[2] == b[2], (net, m)


@pytest.mark.parametrize("n,hidden,B,K", [(4, [16, 16], 8, 5), (3, [64, 32], 40, 4),
                                          (6, [256, 256], 64, 3)])
def test_td3_shared_bitexact(pb, ora, n, hidden, B, K):
    ds, da = 17, 6
    st = pb.make_td3_state(n, ds, da, hidden, 1.0, 28, mode="shared_critic")
    ref = ora.td3(n, ds, da, hidden, 1.0, 28, shared=True)
    assert st.params("critic1").shape[0] == 1 and st.params("policy").shape[0] == n
    hy = pb.Td3Hyper.defaults(n)
    hy.critic_lr = list(np.linspace(3e-4, 1e-3, n))  # only critic_lr[0] / tau[0] reach the critic
    hy.tau = list(np.linspace(0.005, 0.05, n))
    oh = {f: list(getattr(hy, f)) for f in pb.Td3Hyper.FIELDS}
    raw = ora.synthetic_batches(K, n, B, ds, da, 29)
    for k in range(K):
        p2 = st.flatten_member("policy", 2)
        mask = [1, 1] + [0] * (n - 2) if k == 1 else None
        if k == 2:
            mask = [0] * n  # nobody fires: no policy update, no critic-target Polyak
        pb.td3_update_step(st, to_batch(pb, raw, k), hy, policy_member_mask=mask)
        dl = np.stack(st.last_losses())
        rl = ref.step(raw_at(raw, k), oh, policy_mask=mask)
        assert np.array_equal(dl, rl), (k, dl, rl)
        if k == 1:  # the masked-out half stays frozen (test_algos_td3.cpp:263-274)
            assert np.array_equal(st.flatten_member("policy", 2), p2)
    _state_equal(st, ref, TD3_NETS, n)
    da_, steps = ref.counters()
    assert np.array_equal(st.steps, steps)


def test_td3_shared_k_steps_graph_equals_oracle(pb, ora):
    """update_k_steps through the captured step graph (conditional policy half, PDL chain)."""
    n, ds, da, B, K = 5, 17, 6, 32, 6
    st = pb.make_td3_state(n, ds, da, [32, 32], 1.0, 3, mode="shared_critic")
    ref = ora.td3(n, ds, da, [32, 32], 1.0, 3, shared=True)
    hy = pb.Td3Hyper.defaults(n)
    oh = {f: list(getattr(hy, f)) for f in pb.Td3Hyper.FIELDS}
    raw = ora.synthetic_batches(K, n, B, ds, da, 4)
    it = iter(range(K))
    pb.update_k_steps(st, lambda: to_batch(pb, raw, next(it)), K, hy)
    for k in range(K):
        ref.step(raw_at(raw, k), oh)
    _state_equal(st, ref, TD3_NETS, n)


def test_sac_shared_bitexact(pb, ora):
    n, ds, da, B, K = 4, 17, 6, 16, 3
    st = pb.make_sac_state(n, ds, da, [32, 32], 1.0, 41, mode="shared_critic")
    ref = ora.sac(n, ds, da, [32, 32], 1.0, 41, shared=True)
    hy = pb.SacHyper.defaults(n, da)
    hy.tau = list(np.linspace(0.005, 0.05, n))
    oh = {f: list(getattr(hy, f)) for f in pb.SacHyper.FIELDS}
    raw = ora.synthetic_batches(K, n, B, ds, da, 42)
    for k in range(K):
        pb.sac_update_step(st, to_batch(pb, raw, k), hy)
        dl = np.stack(st.last_losses())
        rl = ref.step(raw_at(raw, k), oh)
        assert np.array_equal(dl, rl), k
    _state_equal(st, ref, SAC_NETS, n)


def test_shared_rejects_member_splitting(pb):
    st = pb.make_td3_state(4, 5, 2, [16], 1.0, 0, mode="shared_critic")
    with pytest.raises(pb.UsageError):
        pb.slice_member(st, 0)  # algos.hpp:427-429
    with pytest.raises(pb.UsageError):
        st.flatten_member("critic1", 1)  # one critic member
    pbt = pb.PBTState(4)
    for m in range(4):
        pbt.record_return(m, float(m))
    hy = pb.Td3Hyper.defaults(4)
    with pytest.raises(pb.UsageError):  # copy_member on the one-member critic (net_pop.hpp:193)
        pb.pbt_evolve_trainer(pbt, st, hy, pb.Td3Prior(), pb.RngSequence(7, 0, 8, 0))


@pytest.mark.parametrize("case", ["S_td3_shared_pop8", "S_sac_shared_pop8",
                                  "S_td3_shared_pop80"])
@pytest.mark.parametrize("precision", ["bf16", "tf32"])
def test_shared_tensor_core_within_derived_tolerance(pb, ora, case, precision):
    check_parity(pb, ora, case, precision)
