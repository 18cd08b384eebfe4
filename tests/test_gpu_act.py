"""Batched action selection on the B200 (act / sac_act, algos.hpp:895-942)
against the C restatement oracle (itself pinned to the reference by tests/test_oracle_vs_ref.py
and tests/golden/act.npz): bit-exact in the FFMA32 check mode, within the tensor-core modes'
forward tolerance otherwise (max |a_dev - a_ref| <= 2e-2 * bound: one TF32 / BF16 forward)."""
import numpy as np
import pytest

from helpers import to_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb(cuda):
    import paper_2206_08888_b200 as pb
    return pb


def _pair(pb, ora, algo, n, ds, da, hidden, bound, seed, precision):
    make = pb.make_td3_state if algo == "td3" else pb.make_sac_state
    st = make(n, ds, da, hidden, bound, seed, precision=precision)
    ref = (ora.td3 if algo == "td3" else ora.sac)(n, ds, da, hidden, bound, seed)
    return st, ref


@pytest.mark.parametrize("algo", ["td3", "sac"])
@pytest.mark.parametrize("rows", [1, 5, 300])
def test_act_ffma32_bitexact(pb, ora, algo, rows):
    n, ds, da = 3, 17, 6
    st, ref = _pair(pb, ora, algo, n, ds, da, [64, 64], 2.0, 7, "ffma32")
    obs = np.random.default_rng(rows).uniform(-1, 1, (n, rows, ds)).astype(np.float32)
    steps = np.asarray([4, 0, 9], np.uint64)
    noise = [0.1, 0.0, 0.3]
    for det in (False, True):
        if algo == "td3":
            got = pb.act(st, obs, noise, 99, steps, det)
        else:
            got = pb.sac_act(st, obs, 99, steps, det)
        want = ref.act(obs, 99, steps, noise, det)
        assert got.shape == (n, rows, da)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (det, np.abs(got - want).max())


@pytest.mark.parametrize("precision", ["tf32", "bf16"])
@pytest.mark.parametrize("algo", ["td3", "sac"])
def test_act_tensor_core_modes(pb, ora, algo, precision):
    n, ds, da, bound = 4, 17, 6, 1.0
    st, ref = _pair(pb, ora, algo, n, ds, da, [256, 256], bound, 5, precision)
    obs = np.random.default_rng(1).uniform(-1, 1, (n, 64, ds)).astype(np.float32)
    steps = np.arange(n, dtype=np.uint64)
    noise = [0.1] * n
    for det in (False, True):
        got = pb.act(st, obs, noise, 3, steps, det) if algo == "td3" else \
            pb.sac_act(st, obs, 3, steps, det)
        want = ref.act(obs, 3, steps, noise, det)
        assert np.abs(got - want).max() <= 2e-2 * bound


def test_act_after_updates_tracks_the_policy(pb, ora):
    """act() reads the current policy (and, in BF16 mode, its refreshed operand copy)."""
    n, B = 2, 256
    st, ref = _pair(pb, ora, "td3", n, 17, 6, [64, 64], 1.0, 3, "ffma32")
    raw = ora.synthetic_batches(2, n, B, 17, 6, 3)
    hy = pb.Td3Hyper.defaults(n)
    hy.policy_delay_ratio = [1.0] * n
    oh = {f: list(getattr(hy, f)) for f in hy.FIELDS}
    for k in range(2):
        pb.td3_update_step(st, to_batch(pb, raw, k), hy)
        ref.step(tuple(x[k] for x in raw), oh)
    obs = np.random.default_rng(9).uniform(-1, 1, (n, 3, 17)).astype(np.float32)
    steps = np.asarray([1, 2], np.uint64)
    got = pb.act(st, obs, [0.2, 0.2], 5, steps)
    want = ref.act(obs, 5, steps, [0.2, 0.2], False)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_act_shape_errors(pb):
    st = pb.make_td3_state(2, 5, 2, [32, 32], 1.0, 1, precision="ffma32")
    with pytest.raises(pb.ShapeError):
        pb.act(st, np.zeros((2, 3, 4), np.float32), [0.1, 0.1], 0, [0, 0])
    with pytest.raises(pb.ShapeError):
        pb.act(st, np.zeros((2, 3, 5), np.float32), [0.1], 0, [0, 0])
