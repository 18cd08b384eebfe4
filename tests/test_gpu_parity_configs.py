"""TF32 / BF16 parity at the configurations the bench measures, against the
exact fp32 oracle, with tolerances derived on the CPU (oracle/derive_tolerances.py ->
tests/golden/tolerances.json: 3x the error of an oracle run whose tensor-core operands are
rounded to the same precision).

* config D shape at pop 40 and 80 (TD3 2x256, B256): the grouped GEMMs run 160-320 tiles on 148
  SMs, so the persistent kernels take several tiles per CTA (second TMEM accumulator buffer,
  phase flips); default policy delay 0.5, so K=4 covers fire and non-fire steps;
* config C (SAC pop 32, 2x256, B256);
* config E (TD3 3x512, B1024, pop 8);
* the replay-driven update (pbrl_update_k: device sample + K steps, k_replay_gather into the
  bf16 / fp32 operand layouts) equals the host-batch path bit for bit in both tensor-core modes,
  so the derived-tolerance parity above carries over to it.
"""
import numpy as np
import pytest

from helpers import TD3_NETS, bits_equal, check_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb(cuda):
    import paper_2206_08888_b200 as pb
    return pb


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
@pytest.mark.parametrize("case", ["D_td3_pop40", "D_td3_pop80", "C_sac_pop32", "E_td3_pop8"])
def test_benchmarked_configs_match_oracle(pb, ora, case, precision):
    check_parity(pb, ora, case, precision)


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
def test_replay_driven_update_equals_host_batches(pb, precision):
    """Config D shape at pop 40: pbrl_update_k (device sampling into the tensor-core operand
    layouts) vs sample_batch to the host + td3_update_step, bitwise, K=4 (fire + non-fire)."""
    n, ds, da, cap, B, K = 40, 17, 6, 2000, 256, 4
    a = pb.make_td3_state(n, ds, da, [256, 256], 1.0, 8, precision=precision)
    b = pb.make_td3_state(n, ds, da, [256, 256], 1.0, 8, precision=precision)
    rep_a, rep_b = pb.DeviceReplay(a, cap), pb.DeviceReplay(b, cap)
    rng = np.random.default_rng(4)
    mem = np.repeat(np.arange(n, dtype=np.uint32), 1500)
    rows = mem.size
    s = rng.uniform(-1, 1, (rows, ds)).astype(np.float32)
    act = rng.uniform(-1, 1, (rows, da)).astype(np.float32)
    r = rng.uniform(-1, 1, rows).astype(np.float32)
    s2 = rng.uniform(-1, 1, (rows, ds)).astype(np.float32)
    d = (rng.random(rows) < 0.02).astype(np.float32)
    for rep in (rep_a, rep_b):
        rep.insert(s, act, r, s2, d, mem)
    hy = pb.Td3Hyper.defaults(n)
    assert pb.update_k_from_replay(a, rep_a, K, hy, B, seed=5, first_draw_id=100, min_size=1000)
    for i in range(K):
        bt = pb.sample_batch(rep_b, B, seed=5, draw_id=100 + i)
        pb.td3_update_step(b, bt, hy)
    for net in TD3_NETS:
        assert bits_equal(a.params(net), b.params(net)), net
    for la, lb in zip(a.last_losses(), b.last_losses()):
        assert np.array_equal(la, lb)
