"""BF16 tensor-core mode vs the CPU oracle: tolerance-based parity (north_star: "TF32/BF16
inputs with fp32 accumulate ... within a stated fp32-relative tolerance").

BF16 mode stores the activations that feed the tensor cores (critic / policy inputs, hidden
activations, hidden cotangents) and the weight operand copies as bf16 (round to nearest, 8
significant bits); every product accumulates in fp32 in TMEM, and biases, output layers, losses,
the TD target, Adam and Polyak run in fp32 on the fp32 master weights.  Same metrics as the TF32
test (per-step loss relative error; weight-delta relative L2 after K steps).  Tolerances
are derived per case on the CPU (3x the error of the oracle run with BF16-rounded tensor-core
operands against the exact fp32 oracle: oracle/derive_tolerances.py -> tests/golden/tolerances.json).
"""
import numpy as np
import pytest

from helpers import TD3_NETS, check_parity, to_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb(cuda):
    import paper_2206_08888_b200 as pb
    return pb


@pytest.mark.parametrize("case", ["A_td3_pop4", "A_sac_pop4", "W_td3_da3", "W_sac_da8",
                                  "H_td3_3x512"])
def test_bf16_matches_oracle_within_derived_tolerance(pb, ora, case):
    """Config-A shapes, other action widths, 3 x 512 hidden (config E's shape: output layers
    outside the fused epilogue)."""
    check_parity(pb, ora, case, "bf16")


def test_bf16_weight_writes_refresh_the_operand_copies(pb, ora):
    """set_member / copy_member write the fp32 masters; the bf16 tensor-core copies must follow:
    a population whose member 1 is overwritten with member 0 computes, for member 1, exactly
    what member 0 computes (same weights, same batch rows, zero target noise -- the only
    member-keyed randomness of a TD3 step)."""
    n, B = 2, 256
    st = pb.make_td3_state(n, 17, 6, [256, 256], 1.0, 5, precision="bf16")
    for net in TD3_NETS:
        st.copy_member(net, 0, 1)
    raw = ora.synthetic_batches(1, n, B, 17, 6, 5)
    s, a, r, s2, d = (x[0].copy() for x in raw)
    for x in (s, a, r, s2, d):
        x[1] = x[0]
    hy = pb.Td3Hyper.defaults(n)
    hy.policy_delay_ratio = [1.0] * n
    hy.target_std = [0.0] * n
    pb.td3_update_step(st, to_batch(pb, (s, a, r, s2, d)), hy)
    for net in TD3_NETS:
        p = st.params(net)
        assert np.array_equal(p[0], p[1]), net


def test_bf16_deterministic(pb, ora):
    n, B = 3, 256
    a = pb.make_td3_state(n, 17, 6, [256, 256], 1.0, 5, precision="bf16")
    b = pb.make_td3_state(n, 17, 6, [256, 256], 1.0, 5, precision="bf16")
    raw = ora.synthetic_batches(3, n, B, 17, 6, 5)
    hy = pb.Td3Hyper.defaults(n)
    for k in range(3):
        pb.td3_update_step(a, to_batch(pb, raw, k), hy)
        pb.td3_update_step(b, to_batch(pb, raw, k), hy)
    for net in TD3_NETS:
        assert np.array_equal(a.params(net), b.params(net))


@pytest.mark.parametrize("case", ["H_td3_128x96", "H_sac_128x128", "H_td3_256x64"])
def test_bf16_fused_forward_hidden_shapes(pb, ora, case):
    """The fused two-layer forward (k_mlp_fwd2) at hidden widths other than 256: 128-wide
    layer 1 (two K chunks), layer-2 widths that leave TMEM columns / epilogue chunks unused."""
    check_parity(pb, ora, case, "bf16")


def test_bf16_large_batch_output_layer_is_a_loud_config_error(pb, ora):
    """Known BF16-mode boundary: with B * n_out > 32768 (policy: 8192 x 6)
    the output layer's backward would be a K = n_out < 8 dX product, which has no tensor-core
    shape and no bf16 CUDA-core fallback -- the update raises ConfigError instead of silently
    computing something else (TF32 / FFMA32 modes run it)."""
    import numpy as np
    from helpers import to_batch
    n, B = 2, 8192
    st = pb.make_td3_state(n, 17, 6, [128, 64], 1.0, 9, precision="bf16")
    raw = ora.synthetic_batches(1, n, B, 17, 6, 9)
    hy = pb.Td3Hyper.defaults(n)
    hy.policy_delay_ratio = [1.0] * n
    with pytest.raises(pb.ConfigError):
        pb.td3_update_step(st, to_batch(pb, raw, 0), hy)
