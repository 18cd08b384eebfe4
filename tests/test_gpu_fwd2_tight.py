"""Tight check of the fused two-layer forward (k_mlp_fwd2, BF16 mode) through deterministic
`act` (algos.hpp:895-915 with the noise off): against a numpy forward that rounds exactly the
operands the kernel rounds -- the policy input and the hidden weights to bf16, layer-1
activations to bf16 after bias + ReLU -- and keeps everything else in fp32/fp64 (layer-2
activations, the output layer on the fp32 master weights, tanh).  What remains is fp32
accumulation order plus the odd one-ulp bf16 flip of an h1 element, so the bound is 10x tighter
than the generic tensor-core tolerance of test_gpu_act.py; any tile / chunk / bias-buffer
mistake in the kernel shows up as an O(1e-1) error.

Shapes: partial last row tiles, several tiles per CTA (b1 double buffer, W2 ring phases, E1/E2
overlap), a 128-wide layer 1, a 96-wide layer 2 (unused TMEM columns), output widths 6 (fixed
instantiation) and 2 (runtime-width instantiation)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 2e-3  # max |a_dev - a_ref| / bound


@pytest.fixture(scope="module")
def pb(cuda):
    import paper_2206_08888_b200 as pb
    return pb


def _bf16(x):
    """fp32 -> bf16 (round to nearest even) -> fp32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def _policy(row, dims, obs, bound):
    off, Ws, bs = 0, [], []
    for i in range(len(dims) - 1):
        k, m = dims[i], dims[i + 1]
        Ws.append(row[off:off + k * m].reshape(k, m).astype(np.float64))
        off += k * m
        bs.append(row[off:off + m].astype(np.float64))
        off += m
    h1 = _bf16(np.maximum(_bf16(obs).astype(np.float64) @ _bf16(Ws[0]) + bs[0], 0.0))
    h2 = np.maximum(h1.astype(np.float64) @ _bf16(Ws[1]).astype(np.float64) + bs[1], 0.0)
    return bound * np.tanh(h2 @ Ws[2] + bs[2])


@pytest.mark.parametrize("n,rows,hidden,da", [(3, 200, [256, 256], 6), (40, 1000, [256, 256], 6),
                                              (5, 300, [128, 96], 2), (2, 129, [256, 64], 6)])
def test_fused_forward_tight(pb, n, rows, hidden, da):
    ds, bound = 17, 2.0
    st = pb.make_td3_state(n, ds, da, hidden, bound, 13, precision="bf16")
    obs = np.random.default_rng(rows).uniform(-2, 2, (n, rows, ds)).astype(np.float32)
    got = pb.act(st, obs, None, 1, np.zeros(n, np.uint64), True)
    params = st.params("policy")
    dims = [ds] + list(hidden) + [da]
    err = 0.0
    for m in range(n):
        want = _policy(params[m], dims, obs[m], bound)
        err = max(err, float(np.abs(got[m] - want).max()) / bound)
    print(f"\nfused forward n={n} rows={rows} {hidden} da={da}: max |d|/bound = {err:.2e}")
    assert err <= TOL
