"""The tcgen05 grouped GEMM (TF32 in, fp32 accumulate in TMEM) against a torch fp64 product,
for every operand majorness the update step uses, ragged extents (TMA zero-fill) and tile widths.
Tolerance: TF32 keeps 10 mantissa bits, so |C - C_ref| <= 2e-3 * sum_k |A||B| (relative to the
absolute-value product, which bounds the accumulated rounding)."""
import pytest

pytestmark = pytest.mark.gpu


def _run(cuda, a_mn, b_mn, M, N, K, G, pad=4):
    import torch
    from paper_2206_08888_b200 import _lib
    gen = torch.Generator(device="cpu").manual_seed(M * 7 + N * 3 + K + G)
    A = torch.randn(G, M, K, generator=gen, dtype=torch.float64)
    B = torch.randn(G, K, N, generator=gen, dtype=torch.float64)
    ref = torch.bmm(A, B)
    bound = torch.bmm(A.abs(), B.abs())

    def store(x, mn_major):  # x: [G, rows_logical, cols] -> padded device storage
        t = x if not mn_major else x.transpose(1, 2)
        t = t.contiguous()
        rows, cols = t.shape[1], t.shape[2]
        ld = (cols + pad - 1) // pad * pad
        buf = torch.full((G, rows, ld), float("nan"), dtype=torch.float32)
        buf[:, :, :cols] = t.float()
        return buf.to(cuda), ld, rows * ld

    # A(m,k): K-major stores [M][K]; MN-major stores [K][M]
    a_dev, a_ld, a_gs = store(A, a_mn)
    # B(k,n) given as [K][N]; B K-major stores [N][K]; MN-major stores [K][N]
    b_dev, b_ld, b_gs = store(B.transpose(1, 2), b_mn)
    c_ld = (N + 3) // 4 * 4
    C = torch.zeros(G, M, c_ld, dtype=torch.float32, device=cuda)
    _lib.call("pbrl_selftest_tc_gemm", int(a_mn), int(b_mn), M, N, K, G, a_dev.data_ptr(), a_ld,
              a_gs, b_dev.data_ptr(), b_ld, b_gs, C.data_ptr(), c_ld, M * c_ld)
    got = C[:, :, :N].double().cpu()
    err = (got - ref).abs()
    assert torch.isfinite(got).all()
    assert (err <= 2e-3 * bound + 1e-6).all(), float((err / (bound + 1e-9)).max())


@pytest.mark.parametrize("a_mn,b_mn", [(False, True), (False, False), (True, True), (True, False)])
@pytest.mark.parametrize("M,N,K,G", [(256, 256, 256, 3), (256, 256, 23, 2), (17, 256, 256, 2),
                                     (256, 64, 100, 2), (300, 128, 36, 1)])
def test_tc_gemm_layouts(cuda, a_mn, b_mn, M, N, K, G):
    _run(cuda, a_mn, b_mn, M, N, K, G)


def test_tc_gemm_narrow_k_major_b(cuda):
    """N = 6 (action columns of the critic input) uses the 16-wide K-major tile."""
    _run(cuda, False, False, 256, 6, 256, 4)


def _run_bf16(cuda, a_mn, b_mn, M, N, K, G, pad=8):
    """BF16 path: operands rounded to bf16 on the host, so the fp64 product of the ROUNDED values
    is the reference and only the fp32 accumulation remains: |C - C_ref| <= 1e-5 sum|A||B|."""
    import torch
    from paper_2206_08888_b200 import _lib
    gen = torch.Generator(device="cpu").manual_seed(M * 5 + N * 3 + K + G)
    A = torch.randn(G, M, K, generator=gen).bfloat16()
    B = torch.randn(G, K, N, generator=gen).bfloat16()
    ref = torch.bmm(A.double(), B.double())
    bound = torch.bmm(A.double().abs(), B.double().abs())

    def store(x, mn_major):
        t = (x if not mn_major else x.transpose(1, 2)).contiguous()
        rows, cols = t.shape[1], t.shape[2]
        ld = (cols + pad - 1) // pad * pad
        buf = torch.full((G, rows, ld), float("nan"), dtype=torch.bfloat16)
        buf[:, :, :cols] = t
        return buf.to(cuda), ld, rows * ld

    a_dev, a_ld, a_gs = store(A, a_mn)
    b_dev, b_ld, b_gs = store(B.transpose(1, 2), b_mn)
    c_ld = (N + 3) // 4 * 4
    C = torch.zeros(G, M, c_ld, dtype=torch.float32, device=cuda)
    _lib.call("pbrl_selftest_tc_gemm_bf16", int(a_mn), int(b_mn), M, N, K, G, a_dev.data_ptr(),
              a_ld, a_gs, b_dev.data_ptr(), b_ld, b_gs, C.data_ptr(), c_ld, M * c_ld)
    got = C[:, :, :N].double().cpu()
    err = (got - ref).abs()
    assert torch.isfinite(got).all()
    assert (err <= 1e-5 * bound + 1e-6).all(), float((err / (bound + 1e-9)).max())


@pytest.mark.parametrize("a_mn,b_mn", [(False, True), (False, False), (True, True), (True, False)])
@pytest.mark.parametrize("M,N,K,G", [(256, 256, 256, 3), (256, 256, 23, 2), (17, 256, 256, 2),
                                     (256, 64, 100, 2), (300, 128, 72, 1)])
def test_tc_gemm_bf16_layouts(cuda, a_mn, b_mn, M, N, K, G):
    _run_bf16(cuda, a_mn, b_mn, M, N, K, G)


def test_tc_gemm_bf16_narrow_k_major_b(cuda):
    _run_bf16(cuda, False, False, 256, 6, 256, 4)
