"""Device ports of glibc tanhf / expf / log1pf are bit-identical to the host libm.

The full 2^32 sweep was run on the CPU against the C transcriptions while writing the ports;
here the DEVICE code is compared with the host libm over every float in the ranges the update
path can reach densely, plus a stride over the whole bit space.
"""
import ctypes as C
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _libm_loop():
    """A tiny C helper compiled on the fly: apply libm tanhf/expf/log1pf to an array."""
    import subprocess
    import tempfile
    from pathlib import Path
    src = r"""
    #include <math.h>
    #include <stdint.h>
    void apply(int fn, const float* x, float* y, uint64_t n) {
      for (uint64_t i = 0; i < n; ++i) y[i] = fn == 0 ? tanhf(x[i]) : (fn == 1 ? expf(x[i]) : log1pf(x[i]));
    }"""
    d = Path(tempfile.mkdtemp())
    (d / "l.c").write_text(src)
    subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-o", str(d / "l.so"),
                    str(d / "l.c"), "-lm"], check=True)
    lib = C.CDLL(str(d / "l.so"))
    lib.apply.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64]
    return lib


@pytest.fixture(scope="module")
def host_libm():
    return _libm_loop()


def _dense(lo, hi, cap=1 << 25):
    """Every float with bits between float(lo) and float(hi) (same sign), thinned to <= cap."""
    ua, ub = sorted((int(np.float32(lo).view(np.uint32)), int(np.float32(hi).view(np.uint32))))
    step = max(1, (ub - ua) // cap)
    return np.arange(ua, ub + 1, step, dtype=np.uint64).astype(np.uint32)


@pytest.mark.parametrize("fn,spans", [
    (0, [(0.25, 4.0), (-0.25, -4.0), (1e-6, 0.25), (4.0, 12.0)]),
    (1, [(0.5, 16.0), (-0.5, -16.0), (-16.0, -104.0), (1e-7, 0.5)]),
    (2, [(1e-7, 0.5), (0.5, 64.0), (-1e-7, -0.5), (-0.5, -0.99999)]),
])
def test_device_libm_matches_host(cuda, host_libm, fn, spans):
    import torch
    from paper_2206_08888_b200 import _lib
    bits = np.concatenate([_dense(a, b) for a, b in spans] +
                          [np.arange(0, 2 ** 32, 7919, dtype=np.uint64).astype(np.uint32)])
    x = bits.view(np.float32)
    x = np.ascontiguousarray(x[~np.isnan(x)])
    want = np.empty_like(x)
    host_libm.apply(fn, x.ctypes.data, want.ctypes.data, x.size)
    xd = torch.from_numpy(x).to(cuda)
    yd = torch.empty_like(xd)
    _lib.call("pbrl_selftest_libm", fn, xd.data_ptr(), yd.data_ptr(), x.size)
    got = yd.cpu().numpy()
    same = (got.view(np.uint32) == want.view(np.uint32)) | (np.isnan(got) & np.isnan(want))
    bad = np.flatnonzero(~same)
    assert bad.size == 0, f"{bad.size} mismatches of {x.size}, first x={x[bad[:5]]}"
