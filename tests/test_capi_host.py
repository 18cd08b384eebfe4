"""CPU-side checks of the drop-in boundary and the host mirror (no GPU needed):
the C-ABI library loads and exports every symbol include/pbrl_b200.h declares, error codes map
onto the reference exception taxonomy, and the host RNG / PBT / hyper logic matches the oracle."""
import ctypes as C
import math
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared_symbols():
    txt = (ROOT / "include" / "pbrl_b200.h").read_text()
    return sorted(set(re.findall(r"^int\s+(pbrl_\w+)\s*\(", txt, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2206_08888_b200 import _lib
    lib = _lib.lib()
    syms = _declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares every one of them
    assert not [s for s in syms if s not in _lib.SIGNATURES], "binding out of sync with header"


def test_error_codes_map_to_reference_exceptions():
    import paper_2206_08888_b200 as pb
    from paper_2206_08888_b200.errors import raise_for
    for code, cls in [(-1, pb.ShapeError), (-2, pb.ConfigError), (-3, pb.UsageError),
                      (-4, pb.NotReadyError), (-5, pb.ResourceError),
                      (-6, pb.DataStarvationError)]:
        with pytest.raises(cls):
            raise_for(code, "x")


def test_null_handle_is_a_usage_error():
    from paper_2206_08888_b200 import _lib
    lib = _lib.lib()
    n = C.c_uint64()
    assert lib.pbrl_param_count(None, 0, C.byref(n)) == -3
    assert "null population handle" in _lib.last_error()


def test_rng_mirror_matches_oracle(ora):
    import paper_2206_08888_b200 as pb
    for seed, stream, use, step in [(0, 0, 1, 0), (7, 3, 4, 99), (2**63 + 5, 12345, 12, 2**40)]:
        s = pb.RngStream.of(seed, stream, use, step)
        assert s.key == ora.stream_key(seed, stream, use, step)
        for c in (0, 1, 77, 2**40):
            assert s.uniform(c) == ora.uniform(s.key, c)
    assert pb.mix64(12345) == ora.mix64(12345)


def test_prior_draws_match_oracle(ora):
    """Td3Prior / SacPrior re-draws (host, exact libm) == the oracle's restatement."""
    import ctypes
    import paper_2206_08888_b200 as pb
    lib = ora.lib
    lib.ora_td3_prior_sample.argtypes = [ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64),
                                         ctypes.POINTER(ctypes.c_double)]
    lib.ora_sac_prior_sample.argtypes = [ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64),
                                         ctypes.c_double, ctypes.POINTER(ctypes.c_double)]
    rng = pb.RngSequence(3, 0, "kDonorChoice")
    nxt = ctypes.c_uint64(0)
    out = (ctypes.c_double * 8)()
    for _ in range(50):
        h = pb.Td3Prior().sample_member(rng)
        lib.ora_td3_prior_sample(rng.stream.key, ctypes.byref(nxt), out)
        assert [getattr(h, f)[0] for f in pb.Td3Hyper.FIELDS] == list(out)
    rng = pb.RngSequence(4, 0, "kDonorChoice")
    nxt = ctypes.c_uint64(0)
    out7 = (ctypes.c_double * 7)()
    for _ in range(50):
        h = pb.SacPrior(default_target_entropy=-6.0).sample_member(rng)
        lib.ora_sac_prior_sample(rng.stream.key, ctypes.byref(nxt), -6.0, out7)
        assert [getattr(h, f)[0] for f in pb.SacHyper.FIELDS] == list(out7)


def test_prior_ranges_and_log_uniform():
    """Acceptance criterion 6 (acceptance_main.cpp:434-470): prior draws stay in range and the
    log-uniform lrs are uniform in log space (KS statistic < 0.01 over 1e5 draws)."""
    import paper_2206_08888_b200 as pb
    rng = pb.RngSequence(9, 0, "kHyperDraw")
    pr = pb.Td3Prior()
    draws = [pr.sample_member(rng) for _ in range(20000)]
    lr = np.sort(np.log([d.critic_lr[0] for d in draws]))
    lo, hi = math.log(3e-5), math.log(3e-3)
    cdf = (lr - lo) / (hi - lo)
    ks = np.max(np.abs(cdf - (np.arange(1, lr.size + 1) / lr.size)))
    assert ks < 0.015
    assert all(0.2 <= d.policy_delay_ratio[0] <= 1.0 and 0.9 <= d.gamma[0] <= 1.0 for d in draws)


def test_pbt_state_and_rank_semantics():
    """evolve.hpp:80-122 / test_evolve.cpp:19-48."""
    import paper_2206_08888_b200 as pb
    st = pb.PBTState(3)
    for m, v in enumerate([5, 1, 9]):
        st.record_return(m, v)
    assert pb.pbt_rank(st) == [2, 0, 1]
    st2 = pb.PBTState(3)
    for m in range(3):
        st2.record_return(m, 3)
    assert pb.pbt_rank(st2) == [0, 1, 2]
    ring = pb.PBTState(1)
    for i in range(25):
        ring.record_return(0, i)
    assert len(ring.returns[0]) == 10 and ring.returns[0][0] == 15.0
    assert ring.mean_return(0) == pytest.approx((15 + 24) / 2.0)
    empty = pb.PBTState(3)
    empty.record_return(0, 1.0)
    with pytest.raises(pb.NotReadyError):
        pb.pbt_rank(empty)


def test_hyper_validation_matches_reference():
    """Td3Hyper::validate (algos.hpp:81-108)."""
    import paper_2206_08888_b200 as pb
    h = pb.Td3Hyper.defaults(2)
    h.validate(2)
    for field, bad in [("critic_lr", 0.0), ("policy_delay_ratio", 1.5), ("target_std", -0.1),
                       ("gamma", 0.5), ("tau", 0.0)]:
        h2 = pb.Td3Hyper.defaults(2)
        getattr(h2, field)[1] = bad
        with pytest.raises(pb.ConfigError):
            h2.validate(2)
    h3 = pb.Td3Hyper.defaults(2)
    h3.gamma = [0.0, 0.99]  # gamma = 0 allowed (tests)
    h3.validate(2)
    with pytest.raises(pb.ConfigError):
        pb.Td3Hyper.defaults(3).validate(2)


def test_cpp_facade_compiles():
    """include/pbrl_b200.hpp (reference names + exception types over the C ABI) builds and
    links against the in-tree library."""
    import subprocess
    r = subprocess.run(["make", "-s", "-B", "-C", str(ROOT / "examples")], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr


def test_harness_host_logic():
    """bench.cpp:20-56 host logic: mode names, config validation, median / IQR, the footprint
    estimate (no device needed)."""
    from paper_2206_08888_b200 import harness as hz
    from paper_2206_08888_b200.errors import ConfigError
    for m in hz.BENCH_MODES:
        assert hz.parse_bench_mode(m) == m
    with pytest.raises(ConfigError):
        hz.parse_bench_mode("gpu")
    with pytest.raises(ConfigError):
        hz.BenchConfig(reps=2).validate()
    r = hz.BenchResult(times_ms=[5.0, 1.0, 4.0, 2.0, 3.0])
    hz.summarize_bench(r)
    assert r.median_ms == 3.0 and r.iqr_ms == 4.0 - 2.0
    cfg = hz.BenchConfig(n=3, k=4, batch=16, obs_dim=5, act_dim=2, hidden=[8, 8])
    pol = 5 * 8 + 8 + 8 * 8 + 8 + 8 * 2 + 2
    q = 7 * 8 + 8 + 8 * 8 + 8 + 8 + 1
    want = 3 * (pol + 2 * q) * 16 + 4 * 3 * 16 * (2 * 5 + 2 + 2) * 4 + 16 * 3 * 16 * 8 * 4
    assert hz.bench_estimated_bytes(cfg) == want
