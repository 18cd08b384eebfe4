"""The DvD host math of the library (pbrl_dvd_loss / pbrl_median_pairwise_distance /
pbrl_dvd_lambda: the n x n log-determinant loss the DvD hook evaluates on the host in double,
evolve.hpp:304-499) against the pinned oracle, bit for bit; plus the host-side argument checks of
the DvD / CEM Python mirror.  CPU only: these entry points never touch the device."""
import numpy as np
import pytest

import paper_2206_08888_b200 as pb


def test_dvd_loss_bitexact_vs_oracle(ora):
    rng = np.random.default_rng(11)
    for n, dim in ((2, 3), (6, 12), (16, 40)):
        e = rng.normal(size=(n, dim))
        for ls, jit, lam in ((0.9, 1e-8, 1.3), (2.0, 0.0, 0.5), (0.3, 1e-6, 0.1)):
            got = pb.dvd_loss(e, ls, jit, lam)
            want = ora.dvd_loss(e, ls, jit, lam)
            assert got.loss == want[0] and got.logdet == want[1]
            assert np.array_equal(got.grad.view(np.uint64), want[2].view(np.uint64))
        assert pb.median_pairwise_distance(e) == ora.median_pairwise_distance(e)
    # permutation invariance is exact (test_evolve.cpp:267-285)
    e = rng.normal(size=(7, 5))
    perm = rng.permutation(7)
    a, b = pb.dvd_loss(e, 0.9, 1e-8, 1.3), pb.dvd_loss(e[perm], 0.9, 1e-8, 1.3)
    assert a.loss == b.loss and np.array_equal(a.grad[perm], b.grad)


def test_dvd_loss_errors_and_schedule(ora):
    same = np.ones((3, 4))
    with pytest.raises(pb.DegeneratePopulationError):
        pb.dvd_loss(same, 1.0, 0.0, 1.0)  # test_evolve.cpp:255-265
    out = pb.dvd_loss(same, 1.0, 1e-3, 1.0)
    assert np.isfinite(out.loss) and out.logdet <= 3 * np.log(1 + 3 + 1e-3)
    with pytest.raises(pb.ConfigError):
        pb.dvd_loss(same[:1], 1.0, 0.0, 1.0)
    with pytest.raises(pb.ConfigError):
        pb.dvd_loss(np.eye(3), 0.0, 0.0, 1.0)
    assert pb.median_pairwise_distance(same) == 1.0
    s = pb.LambdaSchedule(0.1, 0.7, 100)  # test_evolve.cpp:203-215
    assert pb.dvd_lambda(0, s) == 0.1 and pb.dvd_lambda(100, s) == 0.7
    assert pb.dvd_lambda(10**6, s) == 0.7
    for t in (0, 1, 37, 99, 100):
        assert pb.dvd_lambda(t, s) == ora.dvd_lambda(t, 0.1, 0.7, 100)
    prev = pb.dvd_lambda(0, s)
    for t in range(1, 120):
        cur = pb.dvd_lambda(t, s)
        assert cur >= prev
        prev = cur
    with pytest.raises(pb.ConfigError):
        pb.DvDConfig([0.0] * 6, 2, 1.0).validate(3)  # fewer probe states than members
