"""The reference's benchmark harness (bench.hpp / bench.cpp) on the device, mirroring
proj/tests/test_bench.cpp: timed repetitions with the warm-up separated, the three modes doing
identical numerical work (cross-mode audit; exact in the FFMA32 check mode), a vectorized launch
count independent of the population (sequential = N x vectorized), the memory-budget
ResourceError, the SAC path, and k-step batching equal to the chained loop byte for byte."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hz(cuda):
    from paper_2206_08888_b200 import harness
    return harness


def tiny(hz, mode, n):
    return hz.BenchConfig(mode=mode, n=n, k=3, reps=3, batch=16, obs_dim=5, act_dim=2,
                          hidden=[8, 8])


def test_bench_update_repetitions_with_warmup(hz):
    for mode in hz.BENCH_MODES:
        r = hz.bench_update(tiny(hz, mode, 2))
        assert len(r.times_ms) == 3 and r.median_ms > 0 and r.warmup_ms > 0
        assert r.mode == mode
        assert r.csv_row().startswith(mode + ",2,3,3,")


def test_bench_modes_identical_numerical_work(hz):
    assert hz.bench_cross_mode_audit(tiny(hz, "vectorized", 3)) == 0.0


def test_vectorized_launches_independent_of_population(hz):
    c1, c32 = tiny(hz, "vectorized", 1), tiny(hz, "vectorized", 32)
    c1.k = c32.k = 2
    r1, r32 = hz.bench_update(c1), hz.bench_update(c32)
    assert r1.kernel_launches == r32.kernel_launches > 0
    s32 = tiny(hz, "sequential", 32)
    s32.k = 2
    assert hz.bench_update(s32).kernel_launches == 32 * r32.kernel_launches


def test_memory_budget_is_a_resource_error(hz):
    import paper_2206_08888_b200 as pb
    cfg = tiny(hz, "vectorized", 64)
    cfg.memory_budget_bytes = 1024
    with pytest.raises(pb.ResourceError):
        hz.bench_update(cfg)


def test_sac_path_runs(hz):
    cfg = tiny(hz, "vectorized", 2)
    cfg.algo = "sac"
    assert hz.bench_update(cfg).median_ms > 0


@pytest.mark.parametrize("precision", ["ffma32", "bf16"])
def test_k_step_batching_equals_chained_loop(hz, tmp_path, precision):
    cfg = tiny(hz, "vectorized", 2)
    cfg.k = 10
    if precision == "bf16":
        cfg.hidden, cfg.batch = [32, 32], 32
    cfg.precision = precision
    t = hz.time_k_step_batching(cfg, reps=3, scratch_dir=str(tmp_path))
    assert t.bitwise_equal and t.batched_ms > 0 and t.loop_ms > 0
