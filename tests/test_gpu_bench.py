"""bench.py's driver contract on one GPU: one JSON line with the contract keys; `--gpus 2`
spawns two ranks itself (they share the GPU here, collectives on gloo) and the PBT exchange runs
through the library's sharded path with a cross-rank transport."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
        "gpu_launches", "clocks"}


def _bench(*args, timeout=600):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "6", "--warmup", "3",
                        "--no-cpu-baseline", *args], capture_output=True, text=True,
                       timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_single_gpu_line(cuda):
    d = _bench("--pop", "8")
    assert KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["scaling"] == "strong" and d["value"] > 0
    assert d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
    assert d["reps"]["n"] == 5 and d["pbt_exchange"]["replaced"] == 3
    assert d["class_hbm"]["gather_pack"]["gbs"] > 0


def test_bench_two_ranks_spawned(cuda):
    d = _bench("--pop", "8", "--gpus", "2", "--no-e2e")
    assert d["ranks"] == 2 and d["config"]["population"] == 8
    assert d["config"]["population_per_gpu"] == 4
    assert d["pbt_exchange"]["transport"] == "host"


def test_bench_config_b_reports_vectorization_overhead(cuda):
    d = _bench("--config", "B", "--no-e2e")
    assert d["vectorization_overhead"]["ratio"] > 0
