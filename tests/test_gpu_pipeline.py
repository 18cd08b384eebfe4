"""The threaded run_training on the device (include/pbrl_b200_pipeline.hpp, SURVEY.md §8(f)
item 2): actor threads acting through device snapshot refreshes, the ingest thread's batched
device inserts under the ratio guard, device sample + update bursts on the learner thread, PBT,
and the shared-critic strategies: CEM generations (policy mask on the replay-driven update, device
resample / refit) and the DvD hook (pipeline_run.hpp:143-181, :343-409).
Runs examples/run_training_demo (C++) and checks its summary."""
import re
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("precision,pbt", [("bf16", "pbt"), ("ffma32", "none"), ("bf16", "cem"),
                                           ("bf16", "dvd")])
def test_run_training_demo(cuda, precision, pbt):
    subprocess.run(["make", "-s", "-C", str(ROOT / "examples"), "run_training_demo"], check=True)
    total, k, n = 1500, 20, 4
    r = subprocess.run([str(ROOT / "examples" / "run_training_demo"), str(n), "2", str(total),
                        str(k), str(pbt), precision], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    kv = dict(re.findall(r"(\w+)=([\d.]+)", r.stdout.splitlines()[0]))
    assert int(kv["update_steps"]) == total
    env = int(kv["env_steps"])
    nbuf = 1 if pbt in ("cem", "dvd") else n  # CEM / DvD train from one shared ring
    assert env >= nbuf * 200  # at least the warm-up of every ring
    assert int(kv["dropped"]) == 0
    assert int(kv["published"]) >= total // k
    assert int(kv["device_inserts"]) > 0
    # the ratio guard (target 1 update per member env step, slack 5 %): the sample side never
    # runs ahead of target (1 + slack) env steps (replay.hpp:262-266), the insert side never
    # more than (1 + slack) behind plus the warm-up (:267-270)
    assert total <= 1.05 * env / n + k, r.stdout
    assert env <= 1.05 * n * total + nbuf * 200 + 2 * n, r.stdout
    if pbt in ("pbt", "cem"):  # PBT evolutions / CEM generations
        assert int(kv["evolve_events"]) >= 1, r.stdout
    returns = [float(x) for x in r.stdout.splitlines()[1].split()[1:]]
    assert len(returns) == 4 and all(x > -1e9 for x in returns)
