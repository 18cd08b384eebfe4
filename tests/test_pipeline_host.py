"""Host-side pieces of the threaded training pipeline (include/pbrl_b200_pipeline.hpp):
RatioController, BoundedQueue and the built-in environment, compiled with g++ and run on the CPU
(no device, no library link)."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_pipeline_host_logic(tmp_path):
    exe = tmp_path / "test_pipeline_host"
    subprocess.run(["g++", "-std=c++17", "-O1", "-pthread", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "test_pipeline_host.cpp"), "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    assert "OK" in r.stdout
