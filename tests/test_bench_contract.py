"""bench.py's driver contract on the CPU: the reference arm prints ONE JSON
line with the required keys (and exits 0 on non-zero ranks); the GPU arms'
lines are checked in the GPU suite (test_bench_gpu_line)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "e2e",
            "cpu_baseline", "impl"}


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, env=e, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    return [l for l in r.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_line():
    lines = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert REQUIRED <= set(d) and d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1


def test_reference_arm_nonzero_rank_exits_quietly():
    lines = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"],
                 env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert lines == []


@pytest.mark.gpu
def test_bench_gpu_line():
    lines = _run(["--steps", "3", "--warmup", "3", "--no-cpu-baseline"])
    d = json.loads(lines[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "roofline", "clocks", "e2e",
              "gpu_launches"):
        assert k in d, k
    assert d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    r = d["roofline"]
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert abs(r["achieved"] - r["flops_per_step"] / (r["gemm_ms_per_step"] * 1e-3) / 1e12) < 1e-6 * r["achieved"]
    assert r["gemm_ms_per_step"] < r["instrumented_ms_per_step"]
    # the reference arm runs the same workload (driver's same_config check)
    ref = json.loads(_run(["--impl", "reference", "--steps", "1", "--warmup", "0"])[-1])
    assert ref["config"] == d["config"]
