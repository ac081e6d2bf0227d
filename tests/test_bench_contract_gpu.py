"""bench.py's JSON line keeps the driver contract (one line; the keys the
driver and the judge read), on the real workloads: the default C4 batch and
the reference arm's line shape.  A short run (3 steps) -- the numbers are not
checked, only that a value exists, the parity gate passed and the roofline /
e2e records are complete."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "cpu_baseline", "clocks", "gpu_launches",
        "parity"}


def _line(*args):
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("workload", ["c4", "c3"])
def test_bench_line_contract(workload):
    d = _line("--workload", workload, "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert KEYS <= set(d), KEYS - set(d)
    assert d["value"] and d["value"] > 0 and d["parity"]["ok"] is True
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith(workload)
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "kernel", "kernel_ms"):
        assert k in r, k
    assert 0 < r["frac"] < 1 and r["unit"] == "GB/s"
    assert d["gpu_launches"] >= 3
    assert d["clocks"]["sm_mhz"] > 0
