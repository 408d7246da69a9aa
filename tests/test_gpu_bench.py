"""bench.py end to end on a small grid: the JSON line carries every key the
driver and DESIGN.md §5 rely on (headline metric, roofline, clocks, e2e,
gpu_launches, modes)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_line_small_grid(cuda_ok):
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--nrho", "2048", "--ntheta", "64",
         "--steps", "4", "--warmup", "3", "--no-dd", "--no-cpu", "--no-configs",
         "--e2e-steps", "2", "--e2e-lanes", "2"],
        capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "clocks", "e2e", "gpu_launches", "modes", "e2e_advance"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 4 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["gpu_launches"] == 12
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] == r["achieved"] / r["peak"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"f64", "mixed", "mixed-ssprk104"} <= set(d["modes"])
    assert "workload" in d["config"]
    # sustained figure with its own clock record; the drop-in at the driver's
    # observer cadence (round(0.25/dt) steps)
    su = d["sustained"]
    assert su["value"] > 0 and su["timed_s"] >= 2.0 and "sm_mhz" in su["clocks"]
    ep = d["e2e_advance_production"]
    assert ep["hook_every"] > 1 and ep["hook_calls"] == 3 and ep["value"] > 0
