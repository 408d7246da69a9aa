"""CPU tests of the benchmark plumbing: the reference arm's JSON line and the
synthetic BASELINE-shape inputs."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_contract():
    import oracle as O
    if not O.ref_available():
        pytest.skip("reference library not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "2", "--warmup", "1", "--ntheta", "16", "--nrho", "128"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0


def test_synthetic_problem_matches_reference_structure():
    """synthetic.problem: make_grid's rho/theta grid, b <= 0, lam with one sign
    change per theta row (evolve.cpp:19-30), dt as select_dt."""
    from paper_2010_04760_b200 import synthetic
    p = synthetic.problem(256, 64)
    coef = p["coef"]
    assert coef.shape == (9, 64, 256)
    assert np.all(coef[0] <= 0.0)
    lam = coef[1]
    for k in range(64):
        neg = lam[k] < 0
        split = int(np.argmin(neg)) if not neg.all() else 256
        assert neg[:split].all() and not neg[split:].any() and split >= 1
    assert abs(p["rho"][-1] - 20.0) == 0.0
    assert abs(p["theta"][0] - np.pi / 128) < 1e-15
    assert synthetic.select_dt(p) == 0.5 * p["drho"]
    # slabs of the same global grid line up with the whole
    whole = synthetic.problem(300, 32)
    part = synthetic.problem(100, 32, rho_offset=150, nrho_global=300)
    np.testing.assert_array_equal(part["coef"], whole["coef"][:, :, 150:250])
    u = synthetic.initial_state(part)
    assert u.shape == (4, 36, 108) and np.all(u[1] == 0) and np.all(u[3] == 0)
