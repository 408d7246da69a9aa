"""CPU tests: the C restatement (oracle/hweno_oracle.c) against the reference's
own known-answer tests and against golden vectors produced by the unmodified
reference library (tests/golden/make_golden.py)."""
import math

import numpy as np
import pytest

from conftest import golden_cases, load_golden
from helpers import interior, oracle_from_golden, rel_linf
import oracle as O


# ---------------------------------------------------------------- weight KATs
# proj/tests/test_spatial.cpp:33-66
@pytest.mark.parametrize("window", [[7.0] * 5, [0.0, 1.0, 2.0, 3.0, 4.0]])
def test_weno5_weights_linearish(window):
    import ctypes as C
    lib = O.orc_lib()
    a = np.array(window)
    w = np.zeros(3)
    lib.orc_weno5_weights_f64(a.ctypes.data_as(O._dp), 1e-6, w.ctypes.data_as(O._dp))
    assert np.allclose(w, [0.1, 0.6, 0.3], atol=1e-15, rtol=0)
    wf = (C.c_float * 3)()
    lib.orc_weno5_weights_f32(a.ctypes.data_as(O._dp), C.c_float(1e-6), wf)
    assert np.allclose(list(wf), [0.1, 0.6, 0.3], atol=1e-7, rtol=0)


def test_weno5_weights_step_window():
    """Hand-evaluated IS = (0, 4/3, 10/3) for the step (0,0,0,1,1)."""
    lib = O.orc_lib()
    a = np.array([0.0, 0.0, 0.0, 1.0, 1.0])
    w = np.zeros(3)
    eps = 1e-6
    lib.orc_weno5_weights_f64(a.ctypes.data_as(O._dp), eps, w.ctypes.data_as(O._dp))
    a0 = 0.1 / (eps * eps)
    a1 = 0.6 / (eps + 4 / 3) ** 2
    a2 = 0.3 / (eps + 10 / 3) ** 2
    s = a0 + a1 + a2
    assert abs(w[0] - a0 / s) / w[0] <= 1e-14
    assert abs(w[1] - a1 / s) / w[1] <= 1e-13
    assert abs(w[2] - a2 / s) / w[2] <= 1e-13
    assert w[2] <= 1e-10 * w[0]
    assert abs(w.sum() - 1.0) <= 1e-15


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_weights_match_reference_fp64_weights():
    """Reference mixed mode computes the weights in fp64 — the oracle's f64
    weights must agree bitwise (same expression order)."""
    rng = np.random.default_rng(5)
    lib = O.orc_lib()
    for _ in range(200):
        a = rng.normal(size=5) * 10.0 ** rng.integers(-3, 3)
        w = np.zeros(3)
        lib.orc_weno5_weights_f64(a.ctypes.data_as(O._dp), 1e-6, w.ctypes.data_as(O._dp))
        wr = O.ref_weno5_weights(a, 1e-6, "mixed")
        assert np.array_equal(w, wr)


# ---------------------------------------------------------------- row derivative
def _row(u, drho, mode, minus, eps=1e-6):
    lib = O.orc_lib()
    u = np.ascontiguousarray(u, dtype=np.float64)
    n = u.size - 8
    du = np.zeros(n)
    lib.orc_weno5_row_derivative(u[4:].ctypes.data_as(O._dp), n, drho, 0 if mode == "f64" else 1,
                                 eps, int(minus), du.ctypes.data_as(O._dp))
    return du


@pytest.mark.parametrize("mode", ["f64", "mixed"])
@pytest.mark.parametrize("minus", [False, True])
def test_weno5_constant_and_quadratic(mode, minus):
    """proj/tests/test_spatial.cpp:68-93 (constants -> 0; d(x^2) = 2x exactly)."""
    du = _row(np.full(24, 3.25), 0.1, mode, minus)
    assert np.max(np.abs(du)) <= 1e-12
    n, h = 24, 0.1
    x = h * np.arange(-4, n + 4)
    du = _row(x * x, h, mode, minus)
    assert np.max(np.abs(du - 2 * x[4:-4])) <= 1e-12


@pytest.mark.parametrize("minus", [False, True])
def test_weno5_sine_order(minus):
    """proj/tests/test_spatial.cpp:94-110: 5th order on a smooth sine."""
    errs = []
    for N in (64, 128, 256, 512):
        dr = 2.0 / (N - 1)
        x = dr * np.arange(-4, N + 4)
        d = _row(np.sin(x), dr, "f64", minus)
        errs.append(np.max(np.abs(d - np.cos(x[4:-4]))))
    slope = np.mean(np.log2(np.array(errs[:-1]) / np.array(errs[1:])))
    assert slope >= 4.5


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
@pytest.mark.parametrize("minus", [False, True])
def test_row_derivative_vs_reference(minus):
    rng = np.random.default_rng(11)
    u = rng.uniform(-1, 1, 40)
    ref_hi, _ = O.ref_weno5_row(u, 0.05, 1e-6, "full", minus)
    du = _row(u, 0.05, "f64", minus)
    assert np.max(np.abs(du - ref_hi)) / np.max(np.abs(ref_hi)) <= 1e-14


# ---------------------------------------------------------------- golden RHS
@pytest.mark.parametrize("case", golden_cases())
def test_oracle_rhs_matches_reference(case):
    g = load_golden(case)
    orc = oracle_from_golden(g, "f64")
    _, du = orc.rhs(g["u0"])
    assert rel_linf(du, g["rhs_full"]) <= 1e-13
    _, du = orc.rhs(g["urand"])
    assert rel_linf(du, g["rhs_rand_full"]) <= 1e-13
    orm = oracle_from_golden(g, "mixed")
    _, du = orm.rhs(g["u0"])
    assert rel_linf(du, g["rhs_mixed"]) <= 1e-6
    _, du = orm.rhs(g["urand"])
    assert rel_linf(du, g["rhs_rand_mixed"]) <= 1e-6


@pytest.mark.parametrize("case", golden_cases())
def test_oracle_linear_weights(case):
    g = load_golden(case)
    orc = oracle_from_golden(g, "f64", eps=math.inf)
    _, du = orc.rhs(g["urand"])
    assert rel_linf(du, g["rhs_rand_linear"]) <= 1e-13


@pytest.mark.parametrize("case", golden_cases())
def test_oracle_evolution_matches_reference(case):
    g = load_golden(case)
    orc = oracle_from_golden(g, "f64")
    u, st = orc.advance(g["u0"], float(g["dt"][0]), 0, int(g["steps"]), str(g["stepper"]))
    assert not st["blew_up"]
    assert rel_linf(u, g["state_full"]) <= 1e-12
    orm = oracle_from_golden(g, "mixed")
    u, st = orm.advance(g["u0"], float(g["dt"][0]), 0, int(g["steps"]), str(g["stepper"]))
    assert rel_linf(u, g["state_mixed"]) <= 1e-6


@pytest.mark.parametrize("scheme", ["weno5", "weno3", "fd6ko"])
@pytest.mark.parametrize("mode", ["f64", "mixed"])
def test_zero_state_zero_rhs(scheme, mode):
    """proj/tests/test_evolve.cpp:150-170."""
    g = load_golden("extremal_w5")
    orc = oracle_from_golden(g, mode)
    orc = O.OracleSolver(int(g["nrho"]), int(g["ntheta"]), float(g["drho"]), float(g["dtheta"]),
                         int(g["parity"]), g["coef"], g["cotth"], scheme, mode)
    _, du = orc.rhs(np.zeros(orc.shape))
    assert np.all(du == 0.0)


def test_ghosts_cubic_and_parity():
    """proj/tests/test_evolve.cpp:80-148: cubic continuation is exact; theta
    ghosts mirror with sign (-1)^(m+s) bitwise."""
    for case in ("extremal_w5", "oddpar_w5"):
        g = load_golden(case)
        orc = oracle_from_golden(g)
        n, nt = int(g["nrho"]), int(g["ntheta"])
        rho = g["rho"]
        drho = float(g["drho"])
        u = np.zeros(orc.shape)
        for c in range(4):
            for k in range(nt):
                u[c, k + 2, 4:-4] = 1 + c + (2 + k) * rho - 3 * rho ** 2 + 0.5 * (c - 1) * rho ** 3
        ug, _ = orc.rhs(u)
        for c in range(4):
            for k in range(nt):
                cub = lambda r: 1 + c + (2 + k) * r - 3 * r ** 2 + 0.5 * (c - 1) * r ** 3  # noqa: E731
                for t in range(1, 5):
                    rl = rho[0] - drho * t
                    rr = rho[0] + drho * (n - 1 + t)
                    sc = abs(cub(rr)) + 1
                    assert abs(ug[c, k + 2, 4 - t] - cub(rl)) <= 1e-9 * sc
                    assert abs(ug[c, k + 2, 4 + n - 1 + t] - cub(rr)) <= 1e-9 * sc
        rng = np.random.default_rng(77)
        u = np.zeros(orc.shape)
        u[:, 2:-2, 4:-4] = rng.uniform(-1, 1, (4, nt, n))
        ug, _ = orc.rhs(u)
        sgn = int(g["parity"])
        for t in range(2):
            assert np.array_equal(ug[:, 1 - t, 4:-4], sgn * ug[:, 2 + t, 4:-4])
            assert np.array_equal(ug[:, nt + 2 + t, 4:-4], sgn * ug[:, nt + 1 - t, 4:-4])


def test_blowup_semantics():
    """proj/tests/test_evolve.cpp:352-361: |u| > 1e30 -> blew_up at step 1."""
    g = load_golden("extremal_w5")
    orc = oracle_from_golden(g)
    u = g["u0"].copy()
    u[0, 2 + 1, 4 + 30] = 1e31
    assert not orc.admissible(u)
    _, st = orc.advance(u, float(g["dt"][0]), 0, 5)
    assert st == dict(steps_done=1, blew_up=True, blowup_step=1)


def test_threaded_assembly_bitwise_equals_serial():
    """include/hweno_gpu_setup.hpp: the reference's own
    assemble_coefficients on theta-row sub-grids from a thread pool gives the
    serial planes bit for bit (hi and lo limbs, cot theta, max_speed -> dt)."""
    import oracle as O
    if not O.ref_available():
        pytest.skip("reference library not built")
    for phys in (O.Physics(a=1.0, spin=-2, mmode=2), O.Physics(a=0.9, spin=-2, mmode=0),
                 O.Physics(a=0.0, spin=0, mmode=0)):
        serial = O.RefSolver(phys, 96, 13, workers=1)
        threaded = O.RefSolver(phys, 96, 13, workers=4)
        for a, b in ((serial.coef, threaded.coef), (serial.coef_lo, threaded.coef_lo),
                     (serial.cotth, threaded.cotth), (serial.cotth_lo, threaded.cotth_lo)):
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
        assert serial.max_speed == threaded.max_speed
        assert serial.select_dt("ssprk33") == threaded.select_dt("ssprk33")
