"""GPU parity of the device coefficient assembly against
the unmodified reference: hwg_assemble_coefficients vs assemble_coefficients
(proj/src/geometry.cpp:118-168) bit for bit on the reference's own grids,
and hwg_wave_op_coeffs vs the reference's 36-digit known answers
(proj/tests/test_geometry.cpp:119-139) and its host evaluation (bitwise)."""
import os
from fractions import Fraction

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.int64)


def test_wave_op_coeffs_known_answers(cuda_ok):
    from paper_2010_04760_b200 import hwgpu
    z = np.load(os.path.join(GOLDEN, "coef_kat.npz"))
    got = hwgpu.wave_op_coeffs(z["inp"], z["spin_mmode"])
    # bitwise the reference library's host evaluation ...
    assert np.array_equal(bits(got), bits(z["host"]))
    # ... and within the reference test's 1e-26 of the 36-digit values
    for i in range(got.shape[0]):
        for q in range(11):
            w = Fraction(float(z["want"][i, q, 0])) + Fraction(float(z["want"][i, q, 1]))
            g = Fraction(float(got[i, q, 0])) + Fraction(float(got[i, q, 1]))
            assert abs(g - w) <= max(abs(w), 1) * Fraction(1, 10**26)


CASES = [  # (M, a, spin, mmode, nrho, ntheta): m1 and generic kernels, both parities
    (1.0, 1.0, -2, 2, 1024, 32),     # BASELINE C2 physics (extremal Kerr)
    (1.0, 0.9, -2, 0, 512, 16),      # C3 physics (lam changes sign)
    (1.0, 0.0, 0, 0, 1024, 64),      # C1 (Schwarzschild scalar), full size
    (1.0, 0.5, 1, 1, 300, 33),       # odd parity, ragged theta chunk
]


@pytest.mark.parametrize("M,a,spin,mmode,nrho,ntheta", CASES)
def test_assembly_bitwise_vs_reference(cuda_ok, M, a, spin, mmode, nrho, ntheta):
    import oracle as O
    from paper_2010_04760_b200 import hwgpu
    ref = O.RefSolver(O.Physics(M=M, a=a, spin=spin, mmode=mmode), nrho, ntheta, workers=8)
    want, ms = ref.coeffs_all_dd()
    rho, cth = ref.grid_dd()
    got = hwgpu.assemble_coefficients(rho, cth, M=M, a=a, S=20.0, spin=spin, mmode=mmode)
    for q, name in enumerate(hwgpu.COEF_PLANES):
        assert np.array_equal(bits(got[name]), bits(want[q])), name
    assert np.array_equal(bits(got["max_speed"]), bits(ms))
    # split limbs and a plane subset: the same values
    sp = hwgpu.assemble_coefficients(rho, cth, M=M, a=a, spin=spin, mmode=mmode,
                                     planes=("lam", "ath"), layout="split")
    assert set(sp) == {"lam", "ath", "max_speed"}
    assert np.array_equal(bits(sp["lam"][0]), bits(want[1][..., 0]))
    assert np.array_equal(bits(sp["ath"][1]), bits(want[8][..., 1]))


def test_wave_op_coeffs_random_points_bitwise(cuda_ok):
    """Both generated kernels (M == 1 and the generic one: a full grid to
    scri needs M = 1, geometry.hpp) at random points of the chart, random
    spin weights and modes: bitwise the reference's host evaluation."""
    import oracle as O
    from paper_2010_04760_b200 import hwgpu
    rng = np.random.default_rng(2010)
    n = 4000
    inp = np.zeros((n, 5, 2))
    inp[:, 0, 0] = rng.uniform(0.2, 19.9, n)
    inp[:, 0, 1] = inp[:, 0, 0] * rng.uniform(-1, 1, n) * 2.0**-54
    inp[:, 1, 0] = rng.uniform(-0.999, 0.999, n)
    inp[:, 2, 0] = np.where(rng.random(n) < 0.5, 1.0, rng.uniform(0.5, 2.0, n))
    inp[:, 3, 0] = inp[:, 2, 0] * rng.uniform(0.0, 1.0, n)
    inp[:, 4, 0] = rng.choice([15.0, 20.0, 30.0], n)
    sm = np.stack([rng.integers(-2, 3, n), rng.integers(-3, 4, n)], axis=1)
    want = O.ref_wave_op_coeffs(inp, sm)
    got = hwgpu.wave_op_coeffs(inp, sm)
    assert np.array_equal(bits(got), bits(want))


def test_assembly_batches_bitwise(cuda_ok, monkeypatch):
    """Theta-row batches (device output capped at 3 rows per batch here, so
    the C5-width grid runs in batches of 3, 3, 2 rows) give the reference's
    planes and max_speed bit for bit."""
    import oracle as O
    from paper_2010_04760_b200 import hwgpu
    ref = O.RefSolver(O.Physics(a=1.0, spin=-2, mmode=2), 65536, 8, workers=8)
    want, ms = ref.coeffs_all_dd()
    rho, cth = ref.grid_dd()
    monkeypatch.setenv("HWG_COEF_BATCH_BYTES", str(3 * 65536 * 14 * 16))
    got = hwgpu.assemble_coefficients(rho, cth, a=1.0, spin=-2, mmode=2, layout="dd")
    for q, name in enumerate(hwgpu.COEF_PLANES):
        assert np.array_equal(bits(got[name]), bits(want[q])), name
    assert np.array_equal(bits(got["max_speed"]), bits(ms))


def test_hyperbolicity_violation_reported_like_the_reference(cuda_ok):
    """geometry.cpp:146-149: disc2.hi < 0 -> runtime_error at the first such
    point of the (k, j) loop; the chart's rho in (-1, 0) is not hyperbolic."""
    import oracle as O
    from paper_2010_04760_b200 import hwgpu
    n, nt = 64, 4
    rho = np.zeros((n, 2))
    rho[:, 0] = np.linspace(-0.6, 5.0, n)
    cth = np.zeros((nt, 2))
    cth[:, 0] = np.cos((np.arange(nt) + 0.5) * np.pi / nt)
    # the first failing point in the reference's order, from its own kernel
    inp = np.zeros((n * nt, 5, 2))
    inp[:, 0] = np.tile(rho, (nt, 1))
    inp[:, 1] = np.repeat(cth, n, axis=0)
    inp[:, 2, 0], inp[:, 3, 0], inp[:, 4, 0] = 1.0, 0.9, 20.0
    sm = np.tile([[-2, 0]], (n * nt, 1))
    w = O.ref_wave_op_coeffs(inp, sm)
    P, R = w[:, 0, 0], w[:, 1, 0]
    first = int(np.argmax(P * P + 4 * R < 0))
    with pytest.raises(hwgpu.HwgError, match="hyperbolicity violated") as ei:
        hwgpu.assemble_coefficients(rho, cth, a=0.9, spin=-2, mmode=0)
    assert ei.value.bad_jk == (first % n, first // n)
