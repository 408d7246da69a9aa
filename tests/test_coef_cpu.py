"""CPU tests of the coefficient-assembly row: the
known-answer fixture pins the reference library's generated kernels (the
bitwise target of the GPU evaluator) against the reference's own 36-digit
values, and the library was built with the reference's generated kernels."""
import os
from fractions import Fraction

import numpy as np
import pytest

from conftest import GOLDEN

KAT = os.path.join(GOLDEN, "coef_kat.npz")


def dd_exact(p):
    return Fraction(float(p[0])) + Fraction(float(p[1]))


def test_kat_fixture_matches_36_digit_values():
    """proj/tests/test_geometry.cpp:119-139: |got - want| <= max(|want|, 1) * 1e-26."""
    z = np.load(KAT)
    host, want = z["host"], z["want"]
    assert host.shape == want.shape == (42, 11, 2)
    for i in range(host.shape[0]):
        for q in range(11):
            w = dd_exact(want[i, q])
            g = dd_exact(host[i, q])
            assert abs(g - w) <= max(abs(w), 1) * Fraction(1, 10**26), (i, q)


def test_kat_fixture_is_the_reference_library_output():
    import oracle as O
    if not O.ref_available():
        pytest.skip("reference library not built")
    z = np.load(KAT)
    out = O.ref_wave_op_coeffs(z["inp"], z["spin_mmode"])
    assert np.array_equal(out.view(np.int64), z["host"].view(np.int64))


def test_library_has_the_generated_kernels():
    from paper_2010_04760_b200 import hwgpu
    assert hwgpu._lib.hwg_have_coefficient_kernels() == 1


def test_generated_header_only_adds_device_annotations():
    """build.py's device copy of coeff_kernels.hpp (written to a temporary
    directory for the compile only) differs from the reference header only by
    the four __host__ __device__ annotations, and nothing reference-derived is
    left in the repository tree."""
    from paper_2010_04760_b200 import build as b
    inc = b.ref_include()
    if inc is None:
        pytest.skip("reference headers absent")
    gen = b.device_coeff_header_text(inc).split("\n", 1)[1]
    ref = open(os.path.join(inc, "hweno", "coeff_kernels.hpp")).read()
    assert gen.count("__host__ __device__ ") == 4
    assert gen.replace("__host__ __device__ ", "") == ref
    for dirpath, _, files in os.walk(os.path.dirname(b.PKG)):
        assert b.GEN_NAME not in files, dirpath


def test_assembly_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2010_04760_b200 import hwgpu
    with pytest.raises(hwgpu.HwgError):
        hwgpu.assemble_coefficients(np.zeros((16, 2)) + [[1.0, 0.0]], np.zeros((4, 2)), a=0.5)


def test_bench_grid_is_the_reference_grid_in_fp64():
    """planes.grid (the bench's fp64 grid for the device-assembled planes)
    is make_grid's DD grid (geometry.cpp:68-116) rounded: rho within a few
    ulps of the DD value's hi, the last point exactly S, cos(theta) within
    4e-16 of Grid::costh (the fp64 theta's rounding, absolute)."""
    import oracle as O
    if not O.ref_available():
        pytest.skip("reference library not built")
    from paper_2010_04760_b200 import planes
    for a, n, nt in ((1.0, 1024, 64), (0.9, 777, 33), (0.0, 256, 16)):
        ref = O.RefSolver(O.Physics(a=a, spin=-2, mmode=2), n, nt, workers=4)
        rho_dd, cth_dd = ref.grid_dd()
        rho, drho, dtheta, theta = planes.grid(n, nt, a=a)
        assert rho[-1] == 20.0 == rho_dd[-1, 0]
        assert np.max(np.abs(rho - rho_dd[:, 0]) / np.spacing(rho_dd[:, 0])) <= 8
        assert np.max(np.abs(np.cos(theta) - cth_dd[:, 0])) <= 4e-16
        assert abs(drho - ref.drho) <= 2 * np.spacing(ref.drho)


def test_assembly_binding_validates_arguments():
    """Argument errors surface before any device work (ValueError)."""
    from paper_2010_04760_b200 import hwgpu
    rho = np.zeros((16, 2)) + [[1.0, 0.0]]
    cth = np.zeros((4, 2))
    with pytest.raises(ValueError, match="unknown planes"):
        hwgpu.assemble_coefficients(rho, cth, planes=("b", "nope"))
    with pytest.raises(ValueError, match="layout"):
        hwgpu.assemble_coefficients(rho, cth, layout="csv")
