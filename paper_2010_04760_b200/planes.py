"""Coefficient planes of the reference's own physics for throughput runs,
assembled on the GPU.

The grid follows make_grid (proj/src/geometry.cpp:68-116): rho uniform on
[rho_+ - 1/20, S] with the last point exactly S, theta staggered at
(k + 1/2) pi / Ntheta.  Here the grid is formed in fp64 (the reference forms
it in double-double and takes cos theta from its DD sin_cos); the planes are
then the reference's assemble_coefficients (geometry.cpp:118-168) evaluated
by hwg_assemble_coefficients — the reference's generated wave_op_coeffs
kernels in double-double on the device — at those grid points.  The parity
tests (tests/test_gpu_coef.py) feed the reference's own DD grid and get its
planes bit for bit; for a benchmark the fp64 grid is the same physics.

problem() returns the dict synthetic.problem() returns (the bench and tools
take either), for the rows [rho_offset, rho_offset + nrho) of a grid of
nrho_global rows.
"""
from __future__ import annotations

import math

import numpy as np


def horizon_rho(M: float, a: float, S: float) -> float:
    """compactify(r_+) (geometry.hpp: horizon_radius, horizon_rho)."""
    rp = M + math.sqrt(max(M * M - a * a, 0.0))
    return rp / (1.0 + rp / S)


def grid(nrho_global: int, ntheta: int, M=1.0, a=1.0, S=20.0):
    rho_min = horizon_rho(M, a, S) - 1.0 / 20.0
    drho = (S - rho_min) / (nrho_global - 1)
    rho = rho_min + drho * np.arange(nrho_global, dtype=np.float64)
    rho[-1] = S  # exact scri point
    dtheta = math.pi / ntheta
    theta = dtheta * (np.arange(ntheta) + 0.5)
    return rho, drho, dtheta, theta


def available() -> bool:
    """The library carries the reference's generated coefficient kernels
    (built with the reference headers; hwg_have_coefficient_kernels)."""
    from . import hwgpu
    return bool(hwgpu._lib.hwg_have_coefficient_kernels())


def problem_or_synthetic(nrho: int, ntheta: int, rho_offset: int = 0,
                         nrho_global: int | None = None, **phys):
    """problem() where the library has the coefficient kernels, else the
    synthetic planes of the same shape (synthetic.problem) — benchmark input
    data only; the dict's 'planes' key says which."""
    if available():
        p = problem(nrho, ntheta, rho_offset=rho_offset, nrho_global=nrho_global, **phys)
        p["planes"] = "device-assembled"
        return p
    from . import synthetic
    p = synthetic.problem(nrho, ntheta, rho_offset=rho_offset, nrho_global=nrho_global,
                          **{k: v for k, v in phys.items() if k in ("a", "spin", "mmode", "S")})
    p["planes"] = "synthetic"
    return p


def problem(nrho: int, ntheta: int, rho_offset: int = 0, nrho_global: int | None = None,
            M: float = 1.0, a: float = 1.0, spin: int = -2, mmode: int = 2, S: float = 20.0,
            device: int = 0):
    """Planes (9, ntheta, nrho) of rows [rho_offset, rho_offset + nrho): the
    extremal-Kerr s = -2, m = 2 physics of BASELINE configs[1] / [4] by
    default.  max_speed is this slab's (the whole grid's on one GPU)."""
    from . import hwgpu

    ng = nrho_global or nrho
    rho, drho, dtheta, theta = grid(ng, ntheta, M=M, a=a, S=S)
    rho = rho[rho_offset:rho_offset + nrho]
    rho_dd = np.stack([rho, np.zeros_like(rho)], axis=1)
    cth = np.cos(theta)
    cth_dd = np.stack([cth, np.zeros_like(cth)], axis=1)
    coef = np.empty((9, ntheta, nrho))
    out = hwgpu.assemble_coefficients(rho_dd, cth_dd, M=M, a=a, S=S, spin=spin, mmode=mmode,
                                      planes=hwgpu.COEF_PLANES[:9], layout="hi", device=device,
                                      into=coef)
    cotth = np.cos(theta) / np.sin(theta)
    parity = 1 if (mmode + spin) % 2 == 0 else -1
    return dict(coef=coef, cotth=cotth, drho=drho, dtheta=dtheta, parity=parity, rho=rho,
                theta=theta, nrho=nrho, ntheta=ntheta, nrho_global=ng, rho_offset=rho_offset,
                max_speed=float(out["max_speed"][0]),
                physics=dict(M=M, a=a, spin=spin, mmode=mmode, S=S))
