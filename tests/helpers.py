"""Shared helpers for the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

RG, AG = 4, 2


def interior(u):
    return u[:, AG:-AG, RG:-RG]


def rel_linf(x, y, comp=None):
    """Normwise relative L-inf over the interior: max|x-y| / max|y|."""
    xi, yi = interior(x), interior(y)
    if comp is not None:
        xi, yi = xi[comp], yi[comp]
    den = np.max(np.abs(yi))
    return float(np.max(np.abs(xi - yi)) / (den if den > 0 else 1.0))


def oracle_from_golden(g, mode="f64", eps=None):
    from oracle import OracleSolver
    return OracleSolver(int(g["nrho"]), int(g["ntheta"]), float(g["drho"]), float(g["dtheta"]),
                        int(g["parity"]), g["coef"], g["cotth"], str(g["scheme"]), mode,
                        float(g["eps"]) if eps is None else eps, float(g["sigma"]))


def gpu_from_golden(g, mode="f64", eps=None, scheme=None):
    from paper_2010_04760_b200.hwgpu import GpuEvolution, SchemeSpec
    spec = SchemeSpec(scheme or str(g["scheme"]), mode, float(g["eps"]) if eps is None else eps,
                      float(g["sigma"]))
    return GpuEvolution(int(g["nrho"]), int(g["ntheta"]), float(g["drho"]), float(g["dtheta"]),
                        int(g["parity"]), g["coef"], g["cotth"], spec)
