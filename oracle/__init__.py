"""TEST INFRASTRUCTURE ONLY — CPU checkers for the GPU hot path.

Two checkers, both loaded through ctypes:

* ``RefSolver`` drives the *unmodified* reference library (``_ref/libhweno_ref.so``,
  compiled in place from /root/reference/proj/src by ``oracle/Makefile``) —
  double-double state, the reference's own ``full``/``mixed`` modes.
* ``OracleSolver`` drives ``_build/libhweno_oracle.so``, the plain-C fp64/fp32
  restatement in ``hweno_oracle.c``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product package
(``paper_2010_04760_b200``) never does.

States use the reference FieldLayout (proj/include/hweno/evolve.hpp:23-35) as
numpy arrays of shape (4, ntheta + 4, nrho + 8): component, theta row (2
ghosts each side), rho column (4 ghosts each side).  DD states carry a
separate ``lo`` array of the same shape.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libhweno_ref.so")
ORC_SO = os.path.join(HERE, "_build", "libhweno_oracle.so")

RG, AG, NC = 4, 2, 4
SCHEMES = {"weno5": 0, "weno3": 1, "fd6ko": 2}
STEPPERS = {"ssprk33": 0, "ssprk104": 1}

_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_long)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


_ref = None
_orc = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_create.argtypes = [C.c_double, C.c_double, C.c_int, C.c_int, C.c_double,
                                   C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                   C.c_double, C.c_int, C.POINTER(C.c_void_p)]
        lib.ref_create_deeper.argtypes = [C.c_double, C.c_double, C.c_int, C.c_int, C.c_double,
                                          C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                          C.c_double, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        lib.ref_destroy.argtypes = [C.c_void_p]
        lib.ref_info.argtypes = [C.c_void_p, _dp, _dp, C.POINTER(C.c_longlong)]
        lib.ref_coeffs.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp]
        lib.ref_cotth_lo.argtypes = [C.c_void_p, _dp]
        lib.ref_grid_dd.argtypes = [C.c_void_p, _dp, _dp]
        lib.ref_coeffs_all_dd.argtypes = [C.c_void_p, _dp, _dp]
        lib.ref_wave_op_coeffs.argtypes = [C.c_int, _dp, C.POINTER(C.c_int), _dp]
        lib.ref_rat.argtypes = [C.c_longlong, C.c_longlong, _dp]
        lib.ref_initial_data.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double,
                                         C.c_double, _dp]
        lib.ref_rhs.argtypes = [C.c_void_p, _dp, _dp]
        lib.ref_apply_boundaries.argtypes = [C.c_void_p, _dp]
        lib.ref_select_dt.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp]
        lib.ref_advance.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, C.c_long, C.c_long,
                                    _dp, C.c_long, C.c_int, _dp, C.c_long, _lp, _dp]
        lib.ref_advance_timed.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, C.c_long,
                                          C.c_long, _dp, _dp, _lp]
        lib.ref_run_series.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_double,
                                       C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                       _dp, C.c_long, _lp, _dp]
        lib.ref_horizon_weights.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), _dp]
        lib.ref_projection_weights.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        lib.ref_multipole_project.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        lib.ref_weno5_row.argtypes = [_dp, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, _dp]
        lib.ref_weno5_weights.argtypes = [_dp, C.c_double, C.c_int, _dp]
        _ref = lib
    return _ref


def orc_lib():
    global _orc
    if _orc is None:
        lib = C.CDLL(ORC_SO)
        lib.orc_state_size.restype = C.c_size_t
        lib.orc_state_size.argtypes = [C.c_int, C.c_int]
        lib.orc_prepare.argtypes = [C.c_void_p]
        lib.orc_apply_boundaries.argtypes = [C.c_void_p, _dp]
        lib.orc_rhs.argtypes = [C.c_void_p, _dp, _dp]
        lib.orc_ssprk33_step.argtypes = [C.c_void_p, _dp, C.c_double]
        lib.orc_ssprk104_step.argtypes = [C.c_void_p, _dp, C.c_double]
        lib.orc_state_admissible.argtypes = [C.c_void_p, _dp, C.c_double]
        lib.orc_advance.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_long, C.c_long, _dp, _lp]
        lib.orc_weno5_weights_f64.argtypes = [_dp, C.c_double, _dp]
        lib.orc_weno5_weights_f32.argtypes = [_dp, C.c_float, C.POINTER(C.c_float)]
        lib.orc_weno5_interface.restype = C.c_double
        lib.orc_weno5_interface.argtypes = [_dp, C.c_int, C.c_double]
        lib.orc_weno5_row_derivative.argtypes = [_dp, C.c_int, C.c_double, C.c_int, C.c_double,
                                                 C.c_int, _dp]
        _orc = lib
    return _orc


class RefError(RuntimeError):
    pass


def _chk(rc: int):
    if rc != 0:
        msg = ref_lib().ref_last_error().decode()
        if rc == 2:
            raise ValueError(msg)
        raise RefError(msg)


@dataclass
class Physics:
    """PhysicalParams (proj/include/hweno/geometry.hpp:12-20) + InitialDataSpec."""
    M: float = 1.0
    a: float = 1.0
    spin: int = -2
    mmode: int = 0
    S: float = 20.0
    ell: int = 2
    center: float = 1.0
    width: float = 0.22
    amplitude: float = 1.0


# BASELINE.json configs, resolved per SURVEY.md D5/D6/D7 and §8(d).
CONFIGS = {
    "C1": dict(phys=Physics(a=0.0, spin=0, mmode=0, ell=2, center=3.0, width=0.3),
               nrho=1024, ntheta=64, mode="f64", stepper="ssprk33"),
    "C2": dict(phys=Physics(a=1.0, spin=-2, mmode=2, ell=2, center=1.0, width=0.22),
               nrho=4096, ntheta=128, mode="mixed", stepper="ssprk33"),
    "C3": dict(phys=Physics(a=0.9, spin=-2, mmode=0, ell=2, center=3.0, width=0.3),
               nrho=16384, ntheta=128, mode="mixed", stepper="ssprk33"),
    "C4": dict(phys=Physics(a=1.0, spin=-2, mmode=2, ell=2, center=1.0, width=0.22),
               nrho=4096, ntheta=128, mode="mixed", stepper="ssprk33", scheme="fd6ko"),
    "C5": dict(phys=Physics(a=1.0, spin=-2, mmode=2, ell=2, center=1.0, width=0.22),
               nrho=65536, ntheta=512, mode="mixed", stepper="ssprk33"),
}


class RefSolver:
    """The reference library: grid + coefficients + EvolutionRhs + advance_steps."""

    def __init__(self, phys: Physics, nrho: int, ntheta: int, scheme="weno5", mode="full",
                 eps=1e-6, sigma=0.01, workers=1, deeper=0):
        """deeper > 0: excision `deeper` cells below the default grid of
        nrho - deeper points, same spacing (test_evolve.cpp:397-410)."""
        lib = ref_lib()
        h = C.c_void_p()
        _chk(lib.ref_create_deeper(phys.M, phys.a, phys.spin, phys.mmode, phys.S, nrho, ntheta,
                                   SCHEMES[scheme], 0 if mode == "full" else 1, eps, sigma,
                                   workers, deeper, C.byref(h)))
        self.h = h
        self.phys, self.nrho, self.ntheta = phys, nrho, ntheta
        self.scheme, self.mode, self.eps, self.sigma = scheme, mode, eps, sigma
        d = np.zeros(6)
        dlo = np.zeros(6)
        ints = (C.c_longlong * 5)()
        _chk(lib.ref_info(h, _ptr(d), _ptr(dlo), ints))
        self.drho, self.dtheta, self.rho_min, self.max_speed, self.horizon_rho, _ = d
        self.drho_lo, self.dtheta_lo = dlo[0], dlo[1]
        self.parity = int(ints[2])
        self.horizon_index = int(ints[3])
        self.state_size = int(ints[4])
        P = nrho * ntheta
        self.coef = np.zeros(9 * P)
        self.coef_lo = np.zeros(9 * P)
        self.cotth = np.zeros(ntheta)
        self.rho = np.zeros(nrho)
        self.theta = np.zeros(ntheta)
        _chk(lib.ref_coeffs(h, _ptr(self.coef), _ptr(self.coef_lo), _ptr(self.cotth),
                            _ptr(self.rho), _ptr(self.theta)))
        self.cotth_lo = np.zeros(ntheta)
        _chk(lib.ref_cotth_lo(h, _ptr(self.cotth_lo)))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                ref_lib().ref_destroy(self.h)
        except Exception:
            pass

    @property
    def shape(self):
        return (NC, self.ntheta + 2 * AG, self.nrho + 2 * RG)

    def coef_planes(self):
        """(9, ntheta, nrho) view, plane order b, lam, w_re, w_im, bt_re, bt_im, c_re, c_im, ath."""
        return self.coef.reshape(9, self.ntheta, self.nrho)

    def grid_dd(self):
        """Grid::rho (nrho, 2) and Grid::costh (ntheta, 2) as DD {hi, lo} pairs."""
        rho = np.zeros(2 * self.nrho)
        cth = np.zeros(2 * self.ntheta)
        _chk(ref_lib().ref_grid_dd(self.h, _ptr(rho), _ptr(cth)))
        return rho.reshape(-1, 2), cth.reshape(-1, 2)

    def coeffs_all_dd(self):
        """All 14 CoefficientSet planes as (14, ntheta, nrho, 2) DD pairs, and max_speed (2,)."""
        P = self.nrho * self.ntheta
        planes = np.zeros(14 * P * 2)
        ms = np.zeros(2)
        _chk(ref_lib().ref_coeffs_all_dd(self.h, _ptr(planes), _ptr(ms)))
        return planes.reshape(14, self.ntheta, self.nrho, 2), ms

    def initial_data(self, phys: Physics | None = None):
        p = phys or self.phys
        dd = np.zeros(2 * self.state_size)
        _chk(ref_lib().ref_initial_data(self.h, p.ell, p.center, p.width, p.amplitude, _ptr(dd)))
        return split_dd(dd, self.shape)

    def rhs(self, hi, lo=None):
        """EvolutionRhs::operator(); returns (u_hi, u_lo) with ghosts filled and (du_hi, du_lo)."""
        dd = join_dd(hi, lo)
        du = np.zeros_like(dd)
        _chk(ref_lib().ref_rhs(self.h, _ptr(dd), _ptr(du)))
        return split_dd(dd, self.shape), split_dd(du, self.shape)

    def apply_boundaries(self, hi, lo=None):
        dd = join_dd(hi, lo)
        _chk(ref_lib().ref_apply_boundaries(self.h, _ptr(dd)))
        return split_dd(dd, self.shape)

    def select_dt(self, stepper="ssprk33", cfl=0.5):
        dt = np.zeros(2)
        _chk(ref_lib().ref_select_dt(self.h, STEPPERS[stepper], cfl, _ptr(dt)))
        return float(dt[0]), float(dt[1])

    def advance(self, hi, lo, dt, s0, s1, stepper="ssprk33", cfl=0.5, hook_every=0,
                ktheta=-1, max_obs=0):
        dd = join_dd(hi, lo)
        dtv = np.array([dt[0], dt[1]] if isinstance(dt, tuple) else [dt, 0.0])
        obs = np.zeros(max(1, 9 * max_obs))
        stats = (C.c_long * 4)()
        wall = C.c_double()
        _chk(ref_lib().ref_advance(self.h, STEPPERS[stepper], cfl, _ptr(dtv), s0, s1, _ptr(dd),
                                   hook_every, ktheta, _ptr(obs), max_obs, stats, C.byref(wall)))
        u = split_dd(dd, self.shape)
        st = dict(steps_done=stats[0], blew_up=bool(stats[1]), blowup_step=stats[2],
                  n_obs=stats[3], wall_seconds=wall.value)
        return u, st, obs[: 9 * stats[3]].reshape(-1, 9)

    def advance_timed(self, hi, lo, dt, s0, s1, stepper="ssprk33", cfl=0.5):
        """One advance_steps call over [s0, s1) with a timestamp hook:
        returns ((hi, lo), stats, per-step wall seconds (s1 - s0,))."""
        dd = join_dd(hi, lo)
        dtv = np.array([dt[0], dt[1]] if isinstance(dt, tuple) else [dt, 0.0])
        stamps = np.zeros(s1 - s0 + 1)
        stats = (C.c_long * 3)()
        _chk(ref_lib().ref_advance_timed(self.h, STEPPERS[stepper], cfl, _ptr(dtv), s0, s1,
                                         _ptr(dd), _ptr(stamps), stats))
        del hi, lo
        u = split_dd(dd, self.shape)
        st = dict(steps_done=stats[0], blew_up=bool(stats[1]), blowup_step=stats[2])
        return u, st, np.diff(stamps)

    def run_series(self, init: Physics, stepper="ssprk104", cfl=0.5, tau_end=500.0,
                   cadence=0.25, observer_rho=10.0, max_rows=200000):
        """execute_run's time loop + observer hook (driver.cpp:22-93): returns
        (rows (n, 15): tau, phi, dphi1..3, obs, proj, scri as re/im, stats)."""
        out = np.zeros(15 * max_rows)
        stats = (C.c_long * 5)()
        wall = C.c_double()
        _chk(ref_lib().ref_run_series(self.h, init.ell, init.center, init.width, init.amplitude,
                                      STEPPERS[stepper], cfl, tau_end, cadence, observer_rho,
                                      _ptr(out), max_rows, stats, C.byref(wall)))
        n = stats[3]
        return out[:15 * n].reshape(n, 15), dict(steps_done=stats[0], blew_up=bool(stats[1]),
                                                  blowup_step=stats[2], planned=stats[4],
                                                  wall_seconds=wall.value)

    def horizon_weights(self, ktheta):
        j0 = C.c_int()
        w = np.zeros(32)
        _chk(ref_lib().ref_horizon_weights(self.h, ktheta, C.byref(j0), _ptr(w)))
        return j0.value, w.reshape(4, 8)

    def projection_weights(self, ell=None):
        w = np.zeros(self.ntheta)
        _chk(ref_lib().ref_projection_weights(self.ntheta, self.phys.spin, self.phys.mmode,
                                              self.phys.ell if ell is None else ell, _ptr(w)))
        return w


def split_dd(dd: np.ndarray, shape):
    v = dd.reshape(-1, 2)
    return v[:, 0].reshape(shape).copy(), v[:, 1].reshape(shape).copy()


def join_dd(hi: np.ndarray, lo: np.ndarray | None = None) -> np.ndarray:
    out = np.zeros(hi.size * 2)
    out[0::2] = hi.ravel()
    if lo is not None:
        out[1::2] = lo.ravel()
    return out


def ref_weno5_row(u_hi, drho, eps, mode, minus):
    n = u_hi.size - 8
    dd = join_dd(np.ascontiguousarray(u_hi, dtype=np.float64))
    out = np.zeros(2 * n)
    _chk(ref_lib().ref_weno5_row(_ptr(dd), n, drho, eps, 0 if mode == "full" else 1,
                                 int(minus), _ptr(out)))
    return out[0::2].copy(), out[1::2].copy()


def ref_wave_op_coeffs(inp, spin_mmode):
    """wave_op_coeffs<DDReal> at n points: inp (n, 5, 2) DD {rho, cth, M, a, S},
    spin_mmode (n, 2) int -> (n, 11, 2) DD."""
    x = np.ascontiguousarray(inp, dtype=np.float64).reshape(-1)
    sm = np.ascontiguousarray(spin_mmode, dtype=np.int32).reshape(-1)
    n = sm.size // 2
    out = np.zeros(22 * n)
    _chk(ref_lib().ref_wave_op_coeffs(n, _ptr(x), sm.ctypes.data_as(C.POINTER(C.c_int)), _ptr(out)))
    return out.reshape(n, 11, 2)


def ref_rat(p: int, q: int) -> np.ndarray:
    """DDReal(p) / DDReal(q) as a (2,) {hi, lo} pair."""
    out = np.zeros(2)
    _chk(ref_lib().ref_rat(p, q, _ptr(out)))
    return out


def ref_weno5_weights(a5, eps, mode):
    a = np.ascontiguousarray(a5, dtype=np.float64)
    w = np.zeros(3)
    _chk(ref_lib().ref_weno5_weights(_ptr(a), eps, 0 if mode == "full" else 1, _ptr(w)))
    return w


class _OrcProblem(C.Structure):
    _fields_ = [("nrho", C.c_int), ("ntheta", C.c_int), ("drho", C.c_double),
                ("dtheta", C.c_double), ("parity", C.c_int), ("coef", _dp), ("cotth", _dp),
                ("scheme", C.c_int), ("mode", C.c_int), ("eps", C.c_double),
                ("sigma", C.c_double), ("split", C.POINTER(C.c_int))]


class OracleSolver:
    """The plain-C fp64 restatement (weights fp64 for mode 'f64', fp32 for 'mixed')."""

    def __init__(self, nrho, ntheta, drho, dtheta, parity, coef, cotth, scheme="weno5",
                 mode="f64", eps=1e-6, sigma=0.01):
        self.coef = np.ascontiguousarray(coef, dtype=np.float64).ravel()
        self.cotth = np.ascontiguousarray(cotth, dtype=np.float64)
        self.split = (C.c_int * ntheta)()
        self.nrho, self.ntheta = nrho, ntheta
        self.p = _OrcProblem(nrho, ntheta, drho, dtheta, parity, _ptr(self.coef),
                             _ptr(self.cotth), SCHEMES[scheme], 0 if mode == "f64" else 1,
                             eps, sigma, self.split)
        if orc_lib().orc_prepare(C.byref(self.p)) != 0:
            raise RuntimeError("EvolutionRhs: lam changes sign more than once along a row")

    @classmethod
    def from_ref(cls, ref: RefSolver, scheme=None, mode="f64", eps=None, sigma=None):
        return cls(ref.nrho, ref.ntheta, ref.drho, ref.dtheta, ref.parity, ref.coef, ref.cotth,
                   scheme or ref.scheme, mode, ref.eps if eps is None else eps,
                   ref.sigma if sigma is None else sigma)

    @property
    def shape(self):
        return (NC, self.ntheta + 2 * AG, self.nrho + 2 * RG)

    def rhs(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        du = np.zeros_like(u)
        orc_lib().orc_rhs(C.byref(self.p), _ptr(u), _ptr(du))
        return u, du

    def advance(self, u, dt, s0, s1, stepper="ssprk33"):
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        stats = (C.c_long * 3)()
        orc_lib().orc_advance(C.byref(self.p), STEPPERS[stepper], dt, s0, s1, _ptr(u), stats)
        return u, dict(steps_done=stats[0], blew_up=bool(stats[1]), blowup_step=stats[2])

    def admissible(self, u, limit=1e30):
        return bool(orc_lib().orc_state_admissible(C.byref(self.p), _ptr(np.ascontiguousarray(u)), limit))


def interior(u, nrho=None, ntheta=None):
    """Interior view (4, ntheta, nrho) of a reference-layout state."""
    return u[:, AG:-AG, RG:-RG]


def rel_linf(x, y):
    """Normwise relative L-inf over the interior."""
    xi, yi = interior(x), interior(y)
    return float(np.max(np.abs(xi - yi)) / max(np.max(np.abs(yi)), 1e-300))
