"""ctypes binding of libhwgpu.so (include/hweno_gpu.h) and a thin Python
mirror of the reference's hot-path interface:

    GpuEvolution(...)            ~ hweno::EvolutionRhs   (proj/include/hweno/evolve.hpp:56-82)
    GpuEvolution.rhs(u)          ~ EvolutionRhs::operator()(u, du)
    GpuEvolution.advance(...)    ~ hweno::advance_steps  (proj/src/evolve.cpp:237-265)

States on the host use the reference FieldLayout as numpy arrays of shape
(4, ntheta + 4, nrho + 8) (component, theta row incl. 2 ghosts, rho column
incl. 4 ghosts).  There is no CPU fallback: importing this module without
the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from .build import SO

_SO = os.environ.get("HWG_LIB", SO)  # experiment override (alternative builds of the same source)
if not os.path.exists(_SO):
    raise ImportError(f"libhwgpu.so not built ({_SO}); run python -m paper_2010_04760_b200.build")

_lib = C.CDLL(_SO)
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p

SCHEMES = {"weno5": 0, "weno3": 1, "fd6ko": 2}
PRECISIONS = {"f64": 0, "mixed": 1, "dd-full": 2, "dd-mixed": 3}
STEPPERS = {"ssprk33": 0, "ssprk104": 1}
STAGES = {"ssprk33": 3, "ssprk104": 10}
HALO = 4


class HwgDesc(C.Structure):
    _fields_ = [("nrho", C.c_int), ("ntheta", C.c_int), ("drho", C.c_double),
                ("dtheta", C.c_double), ("parity", C.c_int), ("scheme", C.c_int),
                ("precision", C.c_int), ("eps", C.c_double), ("sigma", C.c_double),
                ("device", C.c_int), ("rho_offset", C.c_int), ("nrho_global", C.c_int),
                ("coef_ld", C.c_int), ("coef_row0", C.c_int), ("drho_lo", C.c_double),
                ("dtheta_lo", C.c_double), ("eps_lo", C.c_double), ("sigma_lo", C.c_double)]


class HwgRunStats(C.Structure):
    _fields_ = [("steps_done", C.c_longlong), ("wall_seconds", C.c_double),
                ("blew_up", C.c_int), ("blowup_step", C.c_longlong)]


class HwgObservables(C.Structure):
    _fields_ = [("phi", C.c_double * 2), ("dphi", (C.c_double * 2) * 3), ("obs", C.c_double * 2),
                ("scri", C.c_double * 2), ("proj", C.c_double * 2)]

    def as_dict(self):
        return dict(phi=complex(*self.phi), dphi=[complex(*d) for d in self.dphi],
                    obs=complex(*self.obs), scri=complex(*self.scri),
                    proj=complex(*self.proj))


HOOK = C.CFUNCTYPE(None, C.c_longlong, C.c_double, C.c_double, C.POINTER(HwgObservables), C.c_void_p)

_lib.hwg_last_error.restype = C.c_char_p
_lib.hwg_last_error.argtypes = [_vp]
_lib.hwg_create.argtypes = [C.POINTER(HwgDesc), _dp, _dp, C.POINTER(_vp)]
_lib.hwg_create_dd.argtypes = [C.POINTER(HwgDesc), _dp, _dp, _dp, _dp, C.POINTER(_vp)]
_lib.hwg_destroy.argtypes = [_vp]
_lib.hwg_set_stream.argtypes = [_vp, _vp, C.c_int]
for _f in ("hwg_set_state_dd", "hwg_get_state_dd", "hwg_set_state", "hwg_get_state"):
    getattr(_lib, _f).argtypes = [_vp, _dp]
_lib.hwg_rhs.argtypes = [_vp, _dp, _dp]
_lib.hwg_rhs_dd.argtypes = [_vp, _dp, _dp]
_lib.hwg_abort_advance.argtypes = [_vp]
_lib.hwg_launch_stage_rows.argtypes = [_vp, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_longlong, C.c_int, C.c_int, C.c_int]
_lib.hwg_advance.argtypes = [_vp, C.c_int, C.c_double, C.c_double, C.c_longlong, C.c_longlong,
                             C.c_longlong, HOOK, _vp, C.POINTER(HwgRunStats)]
_lib.hwg_set_observers.argtypes = [_vp, C.c_int, C.c_int, _dp, C.c_int, _dp]
_lib.hwg_observe.argtypes = [_vp, C.POINTER(HwgObservables)]
_lib.hwg_launch_stage.argtypes = [_vp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_longlong]
_lib.hwg_launch_steps.argtypes = [_vp, C.c_int, C.c_double, C.c_double, C.c_longlong, C.c_longlong]
_lib.hwg_stage_input.argtypes = [_vp, C.c_int, C.c_int, C.POINTER(C.c_int)]
_lib.hwg_register_ptr.argtypes = [_vp, C.c_int, C.POINTER(_vp), C.POINTER(C.c_longlong)]
_lib.hwg_current_register.argtypes = [_vp]
_lib.hwg_status.argtypes = [_vp, C.POINTER(C.c_int), C.POINTER(C.c_longlong), C.c_int]
_lib.hwg_launch_info.argtypes = [_vp] + [C.POINTER(C.c_int)] * 5
_lib.hwg_synchronize.argtypes = [_vp]


class HwgPeerDesc(C.Structure):
    """hwg_peer_desc (include/hweno_gpu.h)."""
    _fields_ = [("reg", _vp * 5), ("flag", _vp), ("nrho", C.c_longlong),
                ("row_elems", C.c_longlong), ("device", C.c_int), ("ipc", (C.c_ubyte * 64) * 6)]


_lib.hwg_peer_export.argtypes = [_vp, C.POINTER(HwgPeerDesc)]
_lib.hwg_set_peers.argtypes = [_vp, C.POINTER(HwgPeerDesc), C.POINTER(HwgPeerDesc), C.c_int,
                               C.c_double]
_lib.hwg_peer_prime.argtypes = [_vp]
_lib.hwg_selftest_division.argtypes = [C.c_longlong, C.c_ulonglong, C.POINTER(C.c_longlong),
                                       C.POINTER(C.c_longlong)]
_lib.hwg_peer_stats.argtypes = [_vp, C.POINTER(C.c_longlong)]
_lib.hwg_peer_emulate_steps.argtypes = [C.POINTER(_vp), C.c_int, C.c_int, C.c_double, C.c_double,
                                        C.c_longlong, C.c_longlong, C.c_longlong]

_dpp = C.POINTER(_dp)
_lib.hwg_assemble_coefficients.argtypes = [C.c_int, _dp, C.c_int, _dp, C.c_int, _dp, _dp, _dp,
                                           C.c_int, C.c_int, _dpp, _dp, C.POINTER(C.c_int)]
_lib.hwg_assemble_coefficients_split.argtypes = [C.c_int, _dp, C.c_int, _dp, C.c_int, _dp, _dp,
                                                 _dp, C.c_int, C.c_int, _dpp, _dpp, _dp,
                                                 C.POINTER(C.c_int)]
_lib.hwg_wave_op_coeffs.argtypes = [C.c_int, C.c_int, _dp, C.POINTER(C.c_int), _dp]
_lib.hwg_have_coefficient_kernels.argtypes = []

EXPORTED = ["hwg_create", "hwg_create_dd", "hwg_destroy", "hwg_last_error", "hwg_set_stream", "hwg_set_state_dd",
            "hwg_get_state_dd", "hwg_set_state", "hwg_get_state", "hwg_rhs", "hwg_rhs_dd",
            "hwg_advance", "hwg_set_observers", "hwg_observe", "hwg_launch_stage",
            "hwg_launch_steps", "hwg_stage_input", "hwg_register_ptr",
            "hwg_current_register", "hwg_status", "hwg_launch_info", "hwg_synchronize",
            "hwg_peer_export", "hwg_set_peers", "hwg_peer_prime", "hwg_abort_advance",
            "hwg_launch_stage_rows", "hwg_peer_stats", "hwg_peer_emulate_steps",
            "hwg_selftest_division", "hwg_assemble_coefficients",
            "hwg_assemble_coefficients_split", "hwg_wave_op_coeffs",
            "hwg_have_coefficient_kernels"]


class HwgError(RuntimeError):
    pass


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


# CoefficientSet planes in their order (proj/include/hweno/geometry.hpp:73-90)
COEF_PLANES = ("b", "lam", "w_re", "w_im", "bt_re", "bt_im", "c_re", "c_im", "ath", "p_mix",
               "r_rad", "br_re", "br_im", "bprime")


def _dd2(x) -> np.ndarray:
    """A DD scalar as a (2,) {hi, lo} array (a float is {x, 0})."""
    a = np.zeros(2)
    a[:] = x if np.ndim(x) else (float(x), 0.0)
    return a


def _coef_err(rc: int, bad=None):
    msg = _lib.hwg_last_error(None).decode()
    if rc == 2:
        raise ValueError(msg)
    err = HwgError(msg)
    err.bad_jk = None if bad is None else (bad[0], bad[1])
    raise err


def assemble_coefficients(rho_dd, costh_dd, M=1.0, a=0.0, S=20.0, spin=0, mmode=0,
                          planes=COEF_PLANES, layout="dd", device: int = 0, into=None):
    """assemble_coefficients (proj/src/geometry.cpp:118-168) on the GPU:
    rho_dd (nrho, 2) and costh_dd (ntheta, 2) DD grids (Grid::rho,
    Grid::costh), M / a / S floats or (hi, lo) pairs.
    layout 'dd'   -> {name: (ntheta, nrho, 2) DD pairs}  (CoefficientSet storage)
    layout 'split'-> {name: ((ntheta, nrho) hi, (ntheta, nrho) lo)}
    layout 'hi'   -> {name: (ntheta, nrho) hi}
    plus 'max_speed' -> (2,) DD.  layout 'hi' with `into` (len(planes),
    ntheta, nrho) C-contiguous fp64: written in place (no copies).  Raises
    HwgError (with .bad_jk) where the reference throws 'hyperbolicity
    violated'."""
    rho = np.ascontiguousarray(rho_dd, dtype=np.float64).reshape(-1, 2)
    cth = np.ascontiguousarray(costh_dd, dtype=np.float64).reshape(-1, 2)
    nrho, nt = rho.shape[0], cth.shape[0]
    want = set(planes)
    unknown = want - set(COEF_PLANES)
    if unknown:
        raise ValueError(f"unknown planes {sorted(unknown)}")
    ms = np.zeros(2)
    bad = (C.c_int * 2)()
    out, ptrs, lptrs = {}, (_dp * 14)(), (_dp * 14)()
    for q, name in enumerate(COEF_PLANES):
        if name not in want:
            continue
        if layout == "dd":
            out[name] = np.empty((nt, nrho, 2))
            ptrs[q] = _p(out[name])
        elif layout in ("split", "hi"):
            hi = np.empty((nt, nrho)) if into is None else into[list(planes).index(name)]
            assert hi.shape == (nt, nrho) and hi.dtype == np.float64 and hi.flags.c_contiguous
            ptrs[q] = _p(hi)
            if layout == "split":
                lo = np.empty((nt, nrho))
                lptrs[q] = _p(lo)
                out[name] = (hi, lo)
            else:
                out[name] = hi
        else:
            raise ValueError(f"layout {layout!r}")
    args = (device, _p(rho), nrho, _p(cth), nt, _p(_dd2(M)), _p(_dd2(a)), _p(_dd2(S)),
            int(spin), int(mmode))
    if layout == "dd":
        rc = _lib.hwg_assemble_coefficients(*args, ptrs, _p(ms), bad)
    else:
        rc = _lib.hwg_assemble_coefficients_split(*args, ptrs, lptrs, _p(ms), bad)
    if rc != 0:
        _coef_err(rc, bad)
    out["max_speed"] = ms
    return out


def wave_op_coeffs(inp, spin_mmode, device: int = 0) -> np.ndarray:
    """wave_op_coeffs<DDReal> (coeff_kernels.hpp:661-666) on the GPU at n
    points: inp (n, 5, 2) DD {rho, cth, M, a, S}, spin_mmode (n, 2) ->
    (n, 11, 2) DD {a_tr, a_rr, bt_re, bt_im, br_re, br_im, c_re, c_im, a_th,
    da_tr, da_rr}."""
    x = np.ascontiguousarray(inp, dtype=np.float64).reshape(-1)
    sm = np.ascontiguousarray(spin_mmode, dtype=np.int32).reshape(-1)
    n = sm.size // 2
    out = np.zeros((n, 11, 2))
    rc = _lib.hwg_wave_op_coeffs(device, n, _p(x), sm.ctypes.data_as(C.POINTER(C.c_int)), _p(out))
    if rc != 0:
        _coef_err(rc)
    return out


@dataclass
class SchemeSpec:
    """SchemeSpec (proj/include/hweno/evolve.hpp:37-42); mode is the GPU tier:
    'f64' (fp64 state + weights, ~ reference full), 'mixed' (fp64 state, fp32
    weights, ~ reference mixed) — one tier below the reference —
    or 'dd-full' / 'dd-mixed', the reference's own double-double precisions."""
    scheme: str = "weno5"
    mode: str = "mixed"
    eps: float = 1e-6
    sigma: float = 0.01


class _DevArray:
    """Zero-copy __cuda_array_interface__ view of a device pointer (for torch.as_tensor)."""

    def __init__(self, ptr: int, shape, typestr="<f8"):
        self.__cuda_array_interface__ = dict(shape=tuple(shape), typestr=typestr,
                                             data=(int(ptr), False), version=3, strides=None)


class GpuEvolution:
    """One handle = one GPU (or one radial slab of the grid)."""

    def __init__(self, nrho: int, ntheta: int, drho: float, dtheta: float, parity: int,
                 coef: np.ndarray, cotth: np.ndarray, spec: SchemeSpec = SchemeSpec(),
                 device: int = 0, rho_offset: int = 0, nrho_global: int | None = None,
                 coef_ld: int = 0, coef_row0: int = -1, coef_lo: np.ndarray | None = None,
                 cot_lo: np.ndarray | None = None, drho_lo: float = 0.0, dtheta_lo: float = 0.0,
                 eps_lo: float = 0.0, sigma_lo: float = 0.0):
        self._coef = np.ascontiguousarray(coef, dtype=np.float64).ravel()
        self._cot = np.ascontiguousarray(cotth, dtype=np.float64)
        d = HwgDesc(nrho, ntheta, drho, dtheta, parity, SCHEMES[spec.scheme],
                    PRECISIONS[spec.mode], spec.eps, spec.sigma, device, rho_offset,
                    nrho_global or nrho, coef_ld, coef_row0, drho_lo, dtheta_lo, eps_lo, sigma_lo)
        h = _vp()
        self.dd = spec.mode.startswith("dd")
        if self.dd:
            lo = np.zeros_like(self._coef) if coef_lo is None else np.ascontiguousarray(
                coef_lo, dtype=np.float64).ravel()
            clo = np.zeros_like(self._cot) if cot_lo is None else np.ascontiguousarray(
                cot_lo, dtype=np.float64)
            rc = _lib.hwg_create_dd(C.byref(d), _p(self._coef), _p(lo), _p(self._cot), _p(clo),
                                    C.byref(h))
        else:
            rc = _lib.hwg_create(C.byref(d), _p(self._coef), _p(self._cot), C.byref(h))
        if rc != 0:
            msg = _lib.hwg_last_error(None).decode()
            if rc == 2:
                raise ValueError(msg)
            raise HwgError(msg)
        self.h = h
        self._coef = None  # host copy no longer needed
        self.nrho, self.ntheta, self.spec, self.parity = nrho, ntheta, spec, parity
        self.drho, self.dtheta = drho, dtheta

    @classmethod
    def from_reference(cls, ref, spec: SchemeSpec | None = None, device: int = 0):
        """From a reference handle (oracle.RefSolver) — used by tests only.
        The DD tiers take the reference's low limbs too."""
        spec = spec or SchemeSpec(ref.scheme, "f64" if ref.mode == "full" else "mixed",
                                  ref.eps, ref.sigma)
        kw = {}
        if spec.mode.startswith("dd"):
            kw = dict(coef_lo=ref.coef_lo, cot_lo=ref.cotth_lo, drho_lo=ref.drho_lo,
                      dtheta_lo=ref.dtheta_lo)
        return cls(ref.nrho, ref.ntheta, ref.drho, ref.dtheta, ref.parity, ref.coef, ref.cotth,
                   spec, device, **kw)

    def close(self):
        if getattr(self, "h", None):
            _lib.hwg_destroy(self.h)
            self.h = None

    __del__ = close

    # ------------------------------------------------------------------ util
    def _chk(self, rc):
        if rc != 0:
            msg = _lib.hwg_last_error(self.h).decode()
            if rc == 2:
                raise ValueError(msg)
            raise HwgError(msg)

    @property
    def shape(self):
        return (4, self.ntheta + 4, self.nrho + 8)

    def set_stream(self, stream_ptr: int | None):
        """Launch on this cudaStream_t (0 = legacy default stream); None = own stream."""
        self._chk(_lib.hwg_set_stream(self.h, _vp(stream_ptr or 0), int(stream_ptr is None)))

    # ------------------------------------------------------------------ state
    def set_state(self, u: np.ndarray, lo: np.ndarray | None = None):
        if lo is not None:
            dd = np.empty(u.size * 2)
            dd[0::2] = u.ravel()
            dd[1::2] = lo.ravel()
            self._chk(_lib.hwg_set_state_dd(self.h, _p(dd)))
        else:
            self._chk(_lib.hwg_set_state(self.h, _p(np.ascontiguousarray(u, dtype=np.float64))))

    def get_state(self) -> np.ndarray:
        u = np.zeros(self.shape)
        self._chk(_lib.hwg_get_state(self.h, _p(u)))
        return u

    def get_state_dd(self):
        dd = np.zeros(2 * int(np.prod(self.shape)))
        self._chk(_lib.hwg_get_state_dd(self.h, _p(dd)))
        return dd[0::2].reshape(self.shape).copy(), dd[1::2].reshape(self.shape).copy()

    # ------------------------------------------------------------------ rhs
    def rhs(self, u: np.ndarray, du: np.ndarray | None = None):
        """EvolutionRhs::operator(): returns (u with ghosts filled, du)."""
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        du = np.zeros(self.shape) if du is None else np.ascontiguousarray(du).copy()
        self._chk(_lib.hwg_rhs(self.h, _p(u), _p(du)))
        return u, du

    def rhs_dd(self, hi: np.ndarray, lo: np.ndarray):
        """EvolutionRhs::operator() on a DDReal StateVec: ((u_hi, u_lo), (du_hi, du_lo))."""
        dd = np.empty(hi.size * 2)
        dd[0::2] = hi.ravel()
        dd[1::2] = lo.ravel()
        du = np.zeros_like(dd)
        self._chk(_lib.hwg_rhs_dd(self.h, _p(dd), _p(du)))
        sh = self.shape
        return ((dd[0::2].reshape(sh).copy(), dd[1::2].reshape(sh).copy()),
                (du[0::2].reshape(sh).copy(), du[1::2].reshape(sh).copy()))

    # ------------------------------------------------------------------ loop
    def advance(self, stepper: str, dt, step_begin: int, step_end: int, every: int = 1,
                hook=None):
        """advance_steps: hook(step, (tau_hi, tau_lo), observables dict)."""
        dt_hi, dt_lo = (dt if isinstance(dt, tuple) else (float(dt), 0.0))
        stats = HwgRunStats()
        errors = []

        def _cb(step, thi, tlo, obs, user):
            try:
                hook(int(step), (thi, tlo), obs.contents.as_dict())
            except Exception as e:  # noqa: BLE001 - re-raised below
                errors.append(e)
                _lib.hwg_abort_advance(self.h)  # leave advance_steps now, as the reference does

        cb = HOOK(_cb) if hook is not None else HOOK()
        self._chk(_lib.hwg_advance(self.h, STEPPERS[stepper], dt_hi, dt_lo, step_begin, step_end,
                                   every, cb, None, C.byref(stats)))
        if errors:
            raise errors[0]
        return dict(steps_done=stats.steps_done, wall_seconds=stats.wall_seconds,
                    blew_up=bool(stats.blew_up), blowup_step=stats.blowup_step)

    def set_observers(self, kobs: int, j0: int, hweights, jobs: int, pweights):
        hw = None if hweights is None else np.ascontiguousarray(hweights, dtype=np.float64).ravel()
        pw = None if pweights is None else np.ascontiguousarray(pweights, dtype=np.float64)
        self._chk(_lib.hwg_set_observers(self.h, kobs, j0, _p(hw) if hw is not None else None,
                                         jobs, _p(pw) if pw is not None else None))

    def observe(self) -> dict:
        o = HwgObservables()
        self._chk(_lib.hwg_observe(self.h, C.byref(o)))
        return o.as_dict()

    # ------------------------------------------------------------------ device level
    def launch_stage(self, stepper: str, stage: int, dt, step: int):
        dt_hi, dt_lo = (dt if isinstance(dt, tuple) else (float(dt), 0.0))
        self._chk(_lib.hwg_launch_stage(self.h, STEPPERS[stepper], stage, dt_hi, dt_lo, step))

    def launch_stage_rows(self, stepper: str, stage: int, dt, step: int, row_lo: int,
                          row_hi: int, first: bool, last: bool):
        """One part of a stage: rows [row_lo, row_hi) (hwg_launch_stage_rows)."""
        dt_hi, dt_lo = (dt if isinstance(dt, tuple) else (float(dt), 0.0))
        self._chk(_lib.hwg_launch_stage_rows(self.h, STEPPERS[stepper], stage, dt_hi, dt_lo, step,
                                             row_lo, row_hi, int(first) | 2 * int(last)))

    def launch_steps(self, stepper: str, dt, step_begin: int, nsteps: int):
        dt_hi, dt_lo = (dt if isinstance(dt, tuple) else (float(dt), 0.0))
        self._chk(_lib.hwg_launch_steps(self.h, STEPPERS[stepper], dt_hi, dt_lo, step_begin,
                                        nsteps))

    def stage_input(self, stepper: str, stage: int) -> int:
        r = C.c_int()
        self._chk(_lib.hwg_stage_input(self.h, STEPPERS[stepper], stage, C.byref(r)))
        return r.value

    def current_register(self) -> int:
        return _lib.hwg_current_register(self.h)

    def register_ptr(self, reg: int):
        """(row-0 device pointer, double2 per row) of a state register."""
        a, r = _vp(), C.c_longlong()
        self._chk(_lib.hwg_register_ptr(self.h, reg, C.byref(a), C.byref(r)))
        return a.value, r.value

    def register_view(self, reg: int):
        """torch view (nrho + 8 rows, row doubles) of a state register, halo rows
        included (row index 4 is grid row 0).  A row is contiguous: 32-column
        blocks [Psi(32) | pi(32)] of (re, im) pairs."""
        import torch
        ptr, row = self.register_ptr(reg)
        rows = self.nrho + 2 * HALO
        return torch.as_tensor(_DevArray(ptr - HALO * row * 16, (rows, 2 * row)), device="cuda")

    def status(self, clear: bool = False):
        b, s = C.c_int(), C.c_longlong()
        self._chk(_lib.hwg_status(self.h, C.byref(b), C.byref(s), int(clear)))
        return bool(b.value), s.value

    def launch_info(self):
        v = [C.c_int() for _ in range(5)]
        self._chk(_lib.hwg_launch_info(self.h, *[C.byref(x) for x in v]))
        return dict(zip(("blocks", "threads", "nranges", "nchunks", "pitch"), (x.value for x in v)))

    def synchronize(self):
        self._chk(_lib.hwg_synchronize(self.h))

    # ------------------------------------------------------- fused halo push
    def peer_export(self) -> bytes:
        """This slab's hwg_peer_desc (pointers + IPC handles) as bytes, to hand
        to the neighbours (in-process or over torch.distributed)."""
        d = HwgPeerDesc()
        self._chk(_lib.hwg_peer_export(self.h, C.byref(d)))
        return bytes(d)

    def set_peers(self, lower: bytes | None, upper: bytes | None, ipc: bool = False,
                  timeout_s: float = 10.0):
        """Connect the neighbour slabs: every later stage kernel pushes its
        boundary rows into their halos over peer memory (hwg_set_peers)."""
        def desc(b):
            return C.byref(HwgPeerDesc.from_buffer_copy(b)) if b is not None else None
        self._chk(_lib.hwg_set_peers(self.h, desc(lower), desc(upper), int(ipc), timeout_s))

    def peer_prime(self):
        self._chk(_lib.hwg_peer_prime(self.h))

    def peer_stats(self) -> int:
        """Boundary-warp waits that had to spin since hwg_set_peers."""
        v = C.c_longlong()
        self._chk(_lib.hwg_peer_stats(self.h, C.byref(v)))
        return v.value


def stage_bytes(stepper: str, mode: str = "mixed") -> float:
    """Algorithmic HBM bytes per grid point per stage: fp64
    state 32 B per register touched + 9 fp64 coefficient planes (72 B); the
    double-double tiers move twice that."""
    b = (136 + 168 + 168) / 3.0 if stepper == "ssprk33" else 1520 / 10.0
    return 2 * b if mode.startswith("dd") else b


def peer_emulate_steps(handles, stepper: str, dt, step_begin: int, nsteps: int,
                       skew_ns: int = 0):
    """hwg_peer_emulate_steps: peer-connected slab handles on one device run
    `nsteps` steps in ONE cooperative launch (validation of the fused halo
    push under genuine concurrency; include/hweno_gpu.h)."""
    dt_hi, dt_lo = (dt if isinstance(dt, tuple) else (float(dt), 0.0))
    arr = (_vp * len(handles))(*[h.h for h in handles])
    rc = _lib.hwg_peer_emulate_steps(arr, len(handles), STEPPERS[stepper], dt_hi, dt_lo,
                                     step_begin, nsteps, skew_ns)
    if rc != 0:
        handles[0]._chk(rc)


def selftest_division(n: int, seed: int = 1):
    """hwg_selftest_division: (mismatches, guard_fails) of the DD tiers'
    branch-free division against IEEE division on n random operand pairs."""
    m, f = C.c_longlong(), C.c_longlong()
    rc = _lib.hwg_selftest_division(n, seed, C.byref(m), C.byref(f))
    if rc != 0:
        raise HwgError(f"hwg_selftest_division failed ({rc})")
    return m.value, f.value
