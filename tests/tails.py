"""TEST INFRASTRUCTURE: restatement of the reference's late-time diagnostics
(proj/src/diagnostics.cpp:167-229) in fp64, applied identically to the
reference's and the GPU's observer series, plus a GPU driver that mirrors
execute_run's time loop and hook (proj/src/driver.cpp:22-93)."""
from __future__ import annotations

import numpy as np

# rows (n, 15): tau, phi, dphi1, dphi2, dphi3, obs, proj, scri as (re, im)
COL = dict(tau=0, phi=1, dphi1=3, dphi2=5, dphi3=7, obs=9, proj=11, scri=13)


def series(rows, name):
    c = COL[name]
    return rows[:, 0], rows[:, c] + 1j * rows[:, c + 1]


def local_power_index(tau, z):
    """local_power_index (diagnostics.cpp:167-195): p = tau d|f|/dtau / |f| by
    4th-order centred differences of the modulus; entries whose five-point
    window dips below 1e-25 of the peak are omitted."""
    amp = np.abs(z)
    n = amp.size
    out_t, out_p = [], []
    if n < 5 or amp.max() == 0.0:
        return np.array(out_t), np.array(out_p)
    thr = amp.max() * 1e-25
    for i in range(2, n - 2):
        if np.any(amp[i - 2:i + 3] < thr):
            continue
        h12 = (tau[i + 1] - tau[i - 1]) * 6.0
        da = (-amp[i + 2] + 8.0 * amp[i + 1] - 8.0 * amp[i - 1] + amp[i - 2]) / h12
        out_t.append(tau[i])
        out_p.append(tau[i] * da / amp[i])
    return np.array(out_t), np.array(out_p)


def window_mean(t, v, t0, t1):
    """window_mean_re (diagnostics.cpp:217-229)."""
    m = (t >= t0) & (t <= t1)
    return float(np.mean(v[m])) if m.any() else 0.0


def window_rel_drift(t, z, t0, t1):
    """window_rel_drift (diagnostics.hpp:125-128): (max - min) / |mean| of |z|."""
    m = (t >= t0) & (t <= t1)
    a = np.abs(z[m])
    if a.size == 0:
        return float("nan")
    return float((a.max() - a.min()) / abs(a.mean()))


def window_mean_abs_shift(t, v, shift, t0, t1):
    """artifacts::window_mean_abs_shift (proj/tests/support/artifacts.hpp:95-107):
    mean |v + shift| over the window; None where the reference throws (empty)."""
    m = (t >= t0) & (t <= t1)
    return float(np.mean(np.abs(v[m] + shift))) if m.any() else None


def p_phi_deviation(rows, window):
    """criterion 8's per-scheme figure (acceptance_tails.cpp:45-48): window mean
    of |p(Phi) + 1|."""
    tp, pp = local_power_index(*series(rows, "phi"))
    return window_mean_abs_shift(tp, pp, 1.0, *window)


def summary(rows, window):
    t0, t1 = window
    tau, phi = series(rows, "phi")
    _, dphi = series(rows, "dphi1")
    _, proj = series(rows, "proj")
    tp, pp = local_power_index(tau, phi)
    td, pd = local_power_index(tau, dphi)
    tq, pq = local_power_index(tau, proj)
    m = (tau >= t0) & (tau <= t1)
    return dict(p_phi=window_mean(tp, pp, t0, t1), p_dphi=window_mean(td, pd, t0, t1),
                p_proj=window_mean(tq, pq, t0, t1),
                charge=float(np.mean(np.abs(dphi[m]))) if m.any() else float("nan"),
                charge_drift=window_rel_drift(tau, dphi, t0, t1))


def gpu_run_series(ref, init, spec, stepper="ssprk104", cfl=0.5, tau_end=500.0, cadence=0.25,
                   observer_rho=10.0):
    """The GPU path driven like execute_run: reference setup (grid, coefficients,
    initial data, dt, observer weights), GPU time loop with device observers."""
    import math
    from paper_2010_04760_b200.hwgpu import GpuEvolution
    gpu = GpuEvolution.from_reference(ref, spec)
    u, lo = ref.initial_data(init)
    dt = ref.select_dt(stepper, cfl)
    steps = max(1, math.ceil(tau_end / dt[0] - 1e-9))           # steps_for, evolve.hpp:116-119
    stride = max(1, round(cadence / dt[0]))                      # sample_stride
    kobs = ref.ntheta // 2
    jobs = min(max(0, round((observer_rho - ref.rho_min) / ref.drho)), ref.nrho - 1)
    j0, hw = ref.horizon_weights(kobs)
    pw = ref.projection_weights(init.ell) if ref.phys.mmode == 0 else None
    gpu.set_observers(kobs, j0, hw, jobs, pw)
    gpu.set_state(u, lo if spec.mode.startswith("dd") else None)
    rows = []

    def hook(s, tau, ob):
        rows.append([tau[0], ob["phi"].real, ob["phi"].imag,
                     *[v for d in ob["dphi"] for v in (d.real, d.imag)],
                     ob["obs"].real, ob["obs"].imag, ob["proj"].real, ob["proj"].imag,
                     ob["scri"].real, ob["scri"].imag])

    st = gpu.advance(stepper, dt, 0, steps, every=stride, hook=hook)
    return np.array(rows), st
