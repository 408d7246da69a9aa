"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference
library (oracle/_ref/libhweno_ref.so, compiled in place from
/root/reference/proj/src).  Run in the build container:

    python tests/golden/make_golden.py [--big] [--c2]

Small cases (npz, a few tens of KB each) pin one RHS evaluation and a short
evolution in both reference modes (DD "full" and DD+fp64-weight "mixed") for
every scheme / orientation / parity situation the hot path has.  --big adds
the BASELINE gate runs: config C1 (1024x64, 1000 SSP-RK3 steps, reference
full) and the desk-scale C2 physics (1024x32, 1000 steps, reference mixed).
The fixtures hold the DD .hi limbs.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Physics, RefSolver  # noqa: E402

# (name, physics, nrho, ntheta, scheme, eps, init, steps, stepper)
SMALL = [
    ("extremal_w5", Physics(a=1.0, spin=-2, mmode=0), 64, 8, "weno5", 1e-6,
     dict(ell=2, center=10.0, width=1.0), 40, "ssprk33"),
    ("extremal_m2_w5", Physics(a=1.0, spin=-2, mmode=2), 64, 8, "weno5", 1e-6,
     dict(ell=2, center=3.0, width=0.6), 40, "ssprk33"),
    ("kerr09_w5", Physics(a=0.9, spin=-2, mmode=0), 96, 8, "weno5", 1e-6,
     dict(ell=2, center=3.0, width=0.3), 40, "ssprk33"),
    ("schw_w5", Physics(a=0.0, spin=0, mmode=0), 64, 8, "weno5", 1e-6,
     dict(ell=2, center=3.0, width=0.3), 40, "ssprk33"),
    ("oddpar_w5", Physics(a=0.5, spin=1, mmode=0), 64, 6, "weno5", 1e-6,
     dict(ell=2, center=4.0, width=0.5), 40, "ssprk33"),
    ("kerr09_w5_rk104", Physics(a=0.9, spin=-2, mmode=0), 96, 8, "weno5", 1e-6,
     dict(ell=2, center=3.0, width=0.3), 8, "ssprk104"),
    ("extremal_fd6ko", Physics(a=1.0, spin=-2, mmode=0), 64, 8, "fd6ko", 1e-6,
     dict(ell=2, center=10.0, width=1.0), 40, "ssprk33"),
    ("extremal_w3", Physics(a=1.0, spin=-2, mmode=0), 64, 8, "weno3", 1e-6,
     dict(ell=2, center=10.0, width=1.0), 40, "ssprk33"),
    ("extremal_w5_theta34", Physics(a=1.0, spin=-2, mmode=0), 160, 34, "weno5", 1e-6,
     dict(ell=2, center=8.0, width=1.0), 10, "ssprk33"),
    # one column in the last theta chunk (its south-pole images live in the previous chunk)
    ("oddpar_w5_theta33", Physics(a=0.5, spin=1, mmode=0), 96, 33, "weno5", 1e-6,
     dict(ell=2, center=6.0, width=1.0), 4, "ssprk33"),
]


def _case(name, phys, nrho, ntheta, scheme, eps, init, steps, stepper):
    out = {}
    full = RefSolver(phys, nrho, ntheta, scheme=scheme, mode="full", eps=eps)
    mixed = RefSolver(phys, nrho, ntheta, scheme=scheme, mode="mixed", eps=eps)
    ip = Physics(**{**phys.__dict__, **init})
    u, ulo = full.initial_data(ip)
    rng = np.random.default_rng(1234)
    urand = np.zeros(full.shape)
    urand[:, 2:-2, 4:-4] = rng.uniform(-1.0, 1.0, size=(4, ntheta, nrho))
    for tag, ref in (("full", full), ("mixed", mixed)):
        (_, _), (du, _) = ref.rhs(u, ulo)
        out[f"rhs_{tag}"] = du
        (_, _), (dr, _) = ref.rhs(urand)
        out[f"rhs_rand_{tag}"] = dr
        dt = ref.select_dt(stepper)
        (uf, _), st, _ = ref.advance(u, ulo, dt, 0, steps, stepper=stepper)
        assert not st["blew_up"], (name, tag)
        out[f"state_{tag}"] = uf
    # frozen linear weights (eps = inf): the reconstruction is a linear operator
    lin = RefSolver(phys, nrho, ntheta, scheme=scheme, mode="full", eps=float("inf"))
    (_, _), (dl, _) = lin.rhs(urand)
    out["rhs_rand_linear"] = dl
    dt = full.select_dt(stepper)
    out.update(coef=full.coef, cotth=full.cotth, rho=full.rho, u0=u, urand=urand,
               dt=np.array(dt), drho=full.drho, dtheta=full.dtheta, parity=full.parity,
               nrho=nrho, ntheta=ntheta, steps=steps, scheme=scheme, stepper=stepper, eps=eps,
               sigma=full.sigma, max_speed=full.max_speed, spin=phys.spin, mmode=phys.mmode,
               a=phys.a)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def _big(name, phys, nrho, ntheta, mode, steps, workers):
    ref = RefSolver(phys, nrho, ntheta, scheme="weno5", mode=mode, workers=workers)
    u, ulo = ref.initial_data()
    dt = ref.select_dt("ssprk33")
    t0 = time.time()
    (uf, _), st, _ = ref.advance(u, ulo, dt, 0, steps)
    print(name, st, f"{time.time() - t0:.1f}s")
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), state=uf[:, 2:-2, 4:-4],
                        dt=np.array(dt), drho=ref.drho, steps=steps, mode=mode,
                        nrho=nrho, ntheta=ntheta)


def _c2(workers, steps=1000, every=10):
    """BASELINE configs[1] at its stated physics and size: extremal Kerr a=1,
    s=-2, m=2, 4096x128, reference mixed, SSP-RK3.  Stores the final interior
    .hi state, SHA-256 digests of the final DD state (hi and lo limbs, for
    the bitwise dd-mixed check) and the reference HorizonSampler series at
    k = Ntheta/2 every `every` steps (diagnostics.cpp:145-165; the Aretakis
    charge is dphi[0], :162-165)."""
    import hashlib
    phys = Physics(a=1.0, spin=-2, mmode=2, ell=2, center=1.0, width=0.22)
    ref = RefSolver(phys, 4096, 128, scheme="weno5", mode="mixed", workers=workers)
    u, ulo = ref.initial_data()
    dt = ref.select_dt("ssprk33")
    t0 = time.time()
    (uf, ufl), st, obs = ref.advance(u, ulo, dt, 0, steps, hook_every=every, ktheta=64,
                                     max_obs=steps // every + 2)
    print("c2_mixed_1000", st, f"{time.time() - t0:.1f}s", flush=True)
    hi = np.ascontiguousarray(uf[:, 2:-2, 4:-4])
    lo = np.ascontiguousarray(ufl[:, 2:-2, 4:-4])
    np.savez_compressed(os.path.join(HERE, "c2_mixed_1000.npz"), state=hi,
                        sha_hi=np.frombuffer(hashlib.sha256(hi.tobytes()).digest(), np.uint8),
                        sha_lo=np.frombuffer(hashlib.sha256(lo.tobytes()).digest(), np.uint8),
                        horizon=obs, every=every, ktheta=64, dt=np.array(dt), drho=ref.drho,
                        steps=steps, mode="mixed", nrho=4096, ntheta=128,
                        wall=st["wall_seconds"], workers=workers)


def main():
    only = [a for a in sys.argv[1:] if not a.startswith("--")]
    for c in SMALL:
        if only and c[0] not in only:
            continue
        _case(*c)
        print("wrote", c[0])
    if "--big" in sys.argv:
        workers = os.cpu_count() or 8
        _big("c1_full_1000", Physics(a=0.0, spin=0, mmode=0, ell=2, center=3.0, width=0.3),
             1024, 64, "full", 1000, workers)
        _big("c2desk_mixed_1000", Physics(a=1.0, spin=-2, mmode=2, ell=2, center=1.0,
                                          width=0.22), 1024, 32, "mixed", 1000, workers)


    if "--c2" in sys.argv:
        _c2(os.cpu_count() or 8)


if __name__ == "__main__":
    main()
