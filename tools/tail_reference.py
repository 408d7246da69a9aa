"""Run the reference's production-style tail configs (proj/configs/*.ini)
through the unmodified reference library and store the observer series as
fixtures for the physics gate (tests/test_gpu_physics.py).

    python tools/tail_reference.py [name ...]   # writes tests/golden/tail_<name>.npz

TEST INFRASTRUCTURE (uses oracle/_ref).  Runs take 10-80 CPU-minutes.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import Physics, RefSolver  # noqa: E402

# proj/configs/tail_weno5_mixed.ini, price_schw.ini (τ, windows, observers as there)
RUNS = {
    "weno5_mixed": dict(phys=Physics(a=1.0, spin=-2, mmode=0, ell=2, center=1.0, width=0.22),
                        nrho=2048, ntheta=32, scheme="weno5", mode="mixed", stepper="ssprk104",
                        tau_end=500.0, window=(400.0, 500.0)),
    # criterion 8's comparison runs (tail_weno3_mixed.ini, tail_fd6ko_mixed.ini,
    # fd6ko_nodiss.ini): same physics/grid, other scheme / sigma
    "weno3_mixed": dict(phys=Physics(a=1.0, spin=-2, mmode=0, ell=2, center=1.0, width=0.22),
                        nrho=2048, ntheta=32, scheme="weno3", mode="mixed", stepper="ssprk104",
                        tau_end=500.0, window=(400.0, 500.0)),
    "fd6ko_mixed": dict(phys=Physics(a=1.0, spin=-2, mmode=0, ell=2, center=1.0, width=0.22),
                        nrho=2048, ntheta=32, scheme="fd6ko", mode="mixed", stepper="ssprk104",
                        tau_end=500.0, window=(400.0, 500.0), sigma=0.01),
    "fd6ko_nodiss": dict(phys=Physics(a=1.0, spin=-2, mmode=0, ell=2, center=1.0, width=0.22),
                         nrho=2048, ntheta=32, scheme="fd6ko", mode="mixed", stepper="ssprk104",
                         tau_end=200.0, window=(150.0, 200.0), sigma=0.0),
    "price_schw": dict(phys=Physics(a=0.0, spin=0, mmode=0, ell=2, center=3.0, width=0.3),
                       nrho=1024, ntheta=16, scheme="weno5", mode="mixed", stepper="ssprk104",
                       tau_end=800.0, window=(500.0, 750.0)),
    # BASELINE configs[2] physics (Kerr a = 0.9, s = -2, l = 2 pulse; SURVEY.md
    # D5/D7) at the desk scale D7 prescribes for the tail-exponent parity
    "kerr09_desk": dict(phys=Physics(a=0.9, spin=-2, mmode=0, ell=2, center=3.0, width=0.3),
                        nrho=2048, ntheta=32, scheme="weno5", mode="mixed", stepper="ssprk104",
                        tau_end=500.0, window=(300.0, 500.0)),
}


def run(name):
    c = RUNS[name]
    workers = os.cpu_count() or 8
    ref = RefSolver(c["phys"], c["nrho"], c["ntheta"], scheme=c["scheme"], mode=c["mode"],
                    sigma=c.get("sigma", 0.01), workers=workers)
    t0 = time.time()
    rows, st = ref.run_series(c["phys"], c["stepper"], tau_end=c["tau_end"])
    print(name, st, f"{time.time() - t0:.0f}s", flush=True)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"tail_{name}.npz"), rows=rows,
                        window=np.array(c["window"]), steps=st["steps_done"],
                        planned=st["planned"], wall=st["wall_seconds"], workers=workers,
                        blew_up=st["blew_up"], blowup_step=st["blowup_step"])


if __name__ == "__main__":
    for n in sys.argv[1:] or list(RUNS):
        run(n)
