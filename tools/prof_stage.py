"""Small driver for ncu captures of the stage kernel at a BASELINE shape.

    python tools/prof_stage.py [--mode mixed|f64] [--nrho 65536] [--ntheta 512]
                               [--warmup 3] [--steps 1] [--scheme weno5]

Launches 3*(warmup+steps) stage kernels (SSP-RK3) on one handle; profile
with  -k regex:stage_kernel -s 3*warmup -c 3*steps.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="mixed")
    ap.add_argument("--scheme", default="weno5")
    ap.add_argument("--nrho", type=int, default=65536)
    ap.add_argument("--ntheta", type=int, default=512)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--stepper", default="ssprk33")
    a = ap.parse_args()
    import torch
    from paper_2010_04760_b200 import hwgpu, synthetic
    prob = synthetic.problem(a.nrho, a.ntheta)
    g = hwgpu.GpuEvolution(a.nrho, a.ntheta, prob["drho"], prob["dtheta"], prob["parity"],
                           prob["coef"], prob["cotth"], hwgpu.SchemeSpec(a.scheme, a.mode))
    g.set_state(synthetic.initial_state(prob))
    dt = synthetic.select_dt(prob, a.stepper)
    ns = 3 if a.stepper == "ssprk33" else 10
    g.launch_steps(a.stepper, dt, 0, a.warmup)
    g.synchronize()
    t0 = time.perf_counter()
    g.launch_steps(a.stepper, dt, a.warmup, a.steps)
    g.synchronize()
    wall = time.perf_counter() - t0
    P = a.nrho * a.ntheta
    bps = 157.33 if ns == 3 else 152.0
    rate = P * ns * a.steps / wall
    print(f"{a.mode} {a.scheme} {a.stepper} {a.nrho}x{a.ntheta}: {a.steps} steps {wall * 1e3:.3f} ms, "
          f"{rate:.3e} upd/s, {rate * bps / 1e9:.0f} GB/s algorithmic, launch {g.launch_info()}, "
          f"blew_up={g.status()}")


if __name__ == "__main__":
    main()
