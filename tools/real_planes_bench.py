"""The headline kernels on the reference's REAL C5 coefficient planes.

    python tools/real_planes_bench.py [--nrho 65536] [--ntheta 512] [--steps 50]

bench.py times the stage kernels on synthetic planes (paper_2010_04760_b200/
synthetic.py: the reference's grid, b <= 0, one lam sign change per row)
because its GPU arm may not execute the reference library.  This tool is
test infrastructure (it uses oracle/_ref): it builds the extremal-Kerr
s=-2 m=2 planes of BASELINE configs[4] with the unmodified
assemble_coefficients on host threads (hweno_gpu_setup.hpp: theta-row
sub-grids), times the same SSP-RK3 steps on them and on the synthetic
planes in one process, and prints one JSON line (profiles/<round>_real_planes.json).
The kernels have no data-dependent work apart from the pi orientation, so
the two rates should agree.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rate(g, dt, steps, torch):
    stream = torch.cuda.current_stream()
    g.set_stream(stream.cuda_stream)
    g.launch_steps("ssprk33", dt, 0, 5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g.launch_steps("ssprk33", dt, 5, steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    assert g.status() == (False, -1)
    return g.nrho * g.ntheta * 3 * steps / (ms / 1e3), ms / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nrho", type=int, default=65536)
    ap.add_argument("--ntheta", type=int, default=512)
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()
    import numpy as np
    import torch
    import oracle as O
    from paper_2010_04760_b200 import hwgpu, synthetic
    out = {"grid": f"{a.nrho}x{a.ntheta}", "steps": a.steps}
    workers = max(1, (os.cpu_count() or 2) - 1)
    t0 = time.perf_counter()
    ref = O.RefSolver(O.Physics(a=1.0, spin=-2, mmode=2, ell=2, center=1.0, width=0.22),
                      a.nrho, a.ntheta, mode="mixed", workers=workers)
    out["reference_setup_s"] = time.perf_counter() - t0
    out["setup_workers"] = workers
    u, _ = ref.initial_data()
    dt = ref.select_dt("ssprk33")
    for mode in ("mixed", "f64"):
        g = hwgpu.GpuEvolution.from_reference(ref, hwgpu.SchemeSpec("weno5", mode))
        g.set_state(u)
        v, ms = rate(g, dt, a.steps, torch)
        out[f"real_{mode}"] = {"value": v, "ms_per_step": ms}
        g.close()
    prob = synthetic.problem(a.nrho, a.ntheta)
    for mode in ("mixed", "f64"):
        g = hwgpu.GpuEvolution(a.nrho, a.ntheta, prob["drho"], prob["dtheta"], prob["parity"],
                               prob["coef"], prob["cotth"], hwgpu.SchemeSpec("weno5", mode))
        g.set_state(synthetic.initial_state(prob))
        v, ms = rate(g, synthetic.select_dt(prob), a.steps, torch)
        out[f"synthetic_{mode}"] = {"value": v, "ms_per_step": ms}
        g.close()
    out["real_over_synthetic_mixed"] = out["real_mixed"]["value"] / out["synthetic_mixed"]["value"]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
