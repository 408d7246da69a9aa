"""BASELINE config 3 on the GPU (TEST/EVALUATION INFRASTRUCTURE, not collected
by pytest): Kerr a = 0.9M, s = -2, l = 2 pulse (center 3.0, width 0.3;
SURVEY.md D5/D7), WENO5, 16384 x 128, 10^6 SSP-RK3 steps, fp64 vs mixed.

The reference needs ~20 days for this on 8 cores, so parity is
stated the way D7 prescribes:
  1. full-resolution prefix: 10 steps of the reference (full, DD) vs the GPU
     dd-full tier (bitwise) and f64 tier (<= 1e-12);
  2. the full-length GPU runs (f64 and mixed) with device observers every
     tau = 0.25 (the driver's cadence), reporting the late-time power index
     of Phi at the horizon beside the desk-scale reference values.

    python tests/production_c3.py [--steps 1000000] > profiles/r01_c3_production.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1_000_000)
    ap.add_argument("--prefix", type=int, default=10)
    ap.add_argument("--tiers", default="f64,mixed")
    ap.add_argument("--save", default="")
    args = ap.parse_args()
    import oracle as O
    import tails
    from helpers import interior
    from paper_2010_04760_b200.hwgpu import GpuEvolution, SchemeSpec
    out = {"config": "C3: a=0.9, s=-2, m=0, l=2, center 3.0, width 0.3, 16384x128, WENO5, "
                     "SSP-RK3, cfl 0.5"}
    init = O.Physics(a=0.9, spin=-2, mmode=0, ell=2, center=3.0, width=0.3)
    t0 = time.time()
    ref = O.RefSolver(init, 16384, 128, scheme="weno5", mode="full", workers=os.cpu_count() or 8)
    out["reference_setup_s"] = time.time() - t0
    u, lo = ref.initial_data(init)
    dt = ref.select_dt("ssprk33")
    out["dt"] = dt
    # ---- 1. full-resolution prefix parity
    t0 = time.time()
    (rh, rl), rst, _ = ref.advance(u, lo, dt, 0, args.prefix)
    out["reference_prefix_s"] = time.time() - t0
    g = GpuEvolution.from_reference(ref, SchemeSpec("weno5", "dd-full"))
    g.set_state(u, lo)
    g.advance("ssprk33", dt, 0, args.prefix)
    gh, gl = g.get_state_dd()
    g.close()
    out["prefix_dd_full_bitwise"] = bool(
        np.array_equal(interior(gh).view(np.uint64), interior(rh).view(np.uint64)) and
        np.array_equal(interior(gl).view(np.uint64), interior(rl).view(np.uint64)))
    g = GpuEvolution.from_reference(ref, SchemeSpec("weno5", "f64"))
    g.set_state(u)
    g.advance("ssprk33", dt, 0, args.prefix)
    e = np.max(np.abs(interior(g.get_state()) - interior(rh))) / np.max(np.abs(interior(rh)))
    g.close()
    out["prefix_f64_rel_linf"] = float(e)
    # ---- 2. full-length GPU runs
    tau_end = args.steps * dt[0]
    runs = {}
    for tier in args.tiers.split(","):
        t0 = time.time()
        rows, st = tails.gpu_run_series(ref, init, SchemeSpec("weno5", tier), "ssprk33",
                                        tau_end=tau_end)
        wall = time.time() - t0
        w = (tau_end - 150.0, tau_end)
        s = tails.summary(rows, w)
        runs[tier] = rows
        late = {f"p_phi_{a:.0f}_{b:.0f}": tails.summary(rows, (a, b))["p_phi"]
                for a, b in ((100, 200), (200, 300), (300, 400), (400, 500), (500, tau_end))
                if b <= tau_end + 1e-9}
        out[tier] = dict(steps=st["steps_done"], blew_up=st["blew_up"], wall_s=wall, **late,
                         stage_updates_per_s=16384 * 128 * 3 * st["steps_done"] / st["wall_seconds"],
                         window=w, **s,
                         phi_final=float(abs(rows[-1, 1] + 1j * rows[-1, 2])))
    if args.save:
        np.savez_compressed(args.save, **{k.replace("-", "_"): v for k, v in runs.items()})
    names = list(runs)
    for i in range(len(names)):
        for j in range(i + 1, len(names)):
            a, b = runs[names[i]], runs[names[j]]
            n = min(len(a), len(b))
            pa = np.abs(a[:n, 1] + 1j * a[:n, 2])
            pb = np.abs(b[:n, 1] + 1j * b[:n, 2])
            rel = np.abs(pb - pa) / np.maximum(pa, 1e-300)
            # first tau where the two tiers' |Phi| differ by more than 1 %
            bad = np.nonzero(rel > 0.01)[0]
            out[f"{names[j]}_vs_{names[i]}"] = dict(
                phi_rel_diff_max=float(rel.max()),
                tau_first_1pct=float(a[bad[0], 0]) if bad.size else None)
    out["tau_end"] = tau_end
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
