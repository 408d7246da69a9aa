"""Sustained-load A/B of library builds (HWG_LIB): for each build, the C5
mixed tier is stepped back to back for `warm` seconds, then timed for
`timed` seconds with CUDA events while nvidia-smi samples the SM clock.

    python tools/sustained_ab.py libhwgpu.so libhwgpu_x.so [--rounds 2]

Each build runs in a fresh subprocess (one library per process)."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(warm, timed, mode):
    sys.path.insert(0, ROOT)
    import torch
    import bench
    from paper_2010_04760_b200 import hwgpu, synthetic
    prob = synthetic.problem(65536, 512)
    g = hwgpu.GpuEvolution(65536, 512, prob["drho"], prob["dtheta"], prob["parity"],
                           prob["coef"], prob["cotth"], hwgpu.SchemeSpec("weno5", mode))
    g.set_state(synthetic.initial_state(prob))
    r = bench.sustained_mode(g, None, prob, synthetic.select_dt(prob), torch, bench.ClockSampler,
                             0, warm_s=warm, timed_s=timed)
    print(json.dumps({"value": r["value"], "ms_per_step": r["ms_per_step"],
                      "sm_mhz": r["clocks"]["sm_mhz"], "power_w": r["clocks"].get("power_w_median")}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="*")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--warm", type=float, default=1.0)
    ap.add_argument("--timed", type=float, default=3.0)
    ap.add_argument("--mode", default="mixed")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        return child(a.warm, a.timed, a.mode)
    for r in range(a.rounds):
        for lib in a.libs:
            env = dict(os.environ, HWG_LIB=os.path.join(ROOT, "paper_2010_04760_b200", lib))
            out = subprocess.run([sys.executable, __file__, "--child", "--warm", str(a.warm),
                                  "--timed", str(a.timed), "--mode", a.mode],
                                 capture_output=True, text=True, env=env, timeout=600)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            print(f"r{r} {lib} {line}", flush=True)


if __name__ == "__main__":
    main()
