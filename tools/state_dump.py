"""Run K SSP-RK3 steps of a synthetic problem and save the final state
(for bitwise comparisons between builds: HWG_LIB=... python tools/state_dump.py out.npy)."""
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2010_04760_b200 import hwgpu, synthetic
    out = sys.argv[1]
    mode = sys.argv[2] if len(sys.argv) > 2 else "mixed"
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
    nt = int(sys.argv[4]) if len(sys.argv) > 4 else 128
    K = 20
    prob = synthetic.problem(n, nt)
    g = hwgpu.GpuEvolution(n, nt, prob["drho"], prob["dtheta"], prob["parity"], prob["coef"],
                           prob["cotth"], hwgpu.SchemeSpec("weno5", mode))
    g.set_state(synthetic.initial_state(prob))
    g.launch_steps("ssprk33", synthetic.select_dt(prob), 0, K)
    np.save(out, g.get_state())


if __name__ == "__main__":
    main()
