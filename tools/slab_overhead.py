"""Cost of the multi-GPU slab machinery, measured on ONE GPU.

    python tools/slab_overhead.py [--mode mixed] [--nrho 65536] [--ntheta 512]
                                  [--slabs 2] [--steps 30] [--warmup 3]

Times K SSP-RK3 steps of one nrho x ntheta grid three ways on the same
device, one stream, CUDA events:
  whole   one handle (graph-replayed steps, the bench's single-GPU path);
  peer    the grid cut into S radial slabs with the fused halo push
          (slabs.LocalPeerSlabs: every slab's boundary warps wait for and push
          halo rows, signal counters, take launch tickets), slab by slab and
          stage by stage on one stream, so every wait is already satisfied;
  nccl    the same slabs with DistSlab's overlapped sequence per stage
          (interior rows, halo copy, boundary strips; slabs.LocalSlabs with
          overlap=True, the copies device-local instead of NCCL).
The slab rows add up to the whole grid, so (peer - whole) / whole is the work
the slab protocol adds to one GPU's stage time: the per-slab cost that weak
scaling pays on top of the NVLink transfer latency, which this single-GPU
setup cannot measure.  Prints one JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="mixed")
    ap.add_argument("--nrho", type=int, default=65536)
    ap.add_argument("--ntheta", type=int, default=512)
    ap.add_argument("--slabs", type=int, default=2)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    import torch
    from paper_2010_04760_b200 import hwgpu, slabs, synthetic

    n, nt = a.nrho, a.ntheta
    spec = hwgpu.SchemeSpec("weno5", a.mode)
    full = synthetic.problem(n, nt)
    dt = synthetic.select_dt(full, "ssprk33")
    u0 = synthetic.initial_state(full)
    stream = torch.cuda.Stream()

    def timed(run, stream=stream):
        with torch.cuda.stream(stream):
            run(0, a.warmup)
            stream.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run(a.warmup, a.steps)
            e1.record(stream)
            stream.synchronize()
        return e0.elapsed_time(e1) / a.steps

    out = {"grid": f"{n}x{nt}", "mode": a.mode, "slabs": a.slabs, "steps": a.steps}
    g = hwgpu.GpuEvolution(n, nt, full["drho"], full["dtheta"], full["parity"], full["coef"],
                           full["cotth"], spec, coef_ld=n, coef_row0=0)
    g.set_stream(stream.cuda_stream)
    g.set_state(u0)
    out["whole_ms_per_step"] = timed(lambda s0, k: g.launch_steps("ssprk33", dt, s0, k))
    g.close()

    def make_slabs():
        hs = []
        for off, cnt in slabs.partition(n, a.slabs):
            p = synthetic.problem(cnt, nt, rho_offset=off, nrho_global=n)
            h = hwgpu.GpuEvolution(cnt, nt, p["drho"], p["dtheta"], p["parity"], p["coef"],
                                   p["cotth"], spec, rho_offset=off, nrho_global=n,
                                   coef_ld=cnt, coef_row0=0)
            u = synthetic.initial_state(p)
            h.set_state(u)
            hs.append(h)
        return hs

    hs = make_slabs()
    ps = slabs.LocalPeerSlabs(hs, timeout_s=10.0)
    ps.prime()
    out["peer_ms_per_step"] = timed(lambda s0, k: ps.steps("ssprk33", dt, s0, k), ps.stream)
    assert all(h.status() == (False, -1) for h in hs), [h.status() for h in hs]
    for h in hs:
        h.close()

    hs = make_slabs()
    for h in hs:
        h.set_stream(stream.cuda_stream)
    ls = slabs.LocalSlabs(hs, overlap=True)
    out["nccl_seq_ms_per_step"] = timed(lambda s0, k: ls.steps("ssprk33", dt, s0, k))
    for h in hs:
        h.close()

    w = out["whole_ms_per_step"]
    out["peer_overhead"] = out["peer_ms_per_step"] / w - 1.0
    out["nccl_seq_overhead"] = out["nccl_seq_ms_per_step"] / w - 1.0
    print(json.dumps(out))


if __name__ == "__main__":
    main()
