"""Control for the sustained (power-capped) figure: a plain streaming kernel
with the stage kernel's read/write mix, run back to back for 1 s untimed and
3 s timed with nvidia-smi sampling (bench.ClockSampler), next to the C5
mixed-tier stage kernel under the same protocol (bench.sustained_mode).
If the plain stream holds its burst bandwidth at lower power, the stage
kernel's sustained gap is its own arithmetic's power, not HBM's.

    python tools/sustained_copy_probe.py > gpurun_out/sustained_copy_probe.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def stream(torch, clocks_cls, warm_s=1.0, timed_s=3.0):
    n = 1 << 27  # 1 GiB fp64 per array
    a, b = (torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(2))
    out = torch.empty_like(a)
    nbytes = 3 * n * 8  # 2 reads : 1 write (the stage kernel reads 3.2-4.25x what it writes)

    def step():
        torch.add(a, b, out=out)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        step()
    e1.record()
    torch.cuda.synchronize()
    burst = nbytes * 10 / (e0.elapsed_time(e1) / 1e3) / 1e9
    per = e0.elapsed_time(e1) / 10
    ck = clocks_cls(0)
    ck.start()
    t0 = time.time()
    while time.time() - t0 < warm_s:
        for _ in range(50):
            step()
        torch.cuda.synchronize()
    ck.mark()
    k = int(timed_s * 1e3 / per)
    e0.record()
    for _ in range(k):
        step()
    e1.record()
    torch.cuda.synchronize()
    ck.mark()
    ck.stop()
    sus = nbytes * k / (e0.elapsed_time(e1) / 1e3) / 1e9
    return {"kernel": "torch.add 2R:1W fp64, 3 GiB per launch", "burst_gbs": burst,
            "sustained_gbs": sus, "sustained_over_burst": sus / burst, "clocks": ck.summary()}


def main():
    import torch
    import bench
    from paper_2010_04760_b200 import hwgpu, planes, synthetic
    out = {"stream": stream(torch, bench.ClockSampler)}
    prob = planes.problem_or_synthetic(65536, 512)
    g = hwgpu.GpuEvolution(65536, 512, prob["drho"], prob["dtheta"], prob["parity"],
                           prob["coef"], prob["cotth"], hwgpu.SchemeSpec("weno5", "mixed"))
    g.set_state(synthetic.initial_state(prob))
    dt = synthetic.select_dt(prob)
    r = bench.sustained_mode(g, None, prob, dt, torch, bench.ClockSampler, 0,
                             warm_s=1.0, timed_s=3.0)
    gbs = r["value"] / 3 * 472 / 1e9  # 472 algorithmic bytes per point-step
    out["stage_kernel_c5_mixed"] = {"sustained_gbs": gbs, "value": r["value"],
                                    "clocks": r["clocks"]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
