"""HBM probe: achievable bandwidth of simple streaming kernels with the stage
kernel's read/write mix (stages 2-3 read 4.4x what they write), for context
next to MEASURED_PEAKS.json's copy figure."""
import torch

n = 1 << 27  # 1 GiB of fp64 per array
a, b, c, d, e = (torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(5))
out = torch.empty_like(a)


def bw(f, nbytes, reps=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        s.record(); f(); t.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(t))
    return nbytes / (best / 1e3) / 1e9


B = n * 8
print("copy 1R1W      GB/s %.0f" % bw(lambda: out.copy_(a), 2 * B))
print("add  2R1W      GB/s %.0f" % bw(lambda: torch.add(a, b, out=out), 3 * B))
print("sum4 4R1W      GB/s %.0f" % bw(lambda: torch.add(torch.add(a, b), torch.add(c, d), out=out), 7 * B))
print("read-only sum  GB/s %.0f" % bw(lambda: a.sum(), B))
