import torch, time
n = 1082262528 // 8
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True); h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device='cuda'); d2 = torch.empty(n, dtype=torch.float64, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d1.copy_(h1, non_blocking=True); h2.copy_(d2, non_blocking=True); torch.cuda.synchronize()
def t(f):
    torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter() - a
gb = n * 8 / 1e9
print('h2d alone GB/s', gb / t(lambda: d1.copy_(h1, non_blocking=True)))
print('d2h alone GB/s', gb / t(lambda: h2.copy_(d2, non_blocking=True)))
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print('both, per direction GB/s', gb / t(both))
