"""PCIe probe: 1 GiB pinned host <-> device copies, each direction alone and both concurrently
(the ceiling of bench.py's e2e leg).  python tools/pcie_probe.py"""
import torch, time
n = 1 << 28
h = torch.empty(n, dtype=torch.int32).pin_memory()
h2 = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device="cuda")
d2 = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def h2d():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
def h2d_split(k=4):
    c = n // k
    ss = [torch.cuda.Stream() for _ in range(k)]
    for i in range(k):
        with torch.cuda.stream(ss[i]): d[i*c:(i+1)*c].copy_(h[i*c:(i+1)*c], non_blocking=True)
GB = 4 * n / 1e9
for name, f in [("h2d", h2d), ("d2h", d2h), ("both", both), ("h2d split4", h2d_split)]:
    x = t(f)
    print(f"{name}: {x*1e3:.2f} ms  {GB/x:.1f} GB/s per direction")
