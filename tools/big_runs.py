"""Two-run path at sizes beyond 2^31 bytes of keys (64-bit index arithmetic): 2^31 int32 organ pipe and
ascending + random tail, 2^29 (int64, uint32) pairs with a sorted prefix; checked on the device.
  python tools/big_runs.py"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2106_05123_b200 import DeviceSorter  # noqa: E402

g = torch.Generator(device="cuda")
g.manual_seed(4)


def timed(ds, x, v=None):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ds.run(x, v)
    b.record()
    st = ds.finish()
    return a.elapsed_time(b), st


n = 1 << 31
h = n // 2
x = torch.empty(n, dtype=torch.int32, device="cuda")
x[:h] = torch.arange(h, dtype=torch.int32, device="cuda")
x[h:] = torch.arange(h - 1, -1, -1, dtype=torch.int32, device="cuda")
total = int(x.to(torch.int64).sum().item()) if False else None
ds = DeviceSorter(n, torch.int32, False)
ms, st = timed(ds, x)
ok = bool((x[1:] >= x[:-1]).all().item()) and int(x[0]) == 0 and int(x[-1]) == h - 1 and int(x[n // 2]) == h // 2
print(f"2^31 int32 organ: {ms:.2f} ms split {st['run_split']} kind {st['check_result'] >> 4} ok={ok}", flush=True)
t = n // 100
x[: n - t] = torch.arange(n - t, dtype=torch.int64, device="cuda").to(torch.int32)
x[n - t:] = torch.randint(-(2**31), 2**31, (t,), device="cuda", generator=g, dtype=torch.int64).to(torch.int32)
s0 = int(x.to(torch.int64).sum().item())
ms, st = timed(ds, x)
ok = bool((x[1:] >= x[:-1]).all().item()) and int(x.to(torch.int64).sum().item()) == s0
print(f"2^31 int32 asc_tail: {ms:.2f} ms split {st['run_split']} kind {st['check_result'] >> 4} ok={ok}", flush=True)
del x, ds
torch.cuda.empty_cache()
n = 1 << 29
k = torch.randint(-(2**62), 2**62, (n,), device="cuda", generator=g, dtype=torch.int64)
s = int(0.8 * n)
k[:s] = torch.sort(k[:s]).values
v = torch.arange(n, device="cuda", dtype=torch.int32)
ksum, vsum = int((k >> 8).sum().item()), int(v.to(torch.int64).sum().item())
ds = DeviceSorter(n, torch.int64, True)
ms, st = timed(ds, k, v)
ok = bool((k[1:] >= k[:-1]).all().item()) and int((k >> 8).sum().item()) == ksum and int(v.to(torch.int64).sum().item()) == vsum
print(f"2^29 (int64, u32) sorted prefix 80 %: {ms:.2f} ms split {st['run_split']} kind {st['check_result'] >> 4} ok={ok}", flush=True)
