"""Per-kernel spans of the K4 two-run path on the C2 patterns (device timers):
  python tools/runs_prof.py [log2n] [two_run_min]"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2106_05123_b200 import DeviceSorter, SortConfig, workloads  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
cfg = SortConfig(two_run_min=int(sys.argv[2])) if len(sys.argv) > 2 else SortConfig()
n = 1 << lg
rng = np.random.default_rng(3)
app = np.arange(n, dtype=np.int32)
app[n - n // 100:] = np.sort(rng.integers(n - n // 50, n, n // 100)).astype(np.int32)  # newer keys, overlapping 2 %
half = workloads.c1(n).copy()
half[: n // 2].sort()
cases = {"sort50": half, "asc": workloads.c2("asc", n), "organ": workloads.c2("organ", n), "asc_tail": workloads.c2("asc_tail", n),
         "append_overlap": app, "uniform": workloads.c1(n)}
for name, keys in cases.items():
    src = torch.from_numpy(keys).cuda()
    x = src.clone()
    ds = DeviceSorter(n, x.dtype, False, config=cfg)
    rows = []
    for r in range(6):
        x.copy_(src)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ds.run(x)
        b.record()
        st = ds.finish()
        rows.append((a.elapsed_time(b) * 1e3, st["sort_ns"] / 1e3, st["base_ns"] / 1e3))
    rows.sort()
    t, s_, b_ = rows[len(rows) // 2]
    ok = bool((x[1:] >= x[:-1]).all().item())
    print(f"{name:15s} total {t:7.1f} us  k_sort {s_:7.1f}  leaf+merge {b_:7.1f}  other {t - s_ - b_:6.1f}  split {st['run_split']} "
          f"kind {st['check_result'] >> 4} bytes_base {st['bytes_base']} ok={ok}", flush=True)
    # kernel boundaries from events (they end the programmatic overlap between the kernels)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in ev:
        e.record()
    torch.cuda.synchronize()
    best = None
    for r in range(4):
        x.copy_(src)
        torch.cuda.synchronize()
        ds.run(x, events=ev)
        ds.finish()
        t = (ev[0].elapsed_time(ev[1]) * 1e3, ev[1].elapsed_time(ev[2]) * 1e3, ev[2].elapsed_time(ev[3]) * 1e3)
        best = t if best is None or sum(t) < sum(best) else best
    print(f"{'':15s} events: prologue (memset, check, init) {best[0]:6.1f} us  sorter {best[1]:6.1f}  leaf kernel {best[2]:6.1f}", flush=True)
