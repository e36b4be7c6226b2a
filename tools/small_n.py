"""Small-n latency probe: per-phase device time (prologue = memsets + check + init, k_sort, leaf kernel)
of int32 uniform sorts at 2^16 .. 2^22 (median of 20), and k_sort time when descending stops at depth d
(profiling knob reserved[0]; output unsorted) at 2^20.
  python tools/small_n.py"""
import json
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2106_05123_b200 import DeviceSorter  # noqa: E402

g = torch.Generator(device="cuda")
g.manual_seed(5)
for lg in (16, 18, 20, 22):
    n = 1 << lg
    src = torch.randint(-(2**31), 2**31, (n,), device="cuda", generator=g, dtype=torch.int64).to(torch.int32)
    for depth in ([0] + list(range(1, 9))) if lg == 20 else [0]:
        ds = DeviceSorter(n, torch.int32, False)
        ds._cfg.reserved[0] = depth
        x = src.clone()
        res = []
        for r in range(25):
            x.copy_(src)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            for e in ev:
                e.record()
            torch.cuda.synchronize()
            # only the outer events: inner ones would end the kernels' programmatic overlap; the kernel
            # spans come from the device timers
            ds.run(x, events=[ev[0], None, None, ev[3]])
            st = ds.finish()
            if r >= 5:
                tot = ev[0].elapsed_time(ev[3])
                res.append((tot, tot - (st["sort_ns"] + st["base_ns"]) / 1e6, st["sort_ns"] / 1e6, st["base_ns"] / 1e6))
        med = [statistics.median(c) for c in zip(*res)]
        ok = bool((x[1:] >= x[:-1]).all().item()) if depth == 0 else None
        print(json.dumps({"log2n": lg, "depth_limit": depth, "total_us": round(med[0] * 1e3, 1),
                          "other_us": round(med[1] * 1e3, 1), "k_sort_us": round(med[2] * 1e3, 1),
                          "leaf_us": round(med[3] * 1e3, 1), "partitions": st["partition_right_calls"],
                          "max_depth": st["max_depth"], "tiles": st["tiles"], "ok": ok}), flush=True)
