"""Leaf-kernel time of C4 (float32 N(0,1)) against uniform float32 / int32 keys at 2^26 (device timers):
  python tools/c4probe.py"""
import sys
import numpy as np, torch
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
from paper_2106_05123_b200 import DeviceSorter, workloads
n = 1 << 26
cases = {"C4.normal": workloads.c4("normal", n), "uniform f32": np.random.default_rng(1).random(n, dtype=np.float32),
         "uniform i32": workloads.c1(n)}
for name, keys in cases.items():
    src = torch.from_numpy(keys).cuda()
    x = src.clone()
    ds = DeviceSorter(n, x.dtype, False)
    rows = []
    for r in range(5):
        x.copy_(src); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); ds.run(x); b.record(); st = ds.finish()
        rows.append((a.elapsed_time(b), st["sort_ns"] / 1e6, st["base_ns"] / 1e6))
    rows.sort()
    print(name, "total %.3f ms k_sort %.3f leaf %.3f" % rows[2], "leaves", st["base_cases"], "levels", st["bytes_algorithmic"] / (8 * n))
