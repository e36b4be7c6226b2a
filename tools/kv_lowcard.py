"""Key-value sorts of low-cardinality int64 keys with distinct uint32 payloads (argsort by category):
wall time of sort_device (best of 3) and exact check.  python tools/kv_lowcard.py"""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2106_05123_b200 import sort_device
for k in (2, 16, 1024, 65536):
    n = 1 << 24
    rng = np.random.default_rng(k)
    keys = rng.integers(0, k, n).astype(np.int64) << 30
    vals = np.arange(n, dtype=np.uint32)
    rng.shuffle(vals)
    best = 1e9
    for rep in range(3):
        kd = torch.from_numpy(keys).cuda(); vd = torch.from_numpy(vals.view(np.int32)).cuda()
        torch.cuda.synchronize(); t = time.perf_counter()
        st = sort_device(kd, vd)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    dt = best
    order = np.lexsort((vals, keys))
    ok = np.array_equal(kd.cpu().numpy(), keys[order]) and np.array_equal(vd.cpu().numpy().view(np.uint32), vals[order])
    print(f"k={k} n=2^24 KV: {dt*1e3:.1f} ms ok={ok} leaves={st['base_cases']}")
