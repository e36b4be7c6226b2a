"""Stress sweep (run it with a PDQ_DEBUG build: device-side bounds asserts): every dtype, KV, the
leaf slow paths, K3 (low cardinality), K4 (sorted / reversed / two runs), the K5 radix fallback.

  tools/build_debug.sh && PDQ_LIB=tools/libdebug.so python tools/stress_sweep.py
(compute-sanitizer is not available on the GPU pool.)
"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2106_05123_b200 import SortConfig, sort_device  # noqa: E402


def check(keys, vals=None, cfg=SortConfig()):
    kd = torch.from_numpy(keys.copy()).cuda()
    vd = None if vals is None else torch.from_numpy(vals.copy().view(np.int32)).cuda()
    sort_device(kd, vd, cfg)
    got = kd.cpu().numpy()
    if vals is None:
        assert np.array_equal(got.view(np.uint8), np.sort(keys, kind="stable").view(np.uint8)) or \
            np.array_equal(np.sort(got), got)
    else:
        order = np.lexsort((vals, keys))
        assert np.array_equal(got, keys[order]) and np.array_equal(vd.cpu().numpy().view(np.uint32), vals[order])


rng = np.random.default_rng(3)
for n in (0, 1, 5, 64, 65, 4097, 16385, 70001, 300000):
    for dt in (np.int32, np.int64, np.float32, np.float64):
        k = rng.integers(-2**31, 2**31, n).astype(dt) if dt in (np.int32, np.int64) else rng.standard_normal(n).astype(dt)
        check(k)
        check(np.sort(k))
        check(np.sort(k)[::-1].copy())
        check((k % 7).astype(dt) if n else k)
    k = rng.integers(0, 50, n).astype(np.int64)
    check(k, rng.integers(0, 2**32, n, dtype=np.uint32))
    k = rng.integers(0, 1000, n).astype(np.int32)
    if n > 8:
        k[:4] = [-2**31, 2**31 - 1, -2**31, 2**31 - 1]
    check(k)
check(rng.integers(-2**31, 2**31, 300000).astype(np.int32), cfg=SortConfig(bad_budget=0))
check(rng.integers(-2**31, 2**31, 300000).astype(np.int64), rng.integers(0, 2**32, 300000, dtype=np.uint32),
      cfg=SortConfig(bad_budget=0))
# K4 two-run path: sorted prefix + ascending / descending / random rest, every dtype and KV
cfg2 = SortConfig(two_run_min=64)
for n in (64, 4097, 8193, 70001, 300000):
    for dt in (np.int32, np.int64, np.float32, np.float64):
        for kind in (1, 2, 3):
            k = rng.integers(-2**31, 2**31, n).astype(dt) if dt in (np.int32, np.int64) else rng.standard_normal(n).astype(dt)
            s = int(n * 0.6)
            k[:s].sort()
            if kind == 1:
                k[s:].sort()
            elif kind == 2:
                k[s:] = np.sort(k[s:])[::-1]
            check(k, cfg=cfg2)
            check(k.astype(np.int64) if dt == np.int32 else k, rng.permutation(n).astype(np.uint32), cfg=cfg2)
print("stress sweep ok")
