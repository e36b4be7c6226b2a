"""K4 two-run path check: sorted prefix + (ascending | descending | random) rest, against torch.sort.
  python tools/runs_check.py [i32|all]"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2106_05123_b200 import SortConfig, sort_device  # noqa: E402

only_i32 = len(sys.argv) > 1 and sys.argv[1] == "i32"
rng = np.random.default_rng(7)
bad = 0
cases = 0


def check(name, keys, vals=None, cfg=None, want_kind=None):
    global bad, cases
    cases += 1
    kd = torch.from_numpy(keys.copy()).cuda()
    vd = None if vals is None else torch.from_numpy(vals.copy().view(np.int32)).cuda()
    st = sort_device(kd, vd, config=cfg or SortConfig())
    got = kd.cpu().numpy()
    if vals is None:
        ok = np.array_equal(got, np.sort(keys, kind="stable"))
    else:
        order = np.lexsort((vals, keys))
        ok = np.array_equal(got, keys[order]) and np.array_equal(vd.cpu().numpy().view(np.uint32), vals[order])
    kind = (st["check_result"] >> 4) & 7
    if not ok or (want_kind is not None and kind != want_kind):
        bad += 1
        print("FAIL", name, "ok", ok, "kind", kind, "want", want_kind, "split", st["run_split"], flush=True)


def runs(n, s, kind, dtype, lo=None):
    """sorted prefix of s elements, then ascending / descending / random rest"""
    if np.issubdtype(dtype, np.floating):
        x = rng.standard_normal(n).astype(dtype)
    else:
        info = np.iinfo(dtype)
        x = rng.integers(info.min if lo is None else lo, info.max, n, dtype=np.int64 if dtype != np.int64 else np.int64).astype(dtype)
    x[:s].sort()
    if kind == 1:
        x[s:].sort()
    elif kind == 2:
        x[s:] = np.sort(x[s:])[::-1]
    # the boundary must be a descent for the split to land at s (else the prefix is longer: still fine)
    return x


cfg_small = SortConfig(two_run_min=64)
dtypes = [np.int32] if only_i32 else [np.int32, np.float32, np.int64, np.float64]
for dtype in dtypes:
    for n in (64, 100, 1000, 4097, 8192, 8193, 24577, 70001, 1 << 18, (1 << 20) + 3):
        for frac in (0.5, 0.51, 0.75, 0.99, 1.0 - 2.0 / n):
            s = max(int(n * frac), (n + 1) // 2)
            if s >= n:
                continue
            for kind in (1, 2, 3):
                x = runs(n, s, kind, dtype)
                check(f"{np.dtype(dtype).name} n={n} s={s} kind={kind}", x, cfg=cfg_small)
                # mirrored: sorted suffix of s elements after an ascending / descending / random first run
                y = runs(n, s, 3, dtype)[::-1].copy()  # descending suffix ...
                y[n - s:] = np.sort(y[n - s:])         # ... made ascending
                if kind == 1:
                    y[: n - s].sort()
                elif kind == 2:
                    y[: n - s] = np.sort(y[: n - s])[::-1]
                check(f"{np.dtype(dtype).name} n={n} s={s} kind={kind} mirror", y, cfg=cfg_small)
                if not only_i32 and n <= (1 << 18):
                    v = rng.permutation(n).astype(np.uint32)
                    check(f"{np.dtype(dtype).name}+kv n={n} s={s} kind={kind}", x, v, cfg=cfg_small)
    # duplicates across the runs, keys-only and with payloads
    n = 100000
    x = np.sort(rng.integers(0, 50, n)).astype(dtype)
    x[60000:] = np.sort(rng.integers(0, 50, 40000)).astype(dtype)
    check(f"{np.dtype(dtype).name} dup asc", x, cfg=cfg_small, want_kind=1)
    if not only_i32:
        v = rng.integers(0, 5, n).astype(np.uint32)
        # make each run sorted in (key, payload) order
        for a, b in ((0, 60000), (60000, n)):
            o = np.lexsort((v[a:b], x[a:b]))
            x[a:b], v[a:b] = x[a:b][o], v[a:b][o]
        check(f"{np.dtype(dtype).name}+kv dup asc", x, v, cfg=cfg_small)
# default threshold: the BASELINE C2 patterns
n = 1 << 24
x = np.arange(n, dtype=np.int32)
x[n - n // 100:] = rng.integers(-2**31, 2**31, n // 100).astype(np.int32)
check("C2 asc_tail", x, want_kind=3)
h = n // 2
x = np.concatenate([np.arange(h), np.arange(h)[::-1]]).astype(np.int32)
check("C2 organ", x, want_kind=2)
x = np.concatenate([np.arange(0, 2 * h, 2), np.arange(1, 2 * h, 2)]).astype(np.int32)
check("two asc runs", x, want_kind=1)
print(f"{cases} cases, {bad} failures")
sys.exit(1 if bad else 0)
