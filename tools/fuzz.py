"""Randomised differential test of the device sort against numpy (run on the GPU box):
random sizes, element types, payloads, input patterns and config toggles.
  python tools/fuzz.py [seconds] [seed]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2106_05123_b200 import SortConfig, sort_device  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
DT = [np.int32, np.int64, np.float32, np.float64]


def keys_of(n, dt, pattern):
    if np.dtype(dt).kind == "f":
        base = rng.standard_normal(n).astype(dt)
        if pattern == "special" and n:
            base[rng.integers(0, n, max(1, n // 50))] = rng.choice(np.array([np.inf, -np.inf, 0.0, 1e-30, -1e-30], dtype=dt), max(1, n // 50))
    else:
        info = np.iinfo(dt)
        base = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
        if pattern == "special" and n:
            base[rng.integers(0, n, max(1, n // 50))] = rng.choice(np.array([info.min, info.max, 0, -1, 1], dtype=dt), max(1, n // 50))
    x = base
    if pattern == "few":
        k = int(rng.choice([1, 2, 3, 16, 257, 5000]))
        x = base[rng.integers(0, max(1, min(k, n)), n)] if n else base
    elif pattern == "sorted":
        x = np.sort(base)
    elif pattern == "reversed":
        x = np.sort(base)[::-1].copy()
    elif pattern == "runs":  # k ascending or descending runs
        k = int(rng.integers(2, 9))
        cuts = np.sort(rng.integers(0, n + 1, k - 1)) if n else np.zeros(k - 1, dtype=np.int64)
        x = base.copy()
        lo = 0
        for hi in list(cuts) + [n]:
            seg = np.sort(x[lo:hi])
            x[lo:hi] = seg if rng.random() < 0.7 else seg[::-1]
            lo = hi
    elif pattern == "prefix":  # sorted prefix of a random length, then anything
        s = int(rng.integers(0, n + 1))
        x = base.copy()
        x[:s].sort()
        kind = rng.integers(0, 3)
        if kind == 0:
            x[s:].sort()
        elif kind == 1:
            x[s:] = np.sort(x[s:])[::-1]
    elif pattern == "suffix":  # anything, then a sorted suffix from a random position
        s = int(rng.integers(0, n + 1))
        x = base.copy()
        x[s:].sort()
        kind = rng.integers(0, 3)
        if kind == 0:
            x[:s].sort()
        elif kind == 1:
            x[:s] = np.sort(x[:s])[::-1]
    elif pattern == "nearly":
        x = np.sort(base)
        m = max(1, n // 100)
        if n > 1:
            i, j = rng.integers(0, n, m), rng.integers(0, n, m)
            x[i], x[j] = x[j].copy(), x[i].copy()
    elif pattern == "saw":
        p = int(rng.integers(2, 5000))
        x = (np.arange(n) % p).astype(dt)
    elif pattern == "organ":
        h = (n + 1) // 2
        x = np.concatenate([np.arange(h), np.arange(n - h)[::-1]]).astype(dt)
    return np.ascontiguousarray(x)


t0 = time.time()
it = 0
hist = {}
while time.time() - t0 < budget:
    it += 1
    lg = rng.uniform(0, 22.5)
    n = int(2 ** lg) + int(rng.integers(-3, 4))
    n = max(0, n)
    if rng.random() < 0.05:
        n = int(rng.choice([0, 1, 2, 63, 64, 65, 4096, 8188, 8189, 24572, 24573]))
    dt = DT[rng.integers(0, 4)]
    kv = rng.random() < 0.35
    pattern = str(rng.choice(["uniform", "few", "sorted", "reversed", "runs", "prefix", "suffix", "nearly", "saw", "organ", "special"]))
    cfg = SortConfig(use_partition_left=bool(rng.random() < 0.85), use_break_patterns=bool(rng.random() < 0.85),
                     use_partial_insertion=bool(rng.random() < 0.85),
                     bad_partition_shift=int(rng.choice([1, 2, 3, 3, 3, 5])),
                     bad_budget=int(rng.choice([-1, -1, -1, 0, 2])),
                     base_case_size=int(rng.choice([1024, 4096, 32768, 32768])),
                     two_run_min=int(rng.choice([0, 64, 64, 1000, 100000])))
    keys = keys_of(n, dt, pattern)
    vals = None
    if kv:
        vals = (rng.permutation(n) if rng.random() < 0.5 else rng.integers(0, 4, n)).astype(np.uint32)
        if pattern in ("sorted", "prefix", "runs") and n:  # make the pairs follow the pattern too
            o = np.lexsort((vals, keys))
            if pattern == "sorted":
                keys, vals = keys[o], vals[o]
    kd = torch.from_numpy(keys.copy()).cuda()
    vd = None if vals is None else torch.from_numpy(vals.copy().view(np.int32)).cuda()
    try:
        st = sort_device(kd, vd, cfg)
    except Exception as exc:  # a device-side failure: keep the input that caused it
        np.save(f"gpurun_out/fuzz_exc_{seed}_{it}_keys.npy", keys)
        if vals is not None:
            np.save(f"gpurun_out/fuzz_exc_{seed}_{it}_vals.npy", vals)
        print("EXCEPTION", it, n, np.dtype(dt).name, kv, pattern, cfg, repr(exc), flush=True)
        sys.exit(2)
    got = kd.cpu().numpy()
    if vals is None:
        want = np.sort(keys, kind="stable")
        ok = got.tobytes() == want.tobytes() or (np.dtype(dt).kind == "f" and np.array_equal(got, want))
    else:
        o = np.lexsort((vals, keys))
        ok = np.array_equal(got, keys[o]) and np.array_equal(vd.cpu().numpy().view(np.uint32), vals[o])
    key = (pattern, "kv" if kv else "k", (st["check_result"] >> 4) & 7)
    hist[key] = hist.get(key, 0) + 1
    if not ok or st["status"] != 0:
        np.save(f"gpurun_out/fuzz_fail_{seed}_{it}_keys.npy", keys)
        if vals is not None:
            np.save(f"gpurun_out/fuzz_fail_{seed}_{it}_vals.npy", vals)
        print("FAIL", it, n, np.dtype(dt).name, kv, pattern, cfg, st, flush=True)
        sys.exit(1)
two = sum(v for k, v in hist.items() if k[2])
print(f"fuzz ok: {it} sorts in {time.time() - t0:.0f} s (seed {seed}); two-run path taken in {two} sorts", flush=True)
try:
    print("by (pattern, kv, kind):", {k: v for k, v in sorted(hist.items()) if k[2]})
except BrokenPipeError:  # piped into head
    pass
