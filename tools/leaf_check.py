"""Quick int32 keys-only correctness sweep for leaf-kernel variants (PDQ_LIB=tools/libvar_x.so):
sizes around the leaf capacity and distributions that take the fast path, the slow path (big
buckets) and the radix path, against np.sort.  python tools/leaf_check.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2106_05123_b200 import SortConfig, sort_device  # noqa: E402

rng = np.random.default_rng(11)
bad = 0
sizes = [65, 100, 1000, 4095, 4096, 4097, 12000, 16383, 16384, 16385, 24571, 24572, 24573, 30000, 100003, 1 << 20, 3 << 20]
for n in sizes:
    cases = {
        "uniform": rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32),
        "narrow": rng.integers(0, n // 3 + 1, n).astype(np.int32),
        "dups7": rng.integers(0, 7, n).astype(np.int32),
        "clustered": (rng.integers(0, 2, n) * 2**30 + rng.integers(0, 50, n)).astype(np.int32),
        "geom": np.minimum(rng.geometric(0.001, n), 2**31 - 1).astype(np.int32),
        "extremes": rng.choice(np.array([-2**31, 2**31 - 1, 0, -1, 1], dtype=np.int32), n),
        "normal_f": None,
    }
    for name, k in cases.items():
        if k is None:
            k = (rng.standard_normal(n) * 1e6).astype(np.int32)
        for off in (0, 1, 3):
            base = torch.from_numpy(np.concatenate([np.zeros(off, np.int32), k])).cuda()
            view = base[off:]
            if view.data_ptr() % 16:
                kd = view.clone()
            else:
                kd = view
            sort_device(kd)
            ok = np.array_equal(kd.cpu().numpy(), np.sort(k))
            if not ok:
                bad += 1
                print("FAIL", n, name, off, flush=True)
print("leaf_check", "ok" if bad == 0 else f"{bad} failures", flush=True)
