import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2106_05123_b200 import SortConfig, sort_device
rng = np.random.default_rng(5)
for n in (5000, 300000, 1 << 22, 1 << 26):
    for dt in (np.int32, np.int64, np.float32):
        if dt == np.float32:
            keys = rng.standard_normal(n).astype(dt)
        else:
            keys = rng.integers(np.iinfo(dt).min, np.iinfo(dt).max, n, dtype=dt)
        kd = torch.from_numpy(keys).cuda()
        st = sort_device(kd, config=SortConfig(bad_budget=0))
        ok = np.array_equal(kd.cpu().numpy(), np.sort(keys))
        print(n, np.dtype(dt).name, ok, "fallbacks", st["radix_fallbacks"], "segs", st["segments"], flush=True)
    # low cardinality + fallback
    keys = rng.integers(0, 3, n).astype(np.int32)
    kd = torch.from_numpy(keys).cuda()
    st = sort_device(kd, config=SortConfig(bad_budget=0))
    print(n, "k3", np.array_equal(kd.cpu().numpy(), np.sort(keys)), st["radix_fallbacks"])
    k = rng.integers(0, 50, n).astype(np.int64); v = rng.integers(0, 2**32, n, dtype=np.uint32)
    kd = torch.from_numpy(k).cuda(); vd = torch.from_numpy(v.view(np.int32)).cuda()
    st = sort_device(kd, vd, config=SortConfig(bad_budget=0))
    o = np.lexsort((v, k))
    print(n, "kv", np.array_equal(kd.cpu().numpy(), k[o]) and np.array_equal(vd.cpu().numpy().view(np.uint32), v[o]), st["radix_fallbacks"])
