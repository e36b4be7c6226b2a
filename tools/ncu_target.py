"""Workload for one ncu capture of the kernels this round optimised (each sort once, after a warm-up):
2^28 uniform int32 normal sort (k_sort, k_base_big), the same input with the forced K5 fallback
(k_sort running digit passes), and 2^28 (int64, uint32) pairs of the C5 recipe (k_sort, k_base_wide).
  ncu --set full -k regex:'k_sort|k_base' python tools/ncu_target.py
"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2106_05123_b200 import DeviceSorter, SortConfig  # noqa: E402

n = 1 << 28
g = torch.Generator(device="cuda")
g.manual_seed(1)
src = torch.randint(-(2**31), 2**31, (n,), device="cuda", generator=g, dtype=torch.int64).to(torch.int32)
which = sys.argv[1:] or ["normal", "fallback", "c5"]
for w in which:
    if w == "organ":  # K4 two-run path: 2^24 organ pipe (k_check full pass, reversal, merge epilogue of k_base_big)
        from paper_2106_05123_b200 import workloads
        m = 1 << 24
        x = torch.from_numpy(workloads.c2("organ", m)).cuda()
        ds = DeviceSorter(m, torch.int32, False)
        ds.run(x)
        st = ds.finish()
        print(w, bool((x[1:] >= x[:-1]).all().item()), st["run_split"], flush=True)
    elif w in ("normal", "fallback"):
        ds = DeviceSorter(n, torch.int32, False, config=SortConfig(bad_budget=0 if w == "fallback" else -1))
        x = src.clone()
        ds.run(x)
        ds.finish()
        print(w, bool((x[1:] >= x[:-1]).all().item()), flush=True)
    else:
        k = (torch.randperm(n, device="cuda", generator=g) * (1 << 20) +
             torch.randint(0, 1 << 20, (n,), device="cuda", generator=g)).to(torch.int64)
        v = torch.arange(n, device="cuda", dtype=torch.int32)
        ds = DeviceSorter(n, torch.int64, True)
        ds.run(k, v)
        ds.finish()
        print(w, bool((k[1:] > k[:-1]).all().item()), flush=True)
    del ds
    torch.cuda.empty_cache()
