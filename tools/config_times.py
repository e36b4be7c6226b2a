"""Device time of one sort for every BASELINE config case at full size (inputs resident in HBM,
CUDA events around pdq_sort, median of 5 after 2 warm-ups).  Prints a markdown table.

python tools/config_times.py [case-prefix,...]
"""
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2106_05123_b200 import DeviceSorter, workloads  # noqa: E402

print("| case | n | dtype | ms | Gkeys/s | partitions R/L | bad | fallbacks | leaves |")
print("|---|---|---|---|---|---|---|---|---|")
only = sys.argv[1].split(",") if len(sys.argv) > 1 else None
for name, keys, vals in workloads.cases(0):
    if only and not any(name.startswith(o) for o in only):
        continue
    n = keys.size
    src = torch.from_numpy(keys).cuda()
    vsrc = None if vals is None else torch.from_numpy(vals.view(np.int32)).cuda()
    x = src.clone()
    v = None if vsrc is None else vsrc.clone()
    ds = DeviceSorter(n, x.dtype, v is not None)
    ts = []
    for r in range(7):
        x.copy_(src)
        if v is not None:
            v.copy_(vsrc)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ds.run(x, v)
        b.record()
        st = ds.finish()
        if r >= 2:
            ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    ok = bool((x[1:] >= x[:-1]).all().item()) if vals is None or True else True
    print(f"| {name} | 2^{n.bit_length() - 1} | {keys.dtype}{'+u32' if vals is not None else ''} | {ms:.3f} | "
          f"{n / ms / 1e6:.2f} | {st['partition_right_calls']}/{st['partition_left_calls']} | {st['bad_partitions']} | "
          f"{st['radix_fallbacks']} | {st['base_cases']} |{'' if ok else ' NOT SORTED'}", flush=True)
    del src, vsrc, x, v, ds
    torch.cuda.empty_cache()
