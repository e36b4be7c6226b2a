"""K5 fallback timing: the normal sort vs the forced fallback (SortConfig(bad_budget=0): the root starts
with an exhausted budget, so every big segment takes 8-bit digit passes) at full size, per element type.
Prints one JSON line per case: total ms, k_sort ms, k_sort algorithmic GB/s, counters, correctness.

  python tools/fallback_bench.py [log2n]
"""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2106_05123_b200 import DeviceSorter, SortConfig  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
n = 1 << log2n
g = torch.Generator(device="cuda")
g.manual_seed(3)
cases = {
    "int32": (torch.randint(-(2**31), 2**31, (n,), device="cuda", generator=g, dtype=torch.int64).to(torch.int32), None),
    "int64": (torch.randint(-(2**62), 2**62, (n,), device="cuda", generator=g, dtype=torch.int64), None),
    "kv_c5": ((torch.randperm(n, device="cuda", generator=g) * (1 << 20) +
               torch.randint(0, 1 << 20, (n,), device="cuda", generator=g)).to(torch.int64),
              torch.arange(n, device="cuda", dtype=torch.int32)),
    "int32_k16": (torch.randint(0, 16, (n,), device="cuda", generator=g, dtype=torch.int32), None),
}
for name, (k0, v0) in cases.items():
    exp = torch.sort(k0).values if v0 is None else None
    for label, cfg in (("normal", SortConfig()), ("fallback", SortConfig(bad_budget=0))):
        ds = DeviceSorter(n, k0.dtype, v0 is not None, config=cfg)
        ms = []
        for r in range(3):
            k = k0.clone()
            v = v0.clone() if v0 is not None else None
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            for e_ in ev:  # materialise the cudaEvent_t handles (torch creates them on first record)
                e_.record()
            torch.cuda.synchronize()
            ds.run(k, v, events=ev)
            st = ds.finish()
            ms.append((ev[0].elapsed_time(ev[3]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])))
        tot, ks, lf = min(ms)
        if v0 is None:
            ok = bool(torch.equal(k, exp))
        else:
            ok = bool((k[1:] > k[:-1]).all().item()) and bool(torch.equal(k0[v.long()], k))
        print(json.dumps({"case": name, "n": n, "mode": label, "ms": round(tot, 3), "k_sort_ms": round(ks, 3),
                          "leaf_ms": round(lf, 3), "k_sort_alg_GBps": round(st["bytes_algorithmic"] / ks / 1e6, 1),
                          "bytes_per_key": round(st["bytes_algorithmic"] / n, 1), "fallbacks": st["radix_fallbacks"],
                          "partitions": st["partition_right_calls"], "segments": st["segments"],
                          "max_depth": st["max_depth"], "ok": ok}), flush=True)
        del ds
