"""Time pdq_bucket (sample-sort bucketing, row f3) on seeded uniform keys.

python tools/prof_bucket.py [log2n] [dtype i32|i64|f32|kv] [P list, e.g. 2,4,8]
Algorithmic bytes = 3 (w+p) n: the count pass reads the shard, the scatter pass reads and writes it.
"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2106_05123_b200 import distributed as D  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
kind = sys.argv[2] if len(sys.argv) > 2 else "i32"
Ps = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "2,4,8").split(",")]
n = 1 << log2n
g = torch.Generator(device="cuda")
g.manual_seed(1)
dt = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "kv": torch.int64}[kind]
if dt == torch.float32:
    keys = torch.randn(n, device="cuda", generator=g)
elif dt == torch.int32:
    keys = torch.randint(-(2**31), 2**31, (n,), device="cuda", generator=g, dtype=torch.int64).to(torch.int32)
else:
    keys = torch.randint(-(2**62), 2**62, (n,), device="cuda", generator=g, dtype=torch.int64)
vals = torch.arange(n, device="cuda", dtype=torch.int32) if kind == "kv" else None
w = keys.element_size() + (4 if vals is not None else 0)
for P in Ps:
    rows = D.valid_samples(D.local_samples(keys, vals, 0, 256 * P).cpu().numpy())
    sp = D.choose_splitters(rows, P, keys.element_size(), dt == torch.float32)
    for r in range(4):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        bk, bv, c = D._bucket(keys, vals, 0, sp)
        b.record()
        torch.cuda.synchronize()
        del bk, bv
    ms = a.elapsed_time(b)
    cnt = c.cpu().numpy()
    print(f"P={P}: {ms:.3f} ms  {3 * w * n / ms / 1e6:.0f} GB/s alg  buckets min/max {cnt.min() / (n / P):.3f}/"
          f"{cnt.max() / (n / P):.3f} of n/P", flush=True)
