"""One warm-up + one measured device sort of seeded uniform keys (for ncu / quick timing).

python tools/prof_sort.py [log2n] [dtype] [reps]
"""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2106_05123_b200 import DeviceSorter  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
dt = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "kv": torch.int64}[sys.argv[2] if len(sys.argv) > 2 else "i32"]
kv = len(sys.argv) > 2 and sys.argv[2] == "kv"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
n = 1 << log2n
g = torch.Generator(device="cuda")
g.manual_seed(1)
if dt == torch.float32:
    src = torch.randn(n, device="cuda", generator=g)
elif dt == torch.int32:
    src = torch.randint(-(2**31), 2**31, (n,), device="cuda", generator=g, dtype=torch.int64).to(torch.int32)
else:
    src = torch.randint(-(2**62), 2**62, (n,), device="cuda", generator=g, dtype=torch.int64)
vals = torch.arange(n, device="cuda", dtype=torch.int32) if kv else None
ds = DeviceSorter(n, dt, kv)
x = src.clone()
for r in range(reps):
    x.copy_(src)
    if vals is not None:
        vals.copy_(torch.arange(n, device="cuda", dtype=torch.int32))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ds.run(x, vals)
    b.record()
    st = ds.finish()
    ms = a.elapsed_time(b)
    ok = bool((x[1:] >= x[:-1]).all().item())
    tot = st["cycles_wait"] + st["cycles_work"]
    print(f"rep {r}: {ms:.3f} ms  {n / ms / 1e6:.2f} Gkeys/s  alg {st['bytes_algorithmic'] / ms / 1e6:.0f} GB/s  ok={ok} "
          f"wait {st['cycles_wait'] / tot:.3f} base {st['cycles_base'] / tot:.3f} spawn {st['cycles_spawn'] / tot:.3f} "
          f"tiles {st['tiles']} base_cases {st['base_cases']}", flush=True)

# per-level throughput: stop at depth d (profiling knob, output unsorted)
if len(sys.argv) > 4 and sys.argv[4]:
    from paper_2106_05123_b200 import SortConfig
    for d in [int(t) for t in sys.argv[4].split(",")]:
        ds2 = DeviceSorter(n, dt, kv)
        ds2._cfg.reserved[0] = d
        for r in range(2):
            x.copy_(src)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ds2.run(x, vals)
            b.record()
            st = ds2.finish()
        ms = a.elapsed_time(b)
        sch = st['sched_retire'] + st['sched_claim'] + st['sched_fetch'] + st['sched_idle']
        print(f"depth<{d}: {ms:.3f} ms  alg {st['bytes_algorithmic'] / ms / 1e6:.0f} GB/s tiles {st['tiles']} "
              f"wait {st['cycles_wait'] / (st['cycles_wait'] + st['cycles_work']):.3f} per-tile cycles: stage-wait "
              f"{st['sched_claim'] / st['tiles']:.0f} tile {st['sched_idle'] / st['tiles']:.0f} (atomic-wait "
              f"{st['sched_fetch'] / st['tiles']:.0f}) retire/chunk {st['sched_retire'] / max(1, st['tiles'] / 8):.0f}", flush=True)

# kernel split: partition kernel (events from the C ABI) vs whole call
if len(sys.argv) > 5:
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    ev[0].record()
    ev[1].record()
    torch.cuda.synchronize()
    for r in range(3):
        x.copy_(src)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ds.run(x, vals, events=ev)
        b.record()
        st = ds.finish()
    tot = a.elapsed_time(b)
    ks = ev[0].elapsed_time(ev[1])
    print(f"split: total {tot:.3f} ms, partition kernel {ks:.3f} ms ({st['bytes_algorithmic'] / ks / 1e6:.0f} GB/s alg), "
          f"rest (check+init+base) {tot - ks:.3f} ms; base bytes {st['bytes_base'] / 1e9:.2f} GB", flush=True)
