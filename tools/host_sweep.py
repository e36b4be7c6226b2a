"""Sweep pdq_host_sort's staging knobs (threads, chunk, slots, streaming stores) at 2^28 int32: one
process, a new HostSorter per setting (the env is read at create time).
  python tools/host_sweep.py"""
import itertools
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2106_05123_b200 import HostSorter, workloads  # noqa: E402

n = 1 << 28
src = workloads.roofline_input(n)
buf = np.empty_like(src)
print("lscpu:", os.cpu_count(), "cpus", flush=True)
settings = []
if len(sys.argv) > 1 and sys.argv[1] == "coarse":
    for th, ck, sl in itertools.product((8, 12, 16, 24), (512, 1024, 2048, 4096, 8192), (2, 3, 4)):
        settings.append((th, ck, sl, 1, 1))
    settings.append((16, 2048, 2, 0, 1))
else:
    for th, ck, sl in itertools.product((10, 12, 14, 16), (3072, 4096, 6144), (2, 3)):
        settings.append((th, ck, sl, 1, 1))
    for th in (12, 16):
        settings.append((th, 4096, 2, 1, 0))
        settings.append((th, 2048, 2, 1, 1))
for th, ck, sl, nt, ramp in settings:
    os.environ.update(PDQ_HOST_THREADS=str(th), PDQ_HOST_CHUNK_KB=str(ck), PDQ_HOST_SLOTS=str(sl), PDQ_HOST_NT=str(nt), PDQ_HOST_RAMP=str(ramp))
    hs = HostSorter(0, 0)
    rows = []
    for r in range(9):
        np.copyto(buf, src)
        t0 = time.perf_counter()
        _, ph = hs.sort(buf, phases=True)
        t = (time.perf_counter() - t0) * 1e3
        if r:
            rows.append((t,) + tuple(ph))
    hs.close()
    med = [statistics.median(c) for c in zip(*rows)]
    print(f"threads {th:2d} chunk {ck:5d} KB slots {sl} nt {nt} ramp {ramp}: total {med[0]:6.2f} ms  h2d {med[1]:6.2f}  sort-wait {med[2]:5.2f}  "
          f"d2h {med[3]:6.2f}  (device sort {med[4]:.2f})", flush=True)
