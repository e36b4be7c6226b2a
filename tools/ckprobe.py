"""Bytes the K4 check pass reads before it stops on uniform keys, and the prologue time, 2^20 .. 2^28:
  python tools/ckprobe.py"""
import sys, torch
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
from paper_2106_05123_b200 import DeviceSorter
g = torch.Generator(device="cuda"); g.manual_seed(1)
for lg in (20, 22, 24, 26, 28):
    n = 1 << lg
    src = torch.randint(-(2**31), 2**31, (n,), device="cuda", generator=g, dtype=torch.int64).to(torch.int32)
    ds = DeviceSorter(n, torch.int32, False)
    for r in range(3):
        x = src.clone()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        for e in ev: e.record()
        torch.cuda.synchronize()
        ds.run(x, events=ev); st = ds.finish()
    print(lg, "bytes_check", st["bytes_check"], "of", 4 * n, "check_result", st["check_result"], "prologue us", round(ev[0].elapsed_time(ev[1]) * 1e3, 1))
