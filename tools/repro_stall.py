"""Reproduce the task-queue stall found by tools/fuzz.py seed 29 (int32 saw-tooth keys + a 2-bit payload,
forced fallback, base_case_size 1024) and print the device state it leaves:  python tools/repro_stall.py"""
import ctypes
import sys
import numpy as np, torch
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
from paper_2106_05123_b200 import DeviceSorter, SortConfig, _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3356801
period = int(sys.argv[2]) if len(sys.argv) > 2 else 1757
keys = (np.arange(n) % period).astype(np.int32)
vals = np.random.default_rng(29).integers(0, 4, n).astype(np.uint32)
cfg = SortConfig(base_case_size=1024, bad_budget=0)
kd = torch.from_numpy(keys.copy()).cuda()
vd = torch.from_numpy(vals.copy().view(np.int32)).cuda()
ds = DeviceSorter(n, kd.dtype, True, config=cfg)
ds.run(kd, vd)
st = _lib.PdqStats()
rc = _lib.lib().pdq_sort_finish(ctypes.c_void_p(ds.workspace.data_ptr()), ctypes.byref(st),
                                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
print("rc", rc, {k: v for k, v in st.as_dict().items() if not k.startswith(("cycles", "sched"))})
state = ds.workspace[:1024].cpu().numpy().view(np.uint64)
print("q_head", int(state[0]), "q_tail", int(state[16]), "keys_final", int(state[32]), "of", n)
w = ds.workspace[32 * 8 + 8: 32 * 8 + 8 + 24].cpu().numpy().view(np.uint32)
print("done, seg_alloc, status, check_bits, reverse, rslot_alloc:", w.tolist())
if rc != 0:
    a256 = lambda x: (x + 255) & ~255
    off = a256(640) + a256(n * 4 + 16) + a256(n * 4 + 16)
    nseg = int(w[1])
    segs = ds.workspace[off: off + nseg * 128].cpu().numpy()
    i64 = segs.view(np.int64).reshape(nseg, 16)
    u32 = segs.view(np.uint32).reshape(nseg, 32)
    stuck = 0
    for s in range(nseg):
        begin, end = int(i64[s, 0]), int(i64[s, 1])
        pivot_v, lb_v, ntiles, info = (int(x) for x in u32[s, 8:12])
        budget, depth = int(u32[s, 12]), int(u32[s, 13])
        tiles_done, rbit = int(u32[s, 20]), int(u32[s, 21])
        rslot = int(u32[s, 23])
        if tiles_done != ntiles and stuck < 12:
            stuck += 1
            print(f"seg {s}: [{begin}, {end}) m={end - begin} ntiles={ntiles} done={tiles_done} info={info:#x} rbit={rbit} "
                  f"nd={pivot_v} depth={depth} rslot={rslot} cnt_left={int(i64[s, 7]) & 0xFFFFFFFF}/{int(i64[s, 7]) >> 32}")
    print("stuck segments listed:", stuck)
