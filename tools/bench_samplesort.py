"""Sharded sort of one array over N GPUs (row f3, distributed.sample_sort): one JSON line.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
      --master-port 29511 tools/bench_samplesort.py [--log2n 28] [--steps 5] [--warmup 3]

Each rank holds 2^log2n uniform int32 keys (weak scaling: the array is N · 2^log2n keys).  A step
is the whole collective (samples, splitters, pdq_bucket, two all-to-alls, the local sort), timed
with CUDA events between barriers; the reported time is the max over ranks.  Keys/s = N · 2^log2n
per step time.  Inputs are restored from a device copy before every step (outside the timing).
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_05123_b200 import distributed as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=28)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    n = 1 << a.log2n
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    src = torch.randint(-(2**31), 2**31, (n,), device=dev, generator=g, dtype=torch.int64).to(torch.int32)
    keys = torch.empty_like(src)
    times = []
    total_out = 0
    for i in range(a.warmup + a.steps):
        keys.copy_(src)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out, _ = D.sample_sort(keys)
        e1.record()
        torch.cuda.synchronize()
        if i >= a.warmup:
            times.append(e0.elapsed_time(e1))
            total_out = out.numel()
        del out
    ms = torch.tensor([sum(times) / len(times)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    cnt = torch.tensor([total_out], device=dev)
    mx = cnt.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": "sharded sort keys/s", "value": world * n / (ms.item() / 1e3), "unit": "keys/s",
                          "n_gpus": world, "keys_per_rank": n, "ms_per_step": ms.item(), "steps": a.steps,
                          "warmup": a.warmup, "scaling": "weak", "max_slice_over_mean": mx.item() / n}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
