"""Benchmark of the B200 pdqsort path on BASELINE.json's headline workload.

Workload (BASELINE.json metric): sort n = 2^28 uniform int32 keys on one B200
("R" in SURVEY.md §8(d)).  One step = one full sort of a distinct, already
HBM-resident 1 GiB input (inputs are larger than L2, so no flush is needed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--log2n 28]

--impl reference times the reference's CPU algorithm on the host (the C
restatement in oracle/, pinned to the Python reference's outputs and
counters; the Python reference itself is not present on the GPU box) on a
bounded sample of the same workload.  Under torchrun only rank 0 runs it.

N > 1: one process per GPU, each sorting its own replica (the north star is a
one-GPU sort: "replicas only", weak scaling); the timed region is bracketed by
barriers and the max over ranks is reported.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sorted keys/sec and achieved HBM GB/s vs ~8 TB/s at n=2^28 (1 B200) vs reference CPU"
UNIT = "keys/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--log2n", type=int, default=28)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def ncu_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    (profiles/*_ncu_kernels.json, written from the same bench command), or None."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_kernels.json")))
    if not files:
        return None, None
    with open(files[-1]) as f:
        d = json.load(f).get(kernel)
    if not d:
        return None, None
    return (d["dram_read_GB"] + d["dram_write_GB"]) * 1e9, os.path.relpath(files[-1], ROOT)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler running during the timed region (the recipe's clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def wait_first(self, timeout=10.0):
        t0 = time.perf_counter()
        while self.proc and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        """Median SM clock and active throttle reasons over samples taken in [t0, t1]
        (widened to the nearest samples on either side if the window is shorter than
        the sampling period)."""
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sel = self.lines
        if t0 is not None and self.lines:
            before = [x for x in self.lines if x[0] < t0]
            inside = [x for x in self.lines if t0 <= x[0] <= t1]
            after = [x for x in self.lines if x[0] > t1]
            sel = before[-1:] + inside + after[:1]
        for _, ln in sel:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_sample(n_sample: int, min_seconds: float, seed_offset: int = 6):
    """Time the reference algorithm (C restatement, 1 thread) on seeded samples of the
    workload distribution; returns (keys/s, seconds, sorts, n_sample)."""
    import numpy as np

    from oracle import oracle
    from paper_2106_05123_b200 import workloads

    oracle.lib()
    total_t, total_keys, sorts = 0.0, 0, 0
    rng = np.random.Generator(np.random.PCG64(workloads.SEED + 1000 + seed_offset))
    while total_t < min_seconds or sorts < 1:
        a = rng.integers(-(2**31), 2**31, n_sample, dtype=np.int64).astype(np.int32)
        t0 = time.perf_counter_ns()
        oracle.sort(a)  # driver.py:267 restated; list-of-ints default path (block partition)
        t1 = time.perf_counter_ns()
        assert bool(np.all(a[1:] >= a[:-1]))
        total_t += (t1 - t0) / 1e9
        total_keys += n_sample
        sorts += 1
    return total_keys / total_t, total_t, sorts


def reduce_max_ms(ms: float, dist, device) -> float:
    """Max over ranks of a per-rank device time (the contract's multi-GPU clock)."""
    if dist is None:
        return float(ms)
    import torch

    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def weak_scaling_value(n_per_rank: int, steps: int, world: int, max_ms: float) -> float:
    """Whole-job keys/s: every rank sorts its own replica of n keys per step."""
    return n_per_rank * steps * world / (max_ms / 1e3)


def run_reference(args, rank, world):
    if rank != 0:
        return
    n_sample = 1 << 22
    vals = []
    for i in range(args.warmup + args.steps):
        ks, _, _ = cpu_reference_sample(n_sample, 0.0, seed_offset=i)
        if i >= args.warmup:
            vals.append(ks)
    v = statistics.median(vals)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": n_sample / v * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic (seeded PCG64 uniform int32)",
        "config": {"workload": f"R: uniform int32, bounded CPU sample n=2^22 per step of the n=2^{args.log2n} "
                               "workload", "n": 1 << args.log2n, "sample_n": n_sample},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"one sort of 2^22 seeded uniform int32 keys per step, 1 thread "
                                   f"(pdqsort is sequential, SPEC.md:277) of {os.cpu_count()} host cores"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2106_05123_b200 import DeviceSorter, sort_device

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod

        dist = dist_mod
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    n = 1 << args.log2n
    K, W = args.steps, args.warmup
    # distinct seeded inputs, resident in HBM before timing (each 1 GiB > 126 MB L2)
    free, _ = torch.cuda.mem_get_info()
    need_per = n * 4
    n_inputs = max(1, min(K + W, int((free * 0.7 - 3 * need_per) // need_per)))
    g = torch.Generator(device=dev)
    inputs = []
    for i in range(n_inputs):
        g.manual_seed(1000003 * (rank + 1) + i)
        inputs.append(torch.randint(-(2**31), 2**31, (n,), dtype=torch.int64, device=dev,
                                    generator=g).to(torch.int32))
    pristine = None
    if n_inputs < K + W:
        pristine = [x.clone() for x in inputs]
    ds = DeviceSorter(n, torch.int32, False, dev)
    stream = torch.cuda.current_stream(dev)

    def restore(i):
        if pristine is not None:
            inputs[i % n_inputs].copy_(pristine[i % n_inputs])

    clocks = Clocks(local_rank)
    clocks.__enter__()
    clocks.wait_first()
    # warmup (untimed)
    stats = None
    for i in range(W):
        restore(i)
        ds.run(inputs[i % n_inputs])
    if W:
        stats = ds.finish()
    for i in range(W, W + K):
        restore(i)
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for pair in kev:  # materialise the raw cudaEvent_t handles
        pair[0].record(stream)
        pair[1].record(stream)
    torch.cuda.synchronize()
    step_stats = []
    t_wall0 = time.perf_counter()
    try:
        start_all = torch.cuda.Event(enable_timing=True)
        end_all = torch.cuda.Event(enable_timing=True)
        start_all.record(stream)
        for s in range(K):
            ev[s][0].record(stream)
            ds.run(inputs[(W + s) % n_inputs], events=kev[s])
            ev[s][1].record(stream)
            if pristine is not None:
                step_stats.append(ds.finish())
                restore(W + s + 1)
        end_all.record(stream)
        torch.cuda.synchronize()
        t_wall1 = time.perf_counter()
        time.sleep(0.12)  # let the sampler report the tail of the timed region
    finally:
        clocks.__exit__(None, None, None)
    t_wall = t_wall1 - t_wall0
    if pristine is None:
        stats = ds.finish()
    else:
        stats = step_stats[-1]
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ksort_ms = [a.elapsed_time(b) for a, b in kev]
    total_ms = sum(step_ms) if pristine is not None else start_all.elapsed_time(end_all)
    total_ms = reduce_max_ms(total_ms, dist, dev)
    barrier()

    # verify the last timed output (cheap device check)
    last = inputs[(W + K - 1) % n_inputs]
    ok = bool((last[1:] >= last[:-1]).all().item())

    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(n, K, W, dev, rank)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        ks, secs, sorts = cpu_reference_sample(1 << 24, 10.0)
        cpu = {"value": ks, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{sorts} sorts of 2^24 seeded uniform int32 keys ({secs:.1f} s), 1 thread of "
                         f"{os.cpu_count()} host cores; oracle/ C restatement of the reference (the Python "
                         "reference is not on the GPU box)"}

    if rank == 0:
        peak, peak_src = peaks()
        value = weak_scaling_value(n, K, world, total_ms)
        # roofline of the dominant kernel (the persistent sorter k_sort): algorithmic bytes per launch
        # (device counter, SURVEY.md §8(d) byte model over the segments it processed) / its event time
        bytes_launch = stats["bytes_algorithmic"]
        traffic, traffic_src = ncu_traffic("k_sort")
        ks_ms = statistics.mean(ksort_ms)
        achieved = bytes_launch / (ks_ms / 1e3) / 1e9
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": K,
            "warmup": W,
            "ms_per_step": total_ms / K,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "int32",
            "data": "synthetic (seeded uniform int32 over the full range, generated on device)",
            "config": {
                "workload": f"R: uniform int32 keys, n=2^{args.log2n}, keys-only ascending sort, one sort per step",
                "n": n,
                "parallelism": "replicas only" if world > 1 else "1 GPU",
                "l2": "inputs larger than L2 (1 GiB each, distinct per step)" if pristine is None else
                      "inputs restored by D2D copy between steps, outside the per-step events",
                "sort_ok": ok,
            },
            "roofline": {
                "bound": "hbm",
                "kernel": "k_sort (persistent segment-queue partition kernel: K1-K6)",
                "achieved": achieved,
                "peak": peak,
                "peak_source": peak_src,
                "unit": "GB/s",
                "frac": achieved / peak,
                "frac_vs_8tbs": achieved / 8000.0,
                "traffic": traffic,
                "traffic_source": traffic_src,
                "bytes_algorithmic_per_launch": bytes_launch,
                "bytes_per_key": bytes_launch / n,
                "kernel_ms": ks_ms,
                "kernel_share_of_step": ks_ms / (total_ms / K),
                "whole_sort_alg_GBps": (bytes_launch + stats["bytes_base"] + stats["bytes_check"]) / (total_ms / K / 1e3) / 1e9,
                "whole_sort_frac": (bytes_launch + stats["bytes_base"] + stats["bytes_check"]) / (total_ms / K / 1e3) / 1e9 / peak,
            },
            "gpu_launches": 4 * K,
            "device_counters": stats,
            "clocks": clocks.summary(t_wall0, t_wall1),
            "wall_s_timed_region": t_wall,
        }
        if e2e is not None:
            line["e2e"] = e2e
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def e2e_leg(n, K, W, dev, rank):
    """Same metric through the public host-batch API (HostPipeline over the C ABI) with HOST buffers:
    every step copies its input from pinned host memory to the device, sorts it, and copies the
    sorted keys back to pinned host memory; H2D of step i+1, the sort of step i and the D2H of
    step i-1 overlap on three streams.  Timed from the first H2D to the last D2H (CUDA events)."""
    import torch

    from paper_2106_05123_b200 import HostPipeline

    g = torch.Generator()
    g.manual_seed(77 + rank)
    host_in = [torch.randint(-(2**31), 2**31, (n,), dtype=torch.int64, generator=g).to(torch.int32).pin_memory()
               for _ in range(2)]
    host_out = [torch.empty_like(host_in[0]).pin_memory() for _ in range(2)]
    pipe = HostPipeline(n, torch.int32, dev)
    steps = max(4, K)
    ins = [host_in[i % 2] for i in range(steps)]
    outs = [host_out[i % 2] for i in range(steps)]
    pipe.sort(ins[:max(1, W)], outs[:max(1, W)])  # warm-up
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    pipe.sort(ins, outs, events=ev)
    ms = ev[0].elapsed_time(ev[1]) / steps
    ok = all(bool(torch.all(o[1:] >= o[:-1]).item()) for o in host_out)
    ok = ok and all(bool(torch.equal(torch.sort(i).values, o)) for i, o in zip(host_in, host_out))
    return {"value": n / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": n * 4, "d2h_bytes_per_step": n * 4,
            "ms_per_step": ms, "steps": steps, "sorted_ok": ok,
            "how": "HostPipeline: pinned host batch -> H2D -> pdq_sort -> D2H, three streams overlapping "
                   "consecutive steps"}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
