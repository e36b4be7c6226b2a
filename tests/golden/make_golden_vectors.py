"""Generate tests/golden/vectors.json by running the Python REFERENCE
(/root/reference/pkg/src/pdqsort, imported read-only) on small seeded inputs.

Each record stores the input, the reference's exact output permutation, its
return value and the reference's own instrumentation counters
(Metrics, instrumentation.py:20-61, with counting_ordering :69-76).  The C
oracle (oracle/pdq_oracle.c) must reproduce every record exactly; the
counters only agree if the restatement executes the same comparisons and
moves as the reference, step for step.

Run here (needs /root/reference):  python tests/golden/make_golden_vectors.py
"""

from __future__ import annotations

import hashlib
import json
import operator
import os
import random
import sys
from dataclasses import replace

sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import pdqsort  # noqa: E402
from pdqsort import (  # noqa: E402
    DEFAULT_CONFIG,
    BlockBuffers,
    Metrics,
    SortConfig,
    counting_ordering,
    instrumented_sort,
)
from pdqsort.instrumentation import adversary_input  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
TOGGLES = ("use_block_partition", "use_partition_left", "use_break_patterns", "use_partial_insertion")


def mdict(m: Metrics) -> dict:
    return {k: v for k, v in zip(pdqsort.METRIC_FIELDS, m.counter_values())}


def prepare_pivot(arr):
    # pkg/tests/test_partition.py:21-29
    work = list(arr)
    if len(work) == 2:
        if work[1] < work[0]:
            work[0], work[1] = work[1], work[0]
    else:
        pdqsort.sort3(work, len(work) // 2, 0, len(work) - 1)
    return work


def prim(rng):
    out = []

    def rec(kind, inp, res, work, m, **kw):
        d = {"kind": kind, "input": inp, "output": work, "result": res, "metrics": mdict(m)}
        d.update(kw)
        out.append(d)

    for _ in range(120):
        n = rng.randint(2, 70)
        hi = rng.choice([3, 10, 1000])
        arr = prepare_pivot([rng.randint(0, hi) for _ in range(n)])
        b, e = 0, n
        if rng.random() < 0.2 and n > 6:  # subrange with untouched borders
            b, e = 1, n - 1
            arr[b:e] = prepare_pivot(arr[b:e])
        work, m = list(arr), Metrics()
        r = pdqsort.partition_right(work, b, e, counting_ordering(operator.lt, m), m)
        rec("partition_right", arr, [r.pivot_index, r.no_swaps], work, m, begin=b, end=e)
        for bs in (1, 2, 3, 8, 64):
            work, m = list(arr), Metrics()
            r = pdqsort.block_partition_right(work, b, e, counting_ordering(operator.lt, m),
                                              BlockBuffers.for_block_size(bs), m)
            rec("block_partition_right", arr, [r.pivot_index, r.no_swaps], work, m, begin=b, end=e,
                block_size=bs)
        larr = list(arr)
        larr[b] = min(larr[b:e])
        work, m = list(larr), Metrics()
        r = pdqsort.partition_left(work, b, e, counting_ordering(operator.lt, m), m)
        rec("partition_left", larr, [r.pivot_index, r.no_swaps], work, m, begin=b, end=e)
    for n in list(range(3, 20)) + [127, 128, 129, 130, 200, 301]:
        arr = [rng.randint(0, 50) for _ in range(n)]
        for cfg in (DEFAULT_CONFIG, SortConfig(insertion_threshold=3, ninther_threshold=8)):
            work, m = list(arr), Metrics()
            pdqsort.choose_pivot(work, 0, n, counting_ordering(operator.lt, m), cfg, m)
            rec("choose_pivot", arr, None, work, m, begin=0, end=n, ninther_threshold=cfg.ninther_threshold)
    for n in (8, 9, 16, 100, 128, 129, 200, 500):
        arr = [rng.randint(0, 99) for _ in range(n)]
        work, m = list(arr), Metrics()
        pdqsort.break_patterns(work, 0, n, DEFAULT_CONFIG, m)
        rec("break_patterns", arr, None, work, m, begin=0, end=n, ninther_threshold=128)
    for _ in range(60):
        n = rng.randint(0, 60)
        arr = [rng.randint(0, 20) for _ in range(n)]
        work, m = list(arr), Metrics()
        pdqsort.insertion_sort(work, 0, n, counting_ordering(operator.lt, m), m)
        rec("insertion_sort", arr, None, work, m, begin=0, end=n)
        garr = [-1] + arr
        work, m = list(garr), Metrics()
        pdqsort.unguarded_insertion_sort(work, 1, n + 1, counting_ordering(operator.lt, m), m)
        rec("unguarded_insertion_sort", garr, None, work, m, begin=1, end=n + 1)
        for budget in (0, 1, 3, 8):
            near = sorted(arr)
            for _ in range(rng.randint(0, 4)):
                if n > 1:
                    i, j = rng.randrange(n), rng.randrange(n)
                    near[i], near[j] = near[j], near[i]
            work, m = list(near), Metrics()
            ok = pdqsort.partial_insertion_sort(work, 0, n, counting_ordering(operator.lt, m), budget, m)
            rec("partial_insertion_sort", near, ok, work, m, begin=0, end=n, budget=budget)
        work, m = list(arr), Metrics()
        pdqsort.heapsort(work, 0, n, counting_ordering(operator.lt, m), m)
        rec("heapsort", arr, None, work, m, begin=0, end=n)
    for trip in [(1, 2, 3), (3, 2, 1), (2, 3, 1), (1, 1, 0), (5, 5, 5), (2, 1, 3)]:
        for perm in ((0, 1, 2), (1, 0, 2), (2, 0, 1)):
            work, m = list(trip), Metrics()
            pdqsort.sort3(work, *perm, counting_ordering(operator.lt, m), m)
            rec("sort3", list(trip), None, work, m, abc=list(perm))
    return out


def full(rng):
    out = []

    def run(name, arr, lt_kind, cfg, branch_cheap):
        work = list(arr)
        m = instrumented_sort(work, operator.lt, cfg, branch_cheap=branch_cheap)
        assert work == sorted(arr)
        d = {
            "kind": "sort",
            "name": name,
            "elem": lt_kind,
            "config": {f: getattr(cfg, f) for f in (
                "insertion_threshold", "ninther_threshold", "partial_insertion_budget", "block_size",
                "bad_partition_shift") + TOGGLES},
            "use_block": bool(cfg.use_block_partition and branch_cheap),
            "metrics": mdict(m),
        }
        if lt_kind == "kv":
            d["keys"] = [p[0] for p in arr]
            d["vals"] = [p[1] for p in arr]
            d["out_keys"] = [p[0] for p in work]
            d["out_vals"] = [p[1] for p in work]
        else:
            d["input"] = arr
            d["output"] = work
        out.append(d)

    def shapes(n):
        half = (n + 1) // 2
        return {
            "uniform": [rng.randint(-2**31, 2**31 - 1) for _ in range(n)],
            "dups": [rng.randint(0, max(1, n // 16)) for _ in range(n)],
            "k3": [rng.choice([-5, 0, 9]) for _ in range(n)],
            "asc": list(range(n)),
            "desc": list(range(n - 1, -1, -1)),
            "organ": list(range(half)) + list(range(n - half - 1, -1, -1)),
            "ones": [1] * n,
            "asc_tail": list(range(n - n // 10)) + [rng.randint(0, n) for _ in range(n // 10)],
        }

    for n in (0, 1, 2, 3, 23, 24, 25, 100, 129, 1000, 3000):
        for sname, arr in shapes(n).items():
            run(f"{sname}.{n}", arr, "int", DEFAULT_CONFIG, True)        # list -> block path
            run(f"{sname}.{n}.scalar", arr, "int", DEFAULT_CONFIG, False)  # numpy/tuple -> scalar path
    # all 16 toggle combinations (pkg/tests/test_driver.py:223-231)
    import itertools
    for bits in itertools.product((False, True), repeat=4):
        cfg = replace(DEFAULT_CONFIG, **dict(zip(TOGGLES, bits)))
        arr = [rng.randint(-9, 9) for _ in range(400)]
        run("toggles." + "".join(str(int(b)) for b in bits), arr, "int", cfg, True)
    cfg = SortConfig(insertion_threshold=3, ninther_threshold=8, block_size=2)
    run("small_thresholds", [rng.randint(0, 6) for _ in range(120)], "int", cfg, True)
    # floats incl. +-inf (test_driver.py:250-254); float32-representable values
    fl = [float(np.float32(rng.gauss(0, 1))) for _ in range(2000)] + [float("inf"), float("-inf")] * 3
    run("floats", fl, "float", DEFAULT_CONFIG, True)
    # KV tuples: lexicographic, scalar partition (tuples are not branch-cheap)
    kv = [(rng.randint(0, 50), rng.randint(0, 2**32 - 1)) for _ in range(3000)]
    run("kv_dupkeys", kv, "kv", DEFAULT_CONFIG, False)
    kv = [(rng.randint(-2**62, 2**62), i) for i in range(2000)]
    run("kv_distinct", kv, "kv", DEFAULT_CONFIG, False)
    # adversary input drives the scalar kernels into the heapsort fallback
    # (instrumentation.py:112-155, test_instrumentation.py:93-101)
    for n in (256, 2048):
        cfg = replace(DEFAULT_CONFIG, use_block_partition=False)
        run(f"adversary.{n}", adversary_input(n, cfg), "int", cfg, False)
    return out


def main():
    rng = random.Random(210605123)
    data = {"generator": "tests/golden/make_golden_vectors.py", "reference": "pkg/src/pdqsort @ /root/reference",
            "primitives": prim(rng), "sorts": full(rng)}
    path = os.path.join(HERE, "vectors.json")
    with open(path, "w") as f:
        json.dump(data, f, separators=(",", ":"))
    h = hashlib.sha256(open(path, "rb").read()).hexdigest()
    print(path, os.path.getsize(path), "bytes", h)


if __name__ == "__main__":
    main()
