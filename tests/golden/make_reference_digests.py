"""Run the UNMODIFIED Python reference (pdqsort.sort, pkg/src/pdqsort/driver.py:267-270)
on the seeded BASELINE configs and record sha256 digests of its outputs.

This is how the committed ``reference_digests.jsonl`` was produced, in the
build container where ``/root/reference`` exists.  The GPU box never runs
this script (it has no /root/reference); the GPU parity tests regenerate the
same inputs from ``paper_2106_05123_b200.workloads`` and compare digests.

Usage:  python tests/golden/make_reference_digests.py CASE [SHIFT]
        (CASE as in workloads.cases(); SHIFT right-shifts the config size)
Appends one JSON line per run to tests/golden/reference_digests.jsonl.
"""

from __future__ import annotations

import fcntl
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import pdqsort  # noqa: E402  (the reference, imported read-only)
from paper_2106_05123_b200 import workloads  # noqa: E402


def digest(keys: np.ndarray, values=None) -> str:
    h = hashlib.sha256(np.ascontiguousarray(keys).tobytes())
    if values is not None:
        h.update(np.ascontiguousarray(values).tobytes())
    return h.hexdigest()


def main():
    name = sys.argv[1]
    shift = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    base = name.split(".")[0]
    n = max(workloads.FULL_N[base] >> shift, 1)
    keys, vals = workloads.make(name, n)
    if vals is None:
        work = keys.tolist()
        t0 = time.perf_counter_ns()
        pdqsort.sort(work)  # driver.py:267
        t1 = time.perf_counter_ns()
        out_k, out_v = np.array(work, dtype=keys.dtype), None
    else:
        work = list(zip(keys.tolist(), vals.tolist()))
        t0 = time.perf_counter_ns()
        pdqsort.sort(work)  # tuples: lexicographic (key, payload), scalar partition_right path
        t1 = time.perf_counter_ns()
        out_k = np.fromiter((p[0] for p in work), dtype=keys.dtype, count=n)
        out_v = np.fromiter((p[1] for p in work), dtype=vals.dtype, count=n)
    exp_k, exp_v = workloads.expected(keys, vals)
    equal = bool(np.array_equal(out_k, exp_k) and (vals is None or np.array_equal(out_v, exp_v)))
    rec = {
        "case": name,
        "n": n,
        "dtype": str(keys.dtype),
        "payload": None if vals is None else str(vals.dtype),
        "input_sha256": digest(keys, vals),
        "output_sha256": digest(out_k, out_v),
        "equals_numpy_expected": equal,
        "reference_seconds": (t1 - t0) / 1e9,
        "host": f"1 thread of {os.cpu_count()} cores, python {sys.version.split()[0]}",
    }
    line = json.dumps(rec)
    print(line)
    with open(os.path.join(HERE, "reference_digests.jsonl"), "a") as f:
        fcntl.flock(f, fcntl.LOCK_EX)
        f.write(line + "\n")


if __name__ == "__main__":
    main()
