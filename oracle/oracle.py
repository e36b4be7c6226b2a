"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front-end for oracle/liboracle.so, the plain-C restatement of the
reference sort path (see pdq_oracle.c).  Imported only by tests/,
__graft_entry__.smoke() and bench.py's CPU legs; the product package never
imports it.

The functions mirror the reference's Python signatures so tests read like
the reference's own (pkg/tests/test_driver.py, test_partition.py, ...):

* ``sort(arr, config=None, use_block=True, metrics=False)`` – in-place on a
  numpy array (int32/int64/float32/float64); driver.py:267 / :282.
* ``sort_kv(keys, vals, ...)`` – int64 keys + uint32 payload as tuples.
* primitive wrappers over int64 lists: partition_right, partition_left,
  block_partition_right, choose_pivot, break_patterns, insertion_sort,
  unguarded_insertion_sort, partial_insertion_sort, heapsort, sort3.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

METRIC_FIELDS = (
    "comparisons",
    "element_moves",
    "exchanges",
    "partition_right_calls",
    "partition_left_calls",
    "bad_partitions",
    "heapsort_fallbacks",
    "partial_insertion_attempts",
    "partial_insertion_aborts",
    "max_depth",
)

CONFIG_FIELDS = (
    "insertion_threshold",
    "ninther_threshold",
    "partial_insertion_budget",
    "block_size",
    "bad_partition_shift",
    "use_block_partition",
    "use_partition_left",
    "use_break_patterns",
    "use_partial_insertion",
)
DEFAULTS = dict(
    insertion_threshold=24,
    ninther_threshold=128,
    partial_insertion_budget=8,
    block_size=64,
    bad_partition_shift=3,
    use_block_partition=True,
    use_partition_left=True,
    use_break_patterns=True,
    use_partial_insertion=True,
)


class Config(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in CONFIG_FIELDS]


class Metrics(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in METRIC_FIELDS]

    def as_dict(self):
        return {f: getattr(self, f) for f in METRIC_FIELDS}


class PartitionResult(ctypes.Structure):
    _fields_ = [("pivot_index", ctypes.c_int64), ("no_swaps", ctypes.c_int64)]


DTYPE_CODE = {np.dtype(np.int32): 0, np.dtype(np.int64): 1, np.dtype(np.float32): 2, np.dtype(np.float64): 3}

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        _lib.oracle_sort.argtypes = [P, I, I64, ctypes.POINTER(Config), I, ctypes.POINTER(Metrics)]
        _lib.oracle_sort_kv.argtypes = [P, P, I64, ctypes.POINTER(Config), I, ctypes.POINTER(Metrics)]
        _lib.oracle_config_check.argtypes = [ctypes.POINTER(Config)]
        _lib.oracle_is_bad_partition.argtypes = [I64, I64, I64, ctypes.POINTER(Config)]
        for name in ("insertion_sort", "unguarded_insertion_sort", "heapsort"):
            getattr(_lib, "oracle_prim_" + name).argtypes = [P, I64, I64, ctypes.POINTER(Metrics)]
        _lib.oracle_prim_partial_insertion_sort.argtypes = [P, I64, I64, I64, ctypes.POINTER(Metrics)]
        _lib.oracle_prim_sort3.argtypes = [P, I64, I64, I64, ctypes.POINTER(Metrics)]
        for name in ("partition_right", "partition_left"):
            getattr(_lib, "oracle_prim_" + name).argtypes = [
                P, I64, I64, ctypes.POINTER(Metrics), ctypes.POINTER(PartitionResult)]
        _lib.oracle_prim_block_partition_right.argtypes = [
            P, I64, I64, I64, ctypes.POINTER(Metrics), ctypes.POINTER(PartitionResult)]
        for name in ("choose_pivot", "break_patterns"):
            getattr(_lib, "oracle_prim_" + name).argtypes = [
                P, I64, I64, ctypes.POINTER(Config), ctypes.POINTER(Metrics)]
    return _lib


def make_config(**overrides) -> Config:
    vals = dict(DEFAULTS)
    vals.update(overrides)
    return Config(*[int(vals[f]) for f in CONFIG_FIELDS])


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def sort(arr: np.ndarray, config: Config | None = None, use_block: bool = True, metrics: bool = False):
    """In-place oracle sort of a contiguous numpy array (driver.py:282-292)."""
    assert arr.flags.c_contiguous
    cfg = config or make_config()
    m = Metrics() if metrics else None
    rc = lib().oracle_sort(_ptr(arr), DTYPE_CODE[arr.dtype], arr.size, ctypes.byref(cfg),
                           int(bool(use_block) and bool(cfg.use_block_partition)),
                           ctypes.byref(m) if m is not None else None)
    if rc != 0:
        raise TypeError(f"oracle: unsupported dtype {arr.dtype}")
    return m.as_dict() if m is not None else None


def sort_kv(keys: np.ndarray, vals: np.ndarray, config: Config | None = None, use_block: bool = False,
            metrics: bool = False):
    """In-place oracle sort of (int64 key, uint32 payload) tuples.  The
    reference takes the scalar partition for tuples (driver.py:159-164)."""
    assert keys.dtype == np.int64 and vals.dtype == np.uint32 and keys.size == vals.size
    cfg = config or make_config()
    m = Metrics() if metrics else None
    rc = lib().oracle_sort_kv(_ptr(keys), _ptr(vals), keys.size, ctypes.byref(cfg),
                              int(bool(use_block) and bool(cfg.use_block_partition)),
                              ctypes.byref(m) if m is not None else None)
    if rc != 0:
        raise MemoryError("oracle_sort_kv")
    return m.as_dict() if m is not None else None


# ---- primitives over python int lists (returning (new_list, result, metrics)) ------

def _call(name, data, *args, result=False, config=False):
    a = np.array(data, dtype=np.int64)
    m = Metrics()
    extra = list(args)
    if config:
        extra.append(ctypes.byref(config if isinstance(config, Config) else make_config()))
    if result:
        r = PartitionResult()
        getattr(lib(), "oracle_prim_" + name)(_ptr(a), *extra, ctypes.byref(m), ctypes.byref(r))
        return a.tolist(), (r.pivot_index, bool(r.no_swaps)), m.as_dict()
    ret = getattr(lib(), "oracle_prim_" + name)(_ptr(a), *extra, ctypes.byref(m))
    return a.tolist(), ret, m.as_dict()


def partition_right(data, begin=0, end=None):
    return _call("partition_right", data, begin, len(data) if end is None else end, result=True)


def partition_left(data, begin=0, end=None):
    return _call("partition_left", data, begin, len(data) if end is None else end, result=True)


def block_partition_right(data, begin=0, end=None, block_size=64):
    return _call("block_partition_right", data, begin, len(data) if end is None else end, block_size,
                 result=True)


def choose_pivot(data, begin=0, end=None, config=None):
    return _call("choose_pivot", data, begin, len(data) if end is None else end, config=config or True)


def break_patterns(data, begin=0, end=None, config=None):
    return _call("break_patterns", data, begin, len(data) if end is None else end, config=config or True)


def insertion_sort(data, begin=0, end=None):
    return _call("insertion_sort", data, begin, len(data) if end is None else end)


def unguarded_insertion_sort(data, begin, end=None):
    return _call("unguarded_insertion_sort", data, begin, len(data) if end is None else end)


def partial_insertion_sort(data, begin=0, end=None, budget=8):
    out, ret, m = _call("partial_insertion_sort", data, begin, len(data) if end is None else end, budget)
    return out, bool(ret), m


def heapsort(data, begin=0, end=None):
    return _call("heapsort", data, begin, len(data) if end is None else end)


def sort3(data, a, b, c):
    return _call("sort3", data, a, b, c)


def is_bad_partition(left, right, total, config=None):
    return bool(lib().oracle_is_bad_partition(left, right, total, ctypes.byref(config or make_config())))


def config_check(**overrides) -> int:
    return lib().oracle_config_check(ctypes.byref(make_config(**overrides)))
