"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/pdq_b200.h declares; host logic mirrors driver.py.  No kernel
is launched here (no GPU in the build container)."""

import ctypes
import operator
import os
import re

import numpy as np
import pytest

from paper_2106_05123_b200 import DEFAULT_CONFIG, SortConfig, _lib, is_bad_partition, sort_with_config, workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "pdq_b200.h")).read()
    return set(re.findall(r"\b(pdq_[a-z_]+)\s*\(", src))


def test_header_declares_exactly_the_bound_symbols():
    assert header_symbols() == set(_lib.EXPORTS)


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    for name in header_symbols():
        assert hasattr(L, name), name
    assert b"sm_100a" in L.pdq_version()


def test_library_is_sm100a_code():
    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_config_struct_layout_and_defaults():
    L = _lib.lib()
    c = _lib.PdqConfig()
    L.pdq_config_default(ctypes.byref(c))
    assert (c.insertion_threshold, c.ninther_threshold, c.partial_insertion_budget, c.block_size,
            c.bad_partition_shift) == (24, 128, 8, 64, 3)  # driver.py:55-59
    assert c.base_case_size == 32768 and c.bad_budget == -1
    assert ctypes.sizeof(_lib.PdqConfig) == 5 * 8 + 6 * 4 + 4 * 4
    mine = DEFAULT_CONFIG.to_c()
    assert bytes(mine) == bytes(c)
    assert L.pdq_config_validate(ctypes.byref(c)) == 0
    # GPU fields: two_run_min travels in reserved[1] (0 = the library default); out-of-range values raise
    assert SortConfig(two_run_min=64).to_c().reserved[1] == 64 and mine.reserved[1] == 0
    for bad in (-1, 2**31):
        with pytest.raises(ValueError):
            SortConfig(two_run_min=bad)


@pytest.mark.parametrize("kw", [
    {"insertion_threshold": 2}, {"ninther_threshold": 7}, {"insertion_threshold": 40, "ninther_threshold": 39},
    {"block_size": 0}, {"bad_partition_shift": 0}, {"partial_insertion_budget": -1},
])
def test_config_validation_matches_reference(kw):
    # pkg/tests/test_driver.py:51-64 — Python raises ValueError, the C ABI returns PDQ_ERR_CONFIG
    with pytest.raises(ValueError):
        SortConfig(**kw)
    base = {f: getattr(DEFAULT_CONFIG, f) for f in DEFAULT_CONFIG.__dataclass_fields__}
    c = _lib.PdqConfig()
    _lib.lib().pdq_config_default(ctypes.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    assert _lib.lib().pdq_config_validate(ctypes.byref(c)) == -1
    assert base


def test_abi_argument_errors_without_gpu():
    L = _lib.lib()
    c = DEFAULT_CONFIG.to_c()
    # bad dtype / negative n / misaligned keys are rejected before touching the device
    assert L.pdq_sort(None, 9, None, 10, ctypes.byref(c), None, 0, None) == -2
    assert L.pdq_sort(None, 0, None, -1, ctypes.byref(c), None, 0, None) == -7
    assert L.pdq_sort(ctypes.c_void_p(0x1004), 0, None, 10, ctypes.byref(c), None, 0, None) == -3
    assert L.pdq_sort(ctypes.c_void_p(0x1000), 0, None, 10, ctypes.byref(c), None, 0, None) == -4
    assert "workspace" in _lib.last_error()


def test_workspace_bytes_monotone_and_covers_scratch():
    L = _lib.lib()
    for code, w in ((0, 4), (1, 8), (2, 4), (3, 8)):
        prev = 0
        for n in (0, 1, 1000, 1 << 20, 1 << 28):
            b = L.pdq_workspace_bytes(code, 0, n)
            assert b >= n * w and b >= prev
            prev = b
        assert L.pdq_workspace_bytes(code, 1, 1 << 20) >= L.pdq_workspace_bytes(code, 0, 1 << 20) + 4 * (1 << 20)
    assert L.pdq_workspace_bytes(7, 0, 10) == 0
    # 2^28 int32: scratch 1 GiB + small metadata
    assert L.pdq_workspace_bytes(0, 0, 1 << 28) < (1 << 30) * 1.1


def test_is_bad_partition_matches_reference_kats():
    # pkg/tests/test_driver.py:107-123
    assert is_bad_partition(7, 56, 64) is True
    assert is_bad_partition(8, 55, 64) is False
    assert is_bad_partition(32, 31, 64) is False
    cfg = SortConfig(bad_partition_shift=1)
    assert is_bad_partition(31, 32, 64, cfg) is True
    assert is_bad_partition(32, 32, 65, cfg) is False


def test_custom_ordering_is_rejected_not_emulated():
    with pytest.raises(NotImplementedError):
        sort_with_config([3, 1, 2], lambda a, b: b < a, DEFAULT_CONFIG)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        sort_with_config([3, 1, 2], operator.lt, DEFAULT_CONFIG)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2106_05123_b200")
    pat = re.compile(r"(^\s*(from|import)\s+oracle\b)|liboracle|oracle\.py", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not pat.search(src), f


def test_workload_generators_are_deterministic():
    a = workloads.c1(1000)
    b = workloads.c1(1000)
    assert a.dtype == np.int32 and np.array_equal(a, b)
    k, v = workloads.c5(4096)
    assert np.unique(k).size == 4096 and v.dtype == np.uint32
    assert workloads.c2("organ", 10).tolist() == [0, 1, 2, 3, 4, 4, 3, 2, 1, 0]  # datagen.py:121-123
    x = workloads.c4("normal", 1 << 16)
    assert not np.isnan(x).any() and not np.any((x == 0) & np.signbit(x))
    for k_ in workloads.C3_KS[:4]:
        assert np.unique(workloads.c3(k_, 1 << 16)).size <= k_


def test_field_ordering_is_a_plain_comparator():
    # by_field(i) works as the reference's lambda orderings do (test_driver.py:198-204)
    from paper_2106_05123_b200 import by_field

    lt = by_field(0)
    assert lt((1, "b"), (2, "a")) and not lt((2, "a"), (1, "b")) and not lt((1, "x"), (1, "y"))
    gt = by_field(1, descending=True)
    assert gt((0, 5), (0, 3)) and not gt((0, 3), (0, 5))
    assert by_field("w")({"w": 1.0}, {"w": 2.0})
    with pytest.raises(RuntimeError):  # the device path is the only path
        sort_with_config([(2, 0), (1, 1)], lt, DEFAULT_CONFIG)


def test_list_keys_outside_int64_are_rejected():
    from paper_2106_05123_b200 import sort

    with pytest.raises(TypeError):
        sort([2**70, 1])
    with pytest.raises(TypeError):
        sort([1, "a"])


def test_tuple_elements_are_type_checked_before_conversion():
    # float payloads / mixed keys in (key, payload) tuples must raise, never be
    # truncated and written back
    from paper_2106_05123_b200 import sort

    cases = [
        [(1, 0.5), (2, 1)],          # float payload
        [(1, 2), (2.5, 1)],          # mixed int/float keys
        [(1, "7"), (0, 1)],          # string payload
        [("3", 1), (2, 0)],          # string key
        [(1, -1), (0, 1)],           # negative payload
    ]
    for c in cases:
        w = list(c)
        with pytest.raises(TypeError):
            sort(w)
        assert w == c  # untouched


def test_uint64_field_beyond_int64_is_rejected():
    # a uint64 field value >= 2^63 would wrap negative as an int64 key
    from paper_2106_05123_b200 import by_field, sort_with

    rec = np.zeros(2, dtype=[("k", np.uint64), ("v", np.int32)])
    rec["k"] = [2**63 + 1, 5]
    with pytest.raises(TypeError):
        sort_with(rec, by_field("k"))


def test_metrics_columns_follow_the_reference():
    # instrumentation.py:20-31: the CSV counter fragment's column order
    from paper_2106_05123_b200 import Metrics
    from paper_2106_05123_b200.driver import METRIC_FIELDS

    assert METRIC_FIELDS == ("comparisons", "element_moves", "exchanges", "partition_right_calls",
                             "partition_left_calls", "bad_partitions", "heapsort_fallbacks",
                             "partial_insertion_attempts", "partial_insertion_aborts", "max_depth")
    m = Metrics.from_stats({"partition_right_calls": 3, "partition_left_calls": 1, "bad_partitions": 2,
                            "radix_fallbacks": 1, "max_depth": 5})
    assert m.counter_values() == (0, 0, 0, 3, 1, 2, 1, 0, 0, 5)


def test_stratified_adversary_is_a_permutation():
    from paper_2106_05123_b200 import workloads

    for n in (1000, 1 << 20):
        a = workloads.stratified_adversary(n)
        assert a.dtype == np.int32 and np.array_equal(np.sort(a), np.arange(n))
        ns = 256 if n >= 1 << 20 else 64
        pos = ((2 * np.arange(ns) + 1) * n) // (2 * ns)
        assert np.array_equal(np.sort(a[pos]), np.arange(ns))
