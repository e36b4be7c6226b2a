"""Pin the C oracle (oracle/pdq_oracle.c) to the Python reference.

Every record in tests/golden/vectors.json was produced by running the
reference itself (tests/golden/make_golden_vectors.py).  The oracle must
reproduce the exact output permutation, the return value and all ten
instrumentation counters (instrumentation.py:20-61) for each of them.
"""

import json
import os

import numpy as np
import pytest

from oracle import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "vectors.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def _metrics_subset(ref, got):
    return {k: got[k] for k in ref}


def test_primitives_match_reference(golden):
    seen = set()
    for rec in golden["primitives"]:
        kind, inp = rec["kind"], rec["input"]
        b, e = rec.get("begin"), rec.get("end")
        if kind == "partition_right":
            out, res, m = oracle.partition_right(inp, b, e)
            assert [res[0], res[1]] == rec["result"]
        elif kind == "block_partition_right":
            out, res, m = oracle.block_partition_right(inp, b, e, rec["block_size"])
            assert [res[0], res[1]] == rec["result"]
        elif kind == "partition_left":
            out, res, m = oracle.partition_left(inp, b, e)
            assert [res[0], res[1]] == rec["result"]
        elif kind == "choose_pivot":
            cfg = oracle.make_config(insertion_threshold=3 if rec["ninther_threshold"] == 8 else 24,
                                     ninther_threshold=rec["ninther_threshold"])
            out, _, m = oracle.choose_pivot(inp, b, e, cfg)
        elif kind == "break_patterns":
            out, _, m = oracle.break_patterns(inp, b, e)
        elif kind == "insertion_sort":
            out, _, m = oracle.insertion_sort(inp, b, e)
        elif kind == "unguarded_insertion_sort":
            out, _, m = oracle.unguarded_insertion_sort(inp, b, e)
        elif kind == "partial_insertion_sort":
            out, ok, m = oracle.partial_insertion_sort(inp, b, e, rec["budget"])
            assert ok == rec["result"]
        elif kind == "heapsort":
            out, _, m = oracle.heapsort(inp, b, e)
        elif kind == "sort3":
            out, _, m = oracle.sort3(inp, *rec["abc"])
        else:
            raise AssertionError(kind)
        assert out == rec["output"], (kind, inp)
        if kind != "break_patterns":  # reference break_patterns takes no ordering
            assert m["comparisons"] == rec["metrics"]["comparisons"], (kind, inp)
        assert _metrics_subset(rec["metrics"], m) == rec["metrics"] or kind == "break_patterns", (kind, inp)
        assert m["exchanges"] == rec["metrics"]["exchanges"]
        assert m["element_moves"] == rec["metrics"]["element_moves"]
        seen.add(kind)
    assert len(seen) == 10


def test_full_sorts_match_reference(golden):
    for rec in golden["sorts"]:
        cfg = oracle.make_config(**rec["config"])
        if rec["elem"] == "kv":
            k = np.array(rec["keys"], dtype=np.int64)
            v = np.array(rec["vals"], dtype=np.uint32)
            m = oracle.sort_kv(k, v, cfg, use_block=rec["use_block"], metrics=True)
            assert k.tolist() == rec["out_keys"] and v.tolist() == rec["out_vals"], rec["name"]
        else:
            dt = np.float64 if rec["elem"] == "float" else np.int64
            a = np.array(rec["input"], dtype=dt)
            m = oracle.sort(a, cfg, use_block=rec["use_block"], metrics=True)
            assert a.tolist() == rec["output"], rec["name"]
        assert m == rec["metrics"], rec["name"]


def test_float32_path_matches_float64_path(golden):
    rec = next(r for r in golden["sorts"] if r["name"] == "floats")
    a32 = np.array(rec["input"], dtype=np.float32)
    m = oracle.sort(a32, use_block=True, metrics=True)
    assert a32.astype(np.float64).tolist() == rec["output"]
    assert m == rec["metrics"]


def test_int32_path_matches_int64_path(golden):
    for rec in golden["sorts"]:
        if rec["elem"] != "int" or not rec["input"] or max(map(abs, rec["input"])) >= 2**31 - 1:
            continue
        a = np.array(rec["input"], dtype=np.int32)
        m = oracle.sort(a, oracle.make_config(**rec["config"]), use_block=rec["use_block"], metrics=True)
        assert a.tolist() == rec["output"] and m == rec["metrics"], rec["name"]


# ---- the reference's own known-answer tests, restated against the oracle ---------

def test_kat_partition_swapless_trace():
    # pkg/tests/test_partition.py:49-54
    out, (pi, ns), _ = oracle.partition_right([5, 1, 2, 7, 9])
    assert out == [2, 1, 5, 7, 9] and pi == 2 and ns is True


def test_kat_partition_left_examples():
    # pkg/tests/test_partition.py:80-95
    out, (pi, _), _ = oracle.partition_left([2, 2, 3])
    assert pi == 1 and out[:2] == [2, 2] and out[2] == 3
    assert oracle.partition_left([4, 4, 4, 4])[1][0] == 3
    out, (pi, ns), _ = oracle.partition_left([5, 7, 5, 6, 5])
    assert pi == 2 and sorted(out[:3]) == [5, 5, 5] and sorted(out[3:]) == [6, 7] and ns is False


def test_kat_choose_pivot_median_of_three():
    # pkg/tests/test_driver.py:67-72
    assert oracle.choose_pivot([1, 2, 3])[0] == [2, 1, 3]


def test_kat_is_bad_partition():
    # pkg/tests/test_driver.py:107-123
    assert oracle.is_bad_partition(7, 56, 64) is True
    assert oracle.is_bad_partition(8, 55, 64) is False
    assert oracle.is_bad_partition(32, 31, 64) is False
    cfg = oracle.make_config(bad_partition_shift=1)
    assert oracle.is_bad_partition(31, 32, 64, cfg) is True
    assert oracle.is_bad_partition(32, 32, 65, cfg) is False


def test_kat_break_patterns_positions():
    # pkg/tests/test_driver.py:133-137
    out, _, _ = oracle.break_patterns(list(range(16)))
    assert out[0] == 4 and out[15] == 11


def test_kat_reversed_five_insertion_counts():
    # pkg/tests/test_small_sorts.py:56-65: 10 comparisons, 18 moves
    out, _, m = oracle.insertion_sort([5, 4, 3, 2, 1])
    assert out == [1, 2, 3, 4, 5] and m["comparisons"] == 10 and m["element_moves"] == 18


def test_config_validation_rules():
    # driver.py:65-75 / pkg/tests/test_driver.py:51-64
    assert oracle.config_check() == 0
    for kw in ({"insertion_threshold": 2}, {"ninther_threshold": 7},
               {"insertion_threshold": 40, "ninther_threshold": 39}, {"block_size": 0},
               {"bad_partition_shift": 0}, {"partial_insertion_budget": -1}):
        assert oracle.config_check(**kw) != 0


def test_all_equal_single_partition_left():
    # pkg/tests/test_driver.py:176-182
    a = np.ones(4096, dtype=np.int64)
    m = oracle.sort(a, metrics=True)
    assert m["partition_left_calls"] == 1 and m["comparisons"] <= 8 * 4096


def test_ascending_linear():
    # pkg/tests/test_driver.py:171-174
    n = 1 << 14
    a = np.arange(n, dtype=np.int64)
    m = oracle.sort(a, metrics=True)
    assert m["comparisons"] <= 6 * n
