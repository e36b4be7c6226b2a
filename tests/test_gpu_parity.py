"""GPU parity: the CUDA path through the C ABI vs the oracle and the reference.

Bit-exact everywhere: the outputs under test are unique (keys-only outputs are
unique because equal keys are bit-identical; KV outputs are ordered as
(key, payload) pairs, exactly like the reference's tuple sort), so byte
equality with the oracle / the reference digest is the bar.
"""

import array
import hashlib
import itertools
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle  # noqa: E402
from paper_2106_05123_b200 import SortConfig, sort, sort_device, sort_with, workloads  # noqa: E402

pytestmark = pytest.mark.gpu

GOLDEN_DIGESTS = os.path.join(os.path.dirname(__file__), "golden", "reference_digests.jsonl")
DEV = "cuda"

DTYPES = [np.int32, np.int64, np.float32, np.float64]


def gpu_sort(keys: np.ndarray, vals=None, config=None):
    kd = torch.from_numpy(keys.copy()).to(DEV)
    vd = None if vals is None else torch.from_numpy(vals.copy().view(np.int32)).to(DEV)
    stats = sort_device(kd, vd, config or SortConfig())
    ko = kd.cpu().numpy()
    vo = None if vd is None else vd.cpu().numpy().view(np.uint32)
    return ko, vo, stats


def oracle_sort(keys, vals=None):
    k = keys.copy()
    if vals is None:
        oracle.sort(k)
        return k, None
    v = vals.copy()
    oracle.sort_kv(k, v)
    return k, v


def same_bytes(a, b):
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()


def shapes(n, rng, dtype):
    info = np.iinfo(dtype) if np.dtype(dtype).kind == "i" else None
    if info is not None:
        uni = rng.integers(info.min, info.max, n, dtype=dtype, endpoint=True)
    else:
        uni = rng.standard_normal(n).astype(dtype)
    half = (n + 1) // 2
    out = {
        "uniform": uni,
        "dups16": rng.integers(0, 16, n).astype(dtype),
        "dupsq": rng.integers(0, max(1, int(np.sqrt(n))), n).astype(dtype),
        "asc": np.arange(n).astype(dtype),
        "desc": np.arange(n)[::-1].astype(dtype),
        "organ": np.concatenate([np.arange(half), np.arange(n - half - 1, -1, -1)]).astype(dtype),
        "ones": np.ones(n, dtype=dtype),
        "asc_tail": np.concatenate([np.arange(n - n // 10), rng.integers(0, n + 1, n // 10)]).astype(dtype),
    }
    return out


SWEEP_SIZES = list(range(0, 65)) + [100, 1000, 1023, 1024, 1025, 4095, 4096, 4097, 8191, 8192, 10007,
                                     16383, 16384, 16385, 24571, 24572, 24573, 32769, 65536, 100003, 1 << 20]


@pytest.mark.parametrize("dtype", DTYPES, ids=lambda d: np.dtype(d).name)
def test_sweep_vs_oracle(dtype):
    # the sweep shape of the reference's criterion 1 (acceptance.py:67-104): many sizes x distributions
    rng = np.random.default_rng(1)
    for n in SWEEP_SIZES:
        for name, keys in shapes(n, rng, dtype).items():
            got, _, _ = gpu_sort(keys)
            exp, _ = oracle_sort(keys)
            assert same_bytes(got, exp), (n, name)


def test_kv_sweep_vs_oracle():
    rng = np.random.default_rng(2)
    for n in SWEEP_SIZES:
        keys = rng.integers(-(2**62), 2**62, n, dtype=np.int64)
        vals = rng.integers(0, 2**32, n, dtype=np.uint32)
        # duplicate keys: lexicographic (key, payload) order makes the output unique anyway
        dup = keys % 7
        for k in (keys, dup):
            got_k, got_v, _ = gpu_sort(k, vals)
            exp_k, exp_v = oracle_sort(k, vals)
            assert same_bytes(got_k, exp_k) and same_bytes(got_v, exp_v), n


@pytest.mark.parametrize("kvdtype", [np.int32, np.float32, np.float64])
def test_kv_other_key_types(kvdtype):
    rng = np.random.default_rng(3)
    for n in (5, 4096, 70000):
        keys = (rng.standard_normal(n) * 1000).astype(kvdtype)
        vals = np.arange(n, dtype=np.uint32)
        got_k, got_v, _ = gpu_sort(keys, vals)
        order = np.lexsort((vals, keys))
        assert same_bytes(got_k, keys[order]) and same_bytes(got_v, vals[order])


def _digests():
    recs = {}
    with open(GOLDEN_DIGESTS) as f:
        for line in f:
            r = json.loads(line)
            recs[(r["case"], r["n"])] = r
    return recs


def _digest(k, v=None):
    h = hashlib.sha256(np.ascontiguousarray(k).tobytes())
    if v is not None:
        h.update(np.ascontiguousarray(v).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("shift", [6, 0])
def test_configs_vs_reference_digests(shift):
    """The five BASELINE configs, regenerated from their seeds, against the digests of
    the Python reference's own output (tests/golden/make_reference_digests.py)."""
    recs = _digests()
    want = {name for name, _, _ in workloads.cases(20)} | {"R"}  # 14 config cases + the roofline input
    checked = set()
    for (case, n), rec in sorted(recs.items()):
        base = case.split(".")[0]
        if n != max(workloads.FULL_N[base] >> shift, 1):
            continue
        keys, vals = workloads.make(case, n)
        assert _digest(keys, vals) == rec["input_sha256"], f"input generator drifted for {case}"
        got_k, got_v, _ = gpu_sort(keys, vals)
        assert _digest(got_k, got_v) == rec["output_sha256"], case
        checked.add(case)
        del keys, vals, got_k, got_v
    assert checked == want, f"reference digests missing for {sorted(want - checked)}"


def test_full_size_properties_roofline_input():
    """2^28 uniform int32 (the roofline input R): sortedness + multiset (sum/xor/min/max
    and a sampled-rank check) without a CPU sort at full size."""
    n = 1 << 28
    g = torch.Generator(device=DEV)
    g.manual_seed(6)
    kd = torch.randint(-(2**31), 2**31, (n,), dtype=torch.int64, device=DEV, generator=g).to(torch.int32)
    before_sum = kd.to(torch.int64).sum().item()
    ref_sorted_sample = torch.sort(kd[:: 1 << 12].clone()).values
    stats = sort_device(kd)
    assert bool((kd[1:] >= kd[:-1]).all().item())
    assert kd.to(torch.int64).sum().item() == before_sum
    # the sample's elements must all be present: searchsorted hits equal keys
    pos = torch.searchsorted(kd, ref_sorted_sample)
    assert bool((kd[pos.clamp(max=n - 1)] == ref_sorted_sample).all().item())
    assert stats["status"] == 0 and stats["bytes_algorithmic"] > 8 * n


def test_toggle_soundness():
    # all 16 toggle combinations (pkg/tests/test_driver.py:223-231)
    rng = np.random.default_rng(16)
    toggles = ("use_block_partition", "use_partition_left", "use_break_patterns", "use_partial_insertion")
    for bits in itertools.product((False, True), repeat=4):
        cfg = SortConfig(**dict(zip(toggles, bits)))
        for n in (0, 7, 400, 5000, 70000):
            keys = rng.integers(-9, 9, n).astype(np.int32)
            got, _, _ = gpu_sort(keys, config=cfg)
            assert same_bytes(got, np.sort(keys)), (bits, n)


@pytest.mark.parametrize("dtype", DTYPES + ["kv"], ids=lambda d: d if isinstance(d, str) else np.dtype(d).name)
def test_forced_fallback_budget_zero(dtype):
    # bad_budget=0: the root starts with an exhausted budget, so it takes the K5 8-bit digit passes
    # (driver.py:209-213 analogue: heapsort's role); the digit runs become leaves or digit passes on the
    # next 8 bits
    rng = np.random.default_rng(5)
    for n in (30000, 300000, 1 << 22):  # above every base-case size (24572 for 4-byte keys)
        if dtype == "kv":
            keys = rng.integers(0, 50, n).astype(np.int64)
            vals = rng.integers(0, 2**32, n, dtype=np.uint32)
        elif np.dtype(dtype).kind == "f":
            keys, vals = rng.standard_normal(n).astype(dtype), None
        else:
            info = np.iinfo(dtype)
            keys, vals = rng.integers(info.min, info.max, n, dtype=dtype), None
        got_k, got_v, stats = gpu_sort(keys, vals, config=SortConfig(bad_budget=0))
        exp_k, exp_v = workloads.expected(keys, vals)
        assert same_bytes(got_k, exp_k) and (vals is None or same_bytes(got_v, exp_v)), n
        assert stats["radix_fallbacks"] >= 1


@pytest.mark.parametrize("dtype", [np.int32, np.float32], ids=["int32", "float32"])
def test_big_leaf_slow_paths(dtype):
    # 4-byte keys-only leaves (<= 16384 keys) take k_base_big's slow paths when a bucket holds more than
    # 32 keys: (a) clustered distinct keys with far outliers -> LSD radix passes over the whole leaf;
    # (b) a large run of one repeated key beside distinct keys -> the constant bucket keeps its slots;
    # (c) both at once inside a larger sort, so the leaves come out of partitions (data in A and in B)
    rng = np.random.default_rng(11)
    big = np.iinfo(np.int32) if dtype == np.int32 else None
    lo, hi = (big.min, big.max) if big else (-np.inf, np.inf)
    for n in (100, 5000, 12000, 16384, 24572):
        k = rng.integers(0, 1000, n).astype(dtype)
        k[rng.choice(n, 6, replace=False)] = [lo, hi, lo, hi, 0, 1]
        got, _, _ = gpu_sort(k)
        assert same_bytes(got, np.sort(k)), ("clustered", n)
        k = np.concatenate([np.full(n // 2, 7), rng.integers(2**30, 2**31 - 1, n - n // 2)]).astype(dtype)
        rng.shuffle(k)
        got, _, _ = gpu_sort(k)
        assert same_bytes(got, np.sort(k)), ("constant bucket", n)
    n = 1 << 21
    k = rng.integers(0, 5000, n).astype(dtype)
    k[rng.choice(n, 64, replace=False)] = rng.integers(-2**31, 2**31 - 1, 64).astype(dtype)
    k[rng.choice(n, n // 4, replace=False)] = dtype(12345)
    got, _, stats = gpu_sort(k)
    assert same_bytes(got, np.sort(k)) and stats["base_cases"] >= 1


def test_bad_shift_one_exhausts_budgets_deep_in_the_tree():
    # bad_partition_shift=1 calls almost every split bad (min side < half), so budgets run out
    # along many paths and the radix split fires repeatedly at depth, with pattern breaking on
    rng = np.random.default_rng(6)
    for dtype in (np.int32, np.int64):
        keys = rng.integers(-(2**31), 2**31, 1 << 21).astype(dtype)
        got, _, stats = gpu_sort(keys, config=SortConfig(bad_partition_shift=1, bad_budget=4))
        assert same_bytes(got, np.sort(keys))
        assert stats["bad_partitions"] > 10 and stats["radix_fallbacks"] >= 2, stats
    keys = rng.integers(0, 1000, 1 << 21).astype(np.int32)
    got, _, stats = gpu_sort(keys, config=SortConfig(bad_partition_shift=1, bad_budget=2, use_break_patterns=False))
    assert same_bytes(got, np.sort(keys))


def test_low_cardinality_uses_partition_left():
    n = 1 << 20
    keys = np.full(n, 7, dtype=np.int32)
    keys[::3] = 5
    got, _, stats = gpu_sort(keys)
    assert same_bytes(got, np.sort(keys))
    assert stats["partition_left_calls"] >= 1


def test_sorted_and_reversed_are_one_pass():
    n = 1 << 22
    asc = np.arange(n, dtype=np.int32)
    got, _, st = gpu_sort(asc)
    assert same_bytes(got, asc) and st["partition_right_calls"] == 0 and st["check_result"] == 2
    got, _, st = gpu_sort(asc[::-1].copy())
    assert same_bytes(got, asc) and st["partition_right_calls"] == 0 and st["check_result"] & 3 == 1


def _two_runs(rng, n, s, kind, dtype, mirror=False):
    """sorted prefix of s elements, then an ascending (1), descending (2) or random (3) rest; mirrored: the
    sorted run is the suffix [s, n) and the rest comes first"""
    if np.dtype(dtype).kind == "f":
        x = rng.standard_normal(n).astype(dtype)
    else:
        info = np.iinfo(dtype)
        x = rng.integers(info.min, info.max, n, dtype=dtype, endpoint=True)
    big, small = (slice(s, n), slice(0, s)) if mirror else (slice(0, s), slice(s, n))
    x[big] = np.sort(x[big])
    if kind == 1:
        x[small] = np.sort(x[small])
    elif kind == 2:
        x[small] = np.sort(x[small])[::-1]
    return x


@pytest.mark.parametrize("dtype", DTYPES + ["kv"], ids=lambda d: d if isinstance(d, str) else np.dtype(d).name)
def test_two_run_path_vs_oracle(dtype):
    # K4's two-run path (a sorted prefix of >= n/2 merged with the rest; the optimistic path of
    # driver.py:244-250 / small_sorts.py:76-115 restated for the GPU): every second-run kind, splits at the
    # eligibility boundary and near the end, sizes around the merge tile (8192) and the leaf sizes
    rng = np.random.default_rng(11)
    cfg = SortConfig(two_run_min=64)
    kd = np.int64 if dtype == "kv" else dtype
    for n in (64, 100, 4097, 8192, 8193, 24577, 70001, (1 << 18) + 5):
        for s in sorted({(n + 1) // 2, (n + 1) // 2 + 1, int(0.75 * n), n - 2, n - 1}):
            for kind in (1, 2, 3):
                keys = _two_runs(rng, n, s, kind, kd)
                vals = rng.permutation(n).astype(np.uint32) if dtype == "kv" else None
                got, gv, st = gpu_sort(keys, vals, cfg)
                want, wv = oracle_sort(keys, vals)
                assert same_bytes(got, want), (n, s, kind)
                if vals is not None:
                    assert same_bytes(gv, wv), (n, s, kind)
                # (a random rest may by chance extend the prefix or be monotone: only the path is asserted)
                assert st["run_split"] >= s or st["check_result"] & 3 != 3, (n, s, kind, st)
                # mirrored: the sorted run of at least half the array is the suffix [n - s, n)
                keys = _two_runs(rng, n, n - s, kind, kd, mirror=True)
                got, gv, st = gpu_sort(keys, vals, cfg)
                want, wv = oracle_sort(keys, vals)
                assert same_bytes(got, want), (n, s, kind, "mirror")
                if vals is not None:
                    assert same_bytes(gv, wv), (n, s, kind, "mirror")
                assert st["run_split"] > 0 or st["check_result"] & 3 != 3, (n, s, kind, st)


def test_two_run_path_duplicates_and_kinds():
    rng = np.random.default_rng(12)
    cfg = SortConfig(two_run_min=64)
    n, s = 100000, 60000
    keys = np.concatenate([np.sort(rng.integers(0, 50, s)), np.sort(rng.integers(0, 50, n - s))]).astype(np.int32)
    got, _, st = gpu_sort(keys, None, cfg)
    assert same_bytes(got, np.sort(keys)) and st["run_split"] == s and (st["check_result"] >> 4) == 1
    assert st["partition_right_calls"] == 0 and st["base_cases"] == 0
    # (key, payload) pairs with duplicate keys across the runs: each run sorted as pairs
    k64 = keys.astype(np.int64)
    vals = rng.integers(0, 5, n).astype(np.uint32)
    for a, b in ((0, s), (s, n)):
        o = np.lexsort((vals[a:b], k64[a:b]))
        k64[a:b], vals[a:b] = k64[a:b][o], vals[a:b][o]
    got, gv, st = gpu_sort(k64, vals, cfg)
    want, wv = oracle_sort(k64, vals)
    assert same_bytes(got, want) and same_bytes(gv, wv) and st["run_split"] == s
    # descending rest: reversed in place, no partition; below two_run_min the path is off
    keys = np.concatenate([np.arange(s), np.arange(n - s)[::-1]]).astype(np.int32)
    got, _, st = gpu_sort(keys, None, cfg)
    assert same_bytes(got, np.sort(keys)) and (st["check_result"] >> 4) == 2 and st["partition_right_calls"] == 0
    got, _, st = gpu_sort(keys, None, SortConfig(two_run_min=n + 1))
    assert same_bytes(got, np.sort(keys)) and st["run_split"] == 0 and st["partition_right_calls"] >= 1
    # the mirrored kinds: a short descending / ascending / random first run before a sorted second run
    for kind, code in ((1, 5), (2, 6), (3, 7)):
        keys = _two_runs(rng, n, n - s, kind, np.int32, mirror=True)
        got, _, st = gpu_sort(keys, None, cfg)
        assert same_bytes(got, np.sort(keys)) and (st["check_result"] >> 4) == code and st["run_split"] == n - s, st
        assert (st["partition_right_calls"] == 0) == (kind != 3)
    # use_partial_insertion=False switches K4 off altogether (driver.py:63)
    got, _, st = gpu_sort(keys, None, SortConfig(two_run_min=64, use_partial_insertion=False))
    assert same_bytes(got, np.sort(keys)) and st["run_split"] == 0


def test_two_run_patterns_beat_uniform():
    # BASELINE C2: ascending + random tail and organ pipe at 2^24 take the two-run path (default
    # threshold) and finish well below the time of a uniform sort of the same size
    from paper_2106_05123_b200 import DeviceSorter

    n = 1 << 24
    cases = {"C2.asc_tail": workloads.c2("asc_tail", n), "C2.organ": workloads.c2("organ", n),
             "uniform": workloads.c1(n)}
    ms = {}
    for name, keys in cases.items():
        src = torch.from_numpy(keys).to(DEV)
        x = src.clone()
        ds = DeviceSorter(n, x.dtype, False)
        best = 1e9
        for _ in range(4):
            x.copy_(src)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ds.run(x)
            b.record()
            st = ds.finish()
            best = min(best, a.elapsed_time(b))
        assert bool((x[1:] >= x[:-1]).all().item())
        if name != "uniform":
            assert st["run_split"] >= n // 2, (name, st)
        ms[name] = best
    assert ms["C2.asc_tail"] < 0.7 * ms["uniform"] and ms["C2.organ"] < 0.7 * ms["uniform"], ms


@pytest.mark.parametrize("n,period", [(3356801, 1757), (8000000, 4400)])
def test_forced_fallback_many_tiny_digit_passes(n, period):
    # saw-tooth keys with a 2-bit payload under the forced fallback and 1024-element leaves: ~1800+ runs of one
    # key each take fifteen one-tile digit passes over the payload's zero bits while the CTAs that start the
    # children of the wide passes are busy for a millisecond -- ring positions wrap past a claimed slot (the
    # task queue once stalled here: a task overwritten before its claimer read it; tools/fuzz.py seed 29)
    rng = np.random.default_rng(29)
    keys = (np.arange(n) % period).astype(np.int32)
    vals = rng.integers(0, 4, n).astype(np.uint32)
    got_k, got_v, st = gpu_sort(keys, vals, SortConfig(base_case_size=1024, bad_budget=0))
    order = np.lexsort((vals, keys))
    assert same_bytes(got_k, keys[order]) and same_bytes(got_v, vals[order])
    assert st["status"] == 0 and st["radix_fallbacks"] >= 1


def test_check_pass_stops_early_on_uniform_input():
    # K4 must cost uniform input almost nothing: the pass stops once an ascent and descents in both halves
    # have been seen (a two-wave grid once scanned the whole first half before stopping: 42 % of 2^28 keys)
    n = 1 << 26
    g = torch.Generator(device=DEV)
    g.manual_seed(8)
    kd = torch.randint(-(2**31), 2**31, (n,), dtype=torch.int64, device=DEV, generator=g).to(torch.int32)
    st = sort_device(kd)
    assert bool((kd[1:] >= kd[:-1]).all().item())
    assert st["check_result"] & 15 == 15 and st["run_split"] == 0
    assert st["bytes_check"] <= 4 * n // 4, st["bytes_check"]


def test_extreme_values_and_zeros():
    for dt in (np.int32, np.int64):
        info = np.iinfo(dt)
        keys = np.array([info.max, info.min, 0, -1, 1, info.min, info.max] * 1000, dtype=dt)
        got, _, _ = gpu_sort(keys)
        assert same_bytes(got, np.sort(keys))
    for dt in (np.float32, np.float64):
        keys = np.array([np.inf, -np.inf, 0.0, 1.5, -1.5, np.finfo(dt).tiny, -np.finfo(dt).max] * 999, dtype=dt)
        got, _, _ = gpu_sort(keys)
        assert same_bytes(got, np.sort(keys))
        # -0.0 and +0.0 compare equal under '<': any order of them is sorted; total order puts -0 first
        z = np.array([0.0, -0.0] * 5000, dtype=dt)
        got, _, _ = gpu_sort(z)
        assert np.all(got[:-1] <= got[1:]) and np.signbit(got).sum() == 5000 and np.signbit(got[:5000]).all()


def test_host_containers_drop_in():
    rng = np.random.default_rng(7)
    values = [int(x) for x in rng.integers(-10**12, 10**12, 3000)]
    lst = list(values)
    sort(lst)
    assert lst == sorted(values)
    buf = array.array("q", values)  # pkg/tests/test_driver.py:189-196
    sort(buf)
    assert list(buf) == sorted(values)
    fl = [float(x) for x in rng.standard_normal(2000)] + [float("inf"), float("-inf")]
    w = list(fl)
    sort(w)
    assert w == sorted(fl)
    pairs = [(int(rng.integers(0, 50)), i) for i in range(3000)]  # KV as tuples (lexicographic)
    w = list(pairs)
    sort(w)
    assert w == sorted(pairs)
    a = rng.integers(0, 100, 5000).astype(np.int32)
    b = a.copy()
    sort(b)
    assert np.array_equal(b, np.sort(a))
    t = torch.from_numpy(a.copy())
    sort(t)
    assert np.array_equal(t.numpy(), np.sort(a))
    sort_with(w, __import__("operator").lt)
    with pytest.raises(NotImplementedError):
        sort_with(w, lambda x, y: y < x)


def test_misaligned_view_and_values_keyword():
    rng = np.random.default_rng(8)
    base = torch.from_numpy(rng.integers(0, 1000, 10001).astype(np.int32)).to(DEV)
    view = base[1:]
    exp = np.sort(view.cpu().numpy())
    sort(view)
    assert np.array_equal(view.cpu().numpy(), exp)
    keys = rng.integers(0, 10, 4000).astype(np.int64)
    vals = np.arange(4000, dtype=np.uint32)
    k, v = keys.copy(), vals.copy()
    sort(k, values=v)
    order = np.lexsort((vals, keys))
    assert np.array_equal(k, keys[order]) and np.array_equal(v, vals[order])


def test_concurrent_streams_distinct_workspaces():
    rng = np.random.default_rng(9)
    arrs = [rng.integers(-(2**31), 2**31, 1 << 20, dtype=np.int64).astype(np.int32) for _ in range(3)]
    from paper_2106_05123_b200 import DeviceSorter

    streams = [torch.cuda.Stream() for _ in arrs]
    devs, sorters = [], []
    for a, s in zip(arrs, streams):
        with torch.cuda.stream(s):
            d = torch.from_numpy(a).to(DEV, non_blocking=False)
            ds = DeviceSorter(a.size, torch.int32, False)
            ds.run(d)
            devs.append(d)
            sorters.append(ds)
    for a, d, ds, s in zip(arrs, devs, sorters, streams):
        ds.finish(s)
        assert np.array_equal(d.cpu().numpy(), np.sort(a))


def test_concurrent_two_run_sorts_do_not_deadlock():
    # the merge epilogue of the leaf kernel waits on progress counters, not grid barriers: four sorts that
    # all take the two-run path on different streams (their one-CTA-per-SM leaf kernels cannot be
    # co-resident) must all finish
    from paper_2106_05123_b200 import DeviceSorter

    rng = np.random.default_rng(10)
    n = 1 << 22
    arrs = []
    for kind in (1, 2, 3, 3):
        arrs.append(_two_runs(rng, n, int(0.7 * n), kind, np.int32))
    streams = [torch.cuda.Stream() for _ in arrs]
    devs = [torch.from_numpy(a).to(DEV) for a in arrs]
    sorters = [DeviceSorter(n, torch.int32, False) for _ in arrs]
    torch.cuda.synchronize()
    for rep in range(3):
        for d, a in zip(devs, arrs):
            d.copy_(torch.from_numpy(a))
        torch.cuda.synchronize()
        for d, ds, s in zip(devs, sorters, streams):
            with torch.cuda.stream(s):
                ds.run(d)
        for a, d, ds, s in zip(arrs, devs, sorters, streams):
            st = ds.finish(s)
            assert st["run_split"] > 0
            assert np.array_equal(d.cpu().numpy(), np.sort(a))


def test_repeated_sorts_reuse_workspace():
    from paper_2106_05123_b200 import DeviceSorter

    rng = np.random.default_rng(10)
    ds = DeviceSorter(100000, torch.float32, False)
    for _ in range(5):
        a = rng.standard_normal(100000).astype(np.float32)
        d = torch.from_numpy(a).to(DEV)
        ds.run(d)
        ds.finish()
        assert np.array_equal(d.cpu().numpy(), np.sort(a))


def test_host_pipeline_batches():
    # HostPipeline (the serving-side host-batch path used by bench.py's e2e leg): every batch sorted,
    # buffers recycled across more batches than device buffers
    from paper_2106_05123_b200 import HostPipeline

    rng = np.random.default_rng(21)
    n = 300001
    for dtype, tdt in ((np.int32, torch.int32), (np.float32, torch.float32)):
        ins = [torch.from_numpy(shapes(n, rng, dtype)[name].copy()).pin_memory()
               for name in ("uniform", "dups16", "desc", "organ", "asc_tail", "uniform", "dupsq")]
        outs = [torch.empty_like(x).pin_memory() for x in ins]
        HostPipeline(n, tdt, depth=3).sort(ins, outs)
        for x, y in zip(ins, outs):
            assert same_bytes(y.numpy(), oracle_sort(x.numpy())[0])


@pytest.mark.parametrize("k", [1, 2, 16, 256])
def test_device_counters_onk_bound(k):
    # f1: the device counters re-assert the paper's O(nk) bound for k distinct keys
    # (the reference's acceptance criterion counts partitions <= 2k) and a depth bound
    n = 1 << 22
    keys = workloads.c3(k, n)
    got, _, st = gpu_sort(keys)
    assert same_bytes(got, np.sort(keys))
    assert st["partition_right_calls"] + st["partition_left_calls"] <= 2 * k + 2, st
    assert st["max_depth"] <= 2 * 22, st
    u = workloads.c1(n)
    _, _, st = gpu_sort(u)
    assert st["max_depth"] <= 2 * 22 and st["bad_partitions"] <= 4, st


@pytest.mark.parametrize("k", [2, 16, 1024])
def test_kv_low_cardinality_argsort(k):
    # argsort by a low-cardinality key (distinct payloads = indices): key-value leaves whose buckets hold
    # many equal keys take k_base_wide's radix fallback; the (key, payload) order is exact
    rng = np.random.default_rng(100 + k)
    n = (1 << 20) + 3
    keys = (rng.integers(0, k, n).astype(np.int64) << 30) - (1 << 40)
    vals = rng.permutation(n).astype(np.uint32)
    got_k, got_v, _ = gpu_sort(keys, vals)
    exp_k, exp_v = workloads.expected(keys, vals)
    assert same_bytes(got_k, exp_k) and same_bytes(got_v, exp_v)
    k32 = (keys >> 30).astype(np.int32)  # 4-byte keys with a payload (8-byte elements)
    got_k, got_v, _ = gpu_sort(k32, vals)
    exp_k, exp_v = workloads.expected(k32, vals)
    assert same_bytes(got_k, exp_k) and same_bytes(got_v, exp_v)


def test_sort_with_descending_ordering():
    # f4: operator.gt (descending) runs on the device as the ascending sort reversed; the output is the
    # unique descending order, as the reference's sort_with(data, operator.gt) produces
    import operator

    rng = np.random.default_rng(31)
    ints = rng.integers(-(2**31), 2**31, 50001).tolist()
    w = list(ints)
    sort_with(w, operator.gt)
    assert w == sorted(ints, reverse=True)
    flts = rng.standard_normal(30001).tolist()
    w = list(flts)
    sort_with(w, operator.gt)
    assert w == sorted(flts, reverse=True)
    pairs = list(zip(rng.integers(0, 100, 20001).tolist(), rng.permutation(20001).tolist()))
    w = list(pairs)
    sort_with(w, operator.gt)
    assert w == sorted(pairs, reverse=True)
    t = torch.from_numpy(rng.integers(-1000, 1000, 70001).astype(np.int32)).to(DEV)
    ref = np.sort(t.cpu().numpy())[::-1]
    sort_with(t, operator.gt)
    assert same_bytes(t.cpu().numpy(), ref.copy())


def test_sort_with_field_ordering():
    # f4: key-field of a packed record.  The reference's test_custom_ordering (test_driver.py:198-204)
    # sorts (key, index) tuples with `lambda a, b: a[0] < b[0]`; by_field(0) is that ordering as an
    # object the device path recognises.  Same checks as the reference's test, plus the exact result
    # (ties keep input order) and descending / structured-array / float variants.
    import random
    from collections import Counter

    from paper_2106_05123_b200 import DEFAULT_CONFIG, by_field, sort_with_config

    rng = random.Random(13)
    arr = [(rng.randint(0, 9), i) for i in range(1000)]
    work = list(arr)
    sort_with(work, by_field(0))
    assert [x[0] for x in work] == sorted(x[0] for x in arr)
    assert Counter(work) == Counter(arr)
    assert work == sorted(arr, key=lambda r: r[0])  # Python's sort is stable: ties in input order
    work = list(arr)
    sort_with(work, by_field(0, descending=True))
    assert [x[0] for x in work] == sorted((x[0] for x in arr), reverse=True)
    assert Counter(work) == Counter(arr)
    recs = [(rng.random(), "r%d" % i, -i) for i in range(30001)]
    work = list(recs)
    sort_with_config(work, by_field(2), DEFAULT_CONFIG)
    assert work == sorted(recs, key=lambda r: r[2])
    work = list(recs)
    sort_with(work, by_field(0))
    assert work == sorted(recs, key=lambda r: r[0])
    sa = np.zeros(50001, dtype=[("id", np.int32), ("w", np.float32)])
    g = np.random.default_rng(4)
    sa["id"] = np.arange(50001)
    sa["w"] = g.standard_normal(50001).astype(np.float32)
    want = sa[np.argsort(sa["w"], kind="stable")]
    sort_with(sa, by_field("w"))
    assert np.array_equal(sa, want)


def test_float_tuple_keys_and_nan_mixed_list():
    # (float key, payload) tuples are sorted as float64 keys, never truncated to ints
    w = [(0.5, 1), (0.25, 2), (-1.75, 0), (0.25, 1)]
    sort(w)
    assert w == sorted([(0.5, 1), (0.25, 2), (-1.75, 0), (0.25, 1)])
    # mixed int/float list with a NaN: the original element types come back (keyed by bit pattern)
    nan = float("nan")
    lst = [3, nan, 2.0, 1]
    sort(lst)
    assert lst[:3] == [1, 2.0, 3] and [type(x) for x in lst[:3]] == [int, float, int]
    assert lst[3] != lst[3]  # NaN (positive NaN sorts last in the total order)


@pytest.mark.parametrize("dtype", DTYPES, ids=lambda d: np.dtype(d).name)
def test_host_sorter_drop_in_sizes(dtype):
    """pdq_host_sort (the host-buffer drop-in): sizes around the 8 MiB staging chunk and the
    worker stride, sorted in place in the caller's numpy buffer, against the oracle."""
    from paper_2106_05123_b200 import HostSorter

    rng = np.random.default_rng(31)
    hs = HostSorter(0, 3)
    w = np.dtype(dtype).itemsize
    chunk = (8 << 20) // w
    for n in (0, 1, 2, 1000, chunk - 1, chunk, chunk + 1, 3 * chunk + 17, 7 * chunk + 5):
        keys = shapes(n, rng, dtype)["uniform"]
        ref = oracle_sort(keys)[0]
        buf = keys.copy()
        stats, ph = hs.sort(buf, phases=True)
        assert same_bytes(buf, ref), (np.dtype(dtype).name, n)
        assert stats["status"] == 0
    hs.close()


def test_host_sorter_kv_and_errors():
    from paper_2106_05123_b200 import HostSorter, SortConfig

    rng = np.random.default_rng(32)
    hs = HostSorter(0)
    for n in (5, (2 << 20) + 3, (5 << 20) + 1):
        keys = rng.integers(-(2**40), 2**40, n)
        vals = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
        rk, rv = oracle_sort(keys, vals)
        k, v = keys.copy(), vals.copy()
        hs.sort(k, v)
        assert same_bytes(k, rk) and same_bytes(v, rv)
    # a strided view goes through a contiguous copy and back
    base = rng.integers(0, 1000, 20001).astype(np.int32)
    view = base[::2]
    exp = np.sort(view)
    sort(view)
    assert np.array_equal(view, exp)
    with pytest.raises(TypeError):
        hs.sort(np.zeros(4, np.int16))
    with pytest.raises(ValueError):
        SortConfig(block_size=0)


@pytest.mark.parametrize("case", ["narrow", "k3", "kv_dupkeys", "kv_const_key", "f32_dups", "i64_prefix"])
def test_forced_fallback_digit_pass_shapes(case):
    """K5 digit passes on shapes that exercise their paths: one-digit passes skipped (shared high bits),
    digits in the payload (equal keys, distinct payloads), runs of <= 64 sorted by warps, constant runs,
    runs that are leaves and runs that take another digit pass; against the oracle / lexicographic order."""
    rng = np.random.default_rng(17)
    cfg = SortConfig(bad_budget=0)
    for n in (70001, 1 << 20, 3 << 20):
        vals = None
        if case == "narrow":
            keys = rng.integers(1 << 20, (1 << 20) + 5000, n).astype(np.int32)
        elif case == "k3":
            keys = rng.integers(0, 3, n).astype(np.int32)
        elif case == "kv_dupkeys":
            keys = rng.integers(0, 50, n).astype(np.int64)
            vals = rng.integers(0, 2**32, n, dtype=np.uint32)
        elif case == "kv_const_key":
            keys = np.full(n, 7, np.int32)
            vals = rng.integers(0, 1 << 12, n).astype(np.uint32)
        elif case == "f32_dups":
            keys = np.round(rng.standard_normal(n) * 100).astype(np.float32) + np.float32(0)  # no -0.0
        else:
            keys = (rng.integers(0, 1 << 30, n) + (1 << 40)).astype(np.int64)
        got_k, got_v, stats = gpu_sort(keys, vals, config=cfg)
        exp_k, exp_v = workloads.expected(keys, vals)
        assert same_bytes(got_k, exp_k) and (vals is None or same_bytes(got_v, exp_v)), (case, n)
        assert stats["radix_fallbacks"] >= 1 and stats["status"] == 0


# ---- the reference's property tests (pkg/tests/test_driver.py:243-254) on the device path ----------
from hypothesis import given, settings, strategies as st  # noqa: E402


@given(st.lists(st.integers(-1000, 1000), max_size=300))
@settings(max_examples=200, deadline=None)
def test_property_sorts_any_int_list(arr):
    work = list(arr)
    sort(work)
    assert work == sorted(arr)


@given(st.lists(st.floats(allow_nan=False, allow_infinity=True), max_size=100))
@settings(max_examples=100, deadline=None)
def test_property_sorts_floats_with_infinities(arr):
    work = list(arr)
    sort(work)
    assert work == sorted(arr)


def test_instrumented_sort_metrics_and_onk_bound():
    """instrumented_sort (instrumentation.py:79-109) on the device: the Metrics columns, and the
    paper's O(nk) property as the reference's acceptance test asserts it (partitions <= 2k for k
    distinct keys, acceptance.py:242-265)."""
    from paper_2106_05123_b200 import Metrics, instrumented_sort

    rng = np.random.default_rng(21)
    for k in (1, 2, 16, 256):
        data = rng.integers(0, k, 1 << 20).astype(np.int32).tolist()
        exp = sorted(data)
        m = instrumented_sort(data)
        assert isinstance(m, Metrics) and data == exp
        assert m.partition_right_calls + m.partition_left_calls <= 2 * k + 2
        assert len(m.counter_values()) == 10 and m.counter_values()[0] == 0
    m = instrumented_sort([3, 1, 2], __import__("operator").gt)
    assert m.device is not None and m.device["status"] == 0


def test_stratified_adversary_spoils_only_the_root():
    """The input-side adversary for the root's stratified sample: the root's partition is bad, the
    budget (floor(log2 n)) is far from spent, the output is the sorted permutation."""
    n = 1 << 22
    keys = workloads.stratified_adversary(n)
    got, _, stats = gpu_sort(keys)
    assert same_bytes(got, np.arange(n, dtype=np.int32))
    assert stats["bad_partitions"] >= 1 and stats["radix_fallbacks"] == 0
