"""Multi-GPU sample sort, host logic on CPU: gloo ranks (world size 2 and 3)
run paper_2106_05123_b200.distributed.sample_sort end to end -- size exchange, sample all-gather,
splitter choice, count and element all-to-alls -- with the two device steps (pdq_bucket and the
local sort_device) replaced, in this test only, by numpy statements of the same contracts.  The
concatenated rank outputs must equal the sorted global array bit for bit, and heavy duplicates
must spread over the ranks (ties broken by global index).  The device steps themselves are
checked on the B200 in tests/test_distributed_gpu.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2106_05123_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bits(t: torch.Tensor) -> np.ndarray:
    return D._raw_bits(t).numpy().astype(np.int64)


def _key_order(t: torch.Tensor) -> np.ndarray:
    return D.ordered_image(_bits(t), t.element_size(), t.dtype in (torch.float32, torch.float64))


def np_bucket(keys, values, base, splitters):
    """pdq_bucket's contract (include/pdq_b200.h): bucket = #splitters below (key, payload, gidx);
    stable within a bucket."""
    if torch.is_tensor(splitters):
        splitters = splitters.cpu().numpy()
    n = keys.numel()
    k = _key_order(keys)
    v = values.numpy().astype(np.int64) & 0xFFFFFFFF if values is not None else np.zeros(n, np.int64)
    g = base + np.arange(n, dtype=np.int64)
    sk = D.ordered_image(splitters[:, 0], keys.element_size(), keys.dtype in (torch.float32, torch.float64))
    b = np.zeros(n, dtype=np.int64)
    for j in range(splitters.shape[0]):
        svj, sgj = splitters[j, 1], splitters[j, 2]
        below = (sk[j] < k) | ((sk[j] == k) & ((svj < v) | ((svj == v) & (sgj < g))))
        b += below
    order = np.argsort(b, kind="stable")
    nb = splitters.shape[0] + 1
    out_k = keys[torch.from_numpy(order)].clone()
    out_v = values[torch.from_numpy(order)].clone() if values is not None else None
    return out_k, out_v, torch.from_numpy(np.bincount(b, minlength=nb).astype(np.int64))


def np_local_sort(keys, values, config):
    k = _key_order(keys)
    if values is not None:
        order = np.lexsort((values.numpy().astype(np.int64) & 0xFFFFFFFF, k))
    else:
        order = np.argsort(k, kind="stable")
    idx = torch.from_numpy(order)
    keys.copy_(keys[idx].clone())
    if values is not None:
        values.copy_(values[idx].clone())


def make_case(name, world, rank):
    rng = np.random.default_rng(1000 + 17 * world)
    sizes = {"int32": [5000, 3000, 4000], "kv": [4000, 0, 2500], "float": [3000, 3001, 1],
             "equal": [6000, 6000, 6000], "empty": [0, 0, 0], "skewed": [20000, 300, 300]}[name][:world]
    parts = []
    for r in range(world):
        n = sizes[r]
        if name == "int32":
            parts.append((torch.from_numpy(rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)), None))
        elif name == "kv":
            k = torch.from_numpy(rng.integers(-50, 50, n, dtype=np.int64))
            v = torch.from_numpy(rng.integers(0, 2**32, n, dtype=np.int64).astype(np.uint32).view(np.int32))
            parts.append((k, v))
        elif name == "float":
            x = rng.standard_normal(n).astype(np.float32)
            x[::97] = 0.0
            x[1::97] = -0.0
            x[2::101] = np.inf
            x[3::103] = -np.inf
            parts.append((torch.from_numpy(x), None))
        elif name == "equal":
            parts.append((torch.full((n,), 7, dtype=torch.int64), None))
        elif name == "skewed":  # very unequal shards over disjoint key ranges (weighting)
            parts.append((torch.from_numpy(rng.integers(1000 * r, 1000 * r + 1000, n, dtype=np.int64)), None))
        else:
            parts.append((torch.empty(0, dtype=torch.int32), None))
    return parts


def _worker(rank, world, port, name, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    D._bucket = np_bucket
    D._local_sort = np_local_sort
    keys, vals = make_case(name, world, rank)[rank]
    ok, ov = D.sample_sort(keys, vals, oversample=32)
    out[rank] = (_bits(ok).tolist(), None if ov is None else ov.numpy().tolist())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["int32", "kv", "float", "equal", "empty", "skewed"])
def test_sample_sort_gloo(world, name):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), name, out), nprocs=world, join=True)
    parts = make_case(name, world, 0)
    keys = torch.cat([p[0] for p in parts])
    vals = torch.cat([p[1] for p in parts]) if parts[0][1] is not None else None
    np_local_sort(keys, vals, None)
    got_k = sum((out[r][0] for r in range(world)), [])
    assert got_k == _bits(keys).tolist()
    if vals is not None:
        assert sum((out[r][1] for r in range(world)), []) == vals.numpy().tolist()
    if name in ("equal", "skewed"):  # ties by global index; samples weighted by shard size
        tol = 0.1 if name == "equal" else 0.3  # skewed: 96 random samples of the big shard per rank
        for r in range(world):
            assert abs(len(out[r][0]) - keys.numel() / world) < tol * keys.numel() / world


def test_splitter_choice_is_rank_independent_and_ordered():
    rng = np.random.default_rng(5)
    s = np.stack([rng.integers(-2**31, 2**31, 999), rng.integers(0, 4, 999), rng.permutation(999)], axis=1)
    a = D.choose_splitters(s, 4, 4, False)
    b = D.choose_splitters(s[rng.permutation(999)], 4, 4, False)
    assert (a == b).all() and a.shape == (3, 3)
    ok = D.ordered_image(a[:, 0], 4, False)
    assert (np.diff(ok.astype(np.float64)) >= 0).all()
    assert D.choose_splitters(s, 1, 4, False).shape == (0, 3)


def test_weighted_splitters_follow_shard_sizes():
    # rank 0: 10 samples standing for 10000 keys in [0, 100); rank 1: 10 samples for 10 keys in [100, 110)
    s0 = np.stack([np.arange(0, 100, 10), np.zeros(10, np.int64), np.arange(10)], axis=1)
    s1 = np.stack([np.arange(100, 110), np.zeros(10, np.int64), 10000 + np.arange(10)], axis=1)
    s = np.concatenate([s0, s1])
    w = np.concatenate([np.full(10, 1000.0), np.full(10, 1.0)])
    unweighted = D.choose_splitters(s, 2, 8, False)
    weighted = D.choose_splitters(s, 2, 8, False, w)
    assert unweighted[0, 0] == 100            # half the samples: the small shard's range
    assert 40 <= weighted[0, 0] <= 60         # half the weight: the middle of the big shard
    eq = D.choose_splitters(s, 4, 8, False, np.ones(20))
    assert (eq == D.choose_splitters(s, 4, 8, False)).all()  # equal weights = the unweighted picks
    rows = np.zeros((8, 4), np.int64)
    rows[:3, 3] = 300
    rows[4:8, 3] = 40
    assert list(D.sample_weights(rows, 4)) == [100.0] * 3 + [10.0] * 4


@pytest.mark.parametrize("width,is_float", [(4, False), (4, True), (8, False), (8, True)])
def test_device_splitters_follow_the_numpy_rule(width, is_float):
    # device_splitters (torch, what sample_sort runs) = choose_splitters (numpy statement) with weights
    rng = np.random.default_rng(width * 2 + is_float)
    P, S = 4, 64
    sizes = [5000, 0, 300, 12000]
    blocks = []
    for r in range(P):
        m = min(S, sizes[r])
        if width == 4:
            raw = (rng.standard_normal(m).astype(np.float32).view(np.uint32).astype(np.int64) if is_float
                   else rng.integers(0, 2**32, m).astype(np.int64))
        else:
            raw = rng.standard_normal(m).view(np.int64) if is_float else rng.integers(-2**63, 2**63, m)
        raw[: m // 3] = raw[0] if m else raw[: m // 3]  # duplicate keys: ties by payload, then position
        rows = np.zeros((S, 4), np.int64)
        rows[:m, 0] = raw
        rows[:m, 1] = rng.integers(0, 3, m)
        rows[:m, 2] = (r << D.POS_SHIFT) + np.arange(m)
        rows[:m, 3] = sizes[r]
        blocks.append(rows)
    rows = np.concatenate(blocks)
    dev = D.device_splitters(torch.from_numpy(rows), P, S, width, is_float).numpy()
    ref = D.choose_splitters(D.valid_samples(rows), P, width, is_float, D.sample_weights(rows, S))
    assert dev.shape == (P - 1, 3) and (dev == ref).all()


def test_ordered_image_matches_numeric_order():
    x = np.array([-np.inf, -2.5, -0.0, 0.0, 1e-30, 3.0, np.inf], dtype=np.float64)
    img = D.ordered_image(x.view(np.int64), 8, True)
    assert (np.diff(img.astype(object)) > 0).all()
    y = np.array([-2**31, -1, 0, 5, 2**31 - 1], dtype=np.int64)
    img = D.ordered_image(y, 4, False)
    assert list(np.argsort(img)) == [0, 1, 2, 3, 4]
    assert list(D.sample_positions(10, 5)) == [1, 3, 5, 7, 9]
