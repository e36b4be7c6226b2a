"""Multi-GPU sample sort on the B200: the pdq_bucket kernel against the numpy
statement of its contract (exact output order and counts), the P-shard pipeline run shard by shard
on one GPU (no rank waits on another), and sample_sort itself over a one-rank NCCL group."""

import os
import socket

import numpy as np
import pytest
import torch

from paper_2106_05123_b200 import distributed as D
from paper_2106_05123_b200 import sort_device
from test_distributed_cpu import np_bucket, np_local_sort

pytestmark = pytest.mark.gpu

DTYPES = [torch.int32, torch.int64, torch.float32, torch.float64]


def rand_keys(n, dtype, gen, lowcard=False):
    if lowcard:
        x = torch.randint(-3, 3, (n,), generator=gen, dtype=torch.int64)
        return x.to(dtype)
    if dtype == torch.int32:
        return torch.randint(-2**31, 2**31, (n,), generator=gen, dtype=torch.int64).to(torch.int32)
    if dtype == torch.int64:
        return torch.randint(-2**62, 2**62, (n,), generator=gen, dtype=torch.int64)
    x = torch.randn(n, generator=gen, dtype=torch.float64).to(dtype)
    if n > 10:
        x[::7] = 0.0
        x[1::11] = -0.0
        x[2::13] = float("inf")
    return x


def splitters_from(keys, vals, nsplit, gen):
    rows = D.valid_samples(D.local_samples(keys, vals, 1000, max(1, 4 * nsplit)).cpu().numpy())
    return D.choose_splitters(rows, nsplit + 1, keys.element_size(), keys.dtype in (torch.float32, torch.float64))


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("kv", [False, True])
def test_bucket_kernel_matches_contract(dtype, kv):
    gen = torch.Generator().manual_seed(3)
    for n in (1, 255, 256, 257, 5000, 100_003, 1 << 21):
        for nsplit in (0, 1, 3, 7, 31, 32, 63):
            for lowcard in (False, True):
                keys = rand_keys(n, dtype, gen, lowcard)
                vals = (torch.randint(0, 4, (n,), generator=gen, dtype=torch.int32) if kv else None)
                sp = splitters_from(keys, vals, nsplit, gen)
                if sp.shape[0] < nsplit:
                    continue
                want_k, want_v, want_c = np_bucket(keys, vals, 1000, sp)
                got_k, got_v, got_c = D._bucket(keys.cuda(), vals.cuda() if kv else None, 1000, sp)
                assert torch.equal(got_c.cpu(), want_c), (n, nsplit)
                assert torch.equal(D._raw_bits(got_k.cpu()), D._raw_bits(want_k)), (n, nsplit)
                if kv:
                    assert torch.equal(got_v.cpu(), want_v)


def test_bucket_empty_and_errors():
    k = torch.empty(0, dtype=torch.int32, device="cuda")
    sp = np.array([[5, 0, 0]], dtype=np.int64)
    ok, ov, c = D._bucket(k, None, 0, sp)
    assert c.cpu().tolist() == [0, 0]
    with pytest.raises(RuntimeError, match="nsplit"):
        D._bucket(torch.zeros(8, dtype=torch.int32, device="cuda"), None, 0, np.zeros((64, 3), np.int64))


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("case", ["i32", "kv", "f64", "equal"])
def test_sharded_pipeline_one_gpu(P, case):
    """The sample sort's data path for P shards, shard by shard: samples -> splitters -> pdq_bucket
    -> route bucket r of every shard to slice r -> sort_device per slice; the slices concatenated
    equal the numpy sort of the whole array (device splitter choice, as sample_sort runs it)."""
    gen = torch.Generator().manual_seed(P)
    n = 1 << 20
    dt = {"i32": torch.int32, "kv": torch.int64, "f64": torch.float64, "equal": torch.int32}[case]
    keys = torch.full((n,), 9, dtype=dt) if case == "equal" else rand_keys(n, dt, gen, lowcard=False)
    vals = torch.randint(0, 2**31, (n,), generator=gen, dtype=torch.int32) if case == "kv" else None
    kd, vd = keys.cuda(), (vals.cuda() if vals is not None else None)
    bounds = [(r * n) // P for r in range(P + 1)]
    shards = [(kd[bounds[r]:bounds[r + 1]].contiguous(),
               vd[bounds[r]:bounds[r + 1]].contiguous() if vd is not None else None) for r in range(P)]
    rows = torch.cat([D.local_samples(k, v, r << D.POS_SHIFT, 64 * P) for r, (k, v) in enumerate(shards)])
    sp = D.device_splitters(rows, P, 64 * P, keys.element_size(), dt in (torch.float32, torch.float64))
    routed = [[] for _ in range(P)]
    for r, (k, v) in enumerate(shards):
        bk, bv, c = D._bucket(k, v, r << D.POS_SHIFT, sp)
        off = np.concatenate([[0], np.cumsum(c.cpu().numpy())])
        for d in range(P):
            routed[d].append((bk[off[d]:off[d + 1]], bv[off[d]:off[d + 1]] if bv is not None else None))
    outs_k, outs_v = [], []
    for d in range(P):
        k = torch.cat([x[0] for x in routed[d]])
        v = torch.cat([x[1] for x in routed[d]]) if vd is not None else None
        if k.numel():
            sort_device(k, v)
        outs_k.append(k)
        outs_v.append(v)
        assert k.numel() < 1.5 * n / P  # balanced, duplicates included
    # expected: numpy (total order of the key images, lexicographic with the payload), independent of
    # the device sort
    whole_k = keys.clone()
    whole_v = vals.clone() if vals is not None else None
    np_local_sort(whole_k, whole_v, None)
    assert torch.equal(D._raw_bits(torch.cat(outs_k)).cpu(), D._raw_bits(whole_k))
    if vd is not None:
        assert torch.equal(torch.cat(outs_v).cpu(), whole_v)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sample_sort_nccl_one_rank():
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        gen = torch.Generator().manual_seed(11)
        for dt, kv in ((torch.int32, False), (torch.float32, False), (torch.int64, True)):
            keys = rand_keys(300_001, dt, gen).cuda()
            vals = torch.randint(0, 2**31, (300_001,), generator=gen, dtype=torch.int32).cuda() if kv else None
            ok, ov = D.sample_sort(keys, vals)
            wk, wv = keys.cpu().clone(), (vals.cpu().clone() if kv else None)
            np_local_sort(wk, wv, None)  # numpy expectation, independent of the device sort
            assert torch.equal(D._raw_bits(ok).cpu(), D._raw_bits(wk))
            if kv:
                assert torch.equal(ov.cpu(), wv)
    finally:
        dist.destroy_process_group()
