"""Multi-GPU sample sort: one process per GPU, one exchange step.

The reference is single-process (its sort is `driver.py:267-292` on one sequence); this is the
scale-out the survey plans for arrays larger than one GPU's HBM or sorts spread over a node:

1. every rank draws ``oversample · P`` evenly spaced samples of its shard, each sample tagged with
   its global index (rank offset + position);
2. one all-gather of the samples; every rank orders the same P · S samples by
   (key, payload, global index) and picks the same P − 1 splitters at the sample quantiles;
3. ``pdq_bucket`` (CUDA, csrc/pdq_bucket.cuh) splits the local shard into P buckets by those
   splitters, ties broken by global index so even an all-equal input spreads evenly;
4. an all-to-all of the bucket sizes, then one all-to-all of keys (and payload) over NCCL: rank r
   receives bucket r of every rank;
5. the received elements are sorted in place by the single-GPU sort (``sort_device``).

Rank r's output is the r-th slice of the global sort; the concatenation over ranks in rank order is
the whole array sorted.  Equal elements are bit-identical (keys) or identical pairs, so the result
is the unique sorted array and parity with the single-GPU sort is bit-exact.

Device work (bucketing, exchange, local sort) runs in CUDA and NCCL; only the splitter choice over
the P · S gathered samples (a few thousand values) is host logic.  There is no CPU fallback: the
bucketing and the local sort raise without the CUDA library.
"""

from __future__ import annotations

import ctypes
from typing import Optional, Tuple

import numpy as np

from . import _lib
from .driver import DEFAULT_CONFIG, SortConfig, _dtype_code, _raise, sort_device

DEFAULT_OVERSAMPLE = 256
MAX_RANKS = 64  # buckets per pdq_bucket call


# ---- key images (host side of the device's Ord<U, FLOAT>, pdq_device.cuh) ----------------------

def _raw_bits(keys) -> "torch.Tensor":
    """The keys' bit patterns as a same-width signed-int tensor (no copy)."""
    import torch

    if keys.dtype in (torch.int32, torch.int64):
        return keys
    return keys.view(torch.int32 if keys.dtype == torch.float32 else torch.int64)


def ordered_image(raw: np.ndarray, width: int, is_float: bool) -> np.ndarray:
    """uint64 image whose unsigned order is the sort's key order (ints: flip the sign bit; floats:
    the IEEE total-order map), for raw bit patterns given as int64 (4-byte keys in the low 32 bits)."""
    u = raw.astype(np.uint64)
    if width == 4:
        u &= np.uint64(0xFFFFFFFF)
    sign = np.uint64(1) << np.uint64(8 * width - 1)
    mask = np.uint64((1 << (8 * width)) - 1)
    if is_float:
        neg = (u & sign) != 0
        return np.where(neg, ~u & mask, u ^ sign)
    return u ^ sign


def choose_splitters(samples: np.ndarray, nranks: int, width: int, is_float: bool,
                     weights: Optional[np.ndarray] = None) -> np.ndarray:
    """P − 1 splitters from gathered samples: rows of (raw key bits, payload, global index).

    Samples are ordered by (key in sort order, payload, global index).  Each sample stands for
    ``weights[i]`` elements of its shard (its shard's size over its shard's sample count), so a
    short shard does not count as much as a long one; splitter k is the first sample at which the
    cumulative weight reaches k/P of the total (unweighted: position ⌊k·M/P⌋).  Every rank runs this
    on the same gathered array, so every rank picks the same splitters."""
    m = samples.shape[0]
    if nranks <= 1 or m == 0:
        return np.empty((0, 3), dtype=np.int64)
    ordk = ordered_image(samples[:, 0], width, is_float)
    order = np.lexsort((samples[:, 2], samples[:, 1], ordk))
    if weights is None:
        picks = [(k * m) // nranks for k in range(1, nranks)]
    else:
        cum = np.cumsum(np.asarray(weights, dtype=np.float64)[order])
        tot = cum[-1]
        # the last sample whose exclusive cumulative weight is <= k/P of the total (equal weights:
        # floor(k M / P), the unweighted pick)
        excl = cum - np.asarray(weights, dtype=np.float64)[order]
        picks = [max(0, int(np.searchsorted(excl, k * tot / nranks * (1 + 1e-12), side="right")) - 1)
                 for k in range(1, nranks)]
    return samples[order[picks]]


def sample_positions(n_local: int, count: int) -> np.ndarray:
    """``count`` evenly spaced positions in [0, n_local), centred in their strata."""
    if count <= 0 or n_local <= 0:
        return np.empty(0, dtype=np.int64)
    k = np.arange(count, dtype=np.int64)
    return (2 * k + 1) * n_local // (2 * count)


# ---- device steps ------------------------------------------------------------------------------

def _bucket(keys, values, gidx_base: int, splitters: np.ndarray):
    """pdq_bucket on the device: (bucketed keys, bucketed payload or None, int64 counts[P])."""
    import torch

    dev = keys.device
    nb = splitters.shape[0] + 1
    n = keys.numel()
    code = _dtype_code(keys.dtype)
    raw = _raw_bits(keys)
    width = keys.element_size()
    sk_np = splitters[:, 0]
    sk_np = sk_np.astype(np.uint32).view(np.int32) if width == 4 else sk_np
    sk = torch.from_numpy(np.ascontiguousarray(sk_np)).to(dev).view(raw.dtype).view(keys.dtype)
    sv = torch.from_numpy(np.ascontiguousarray(splitters[:, 1].astype(np.uint32).view(np.int32))).to(dev)
    sg = torch.from_numpy(np.ascontiguousarray(splitters[:, 2])).to(dev)
    out_k = torch.empty_like(keys)
    out_v = torch.empty_like(values) if values is not None else None
    counts = torch.zeros(nb, dtype=torch.int64, device=dev)
    ws_bytes = _lib.lib().pdq_bucket_workspace_bytes(n, nb)
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream(dev)
    P = ctypes.c_void_p
    rc = _lib.lib().pdq_bucket(
        P(keys.data_ptr()), code, P(values.data_ptr() if values is not None else 0), n, int(gidx_base),
        P(sk.data_ptr() if nb > 1 else 0), P(sv.data_ptr() if nb > 1 and values is not None else 0),
        P(sg.data_ptr() if nb > 1 else 0), nb - 1, P(out_k.data_ptr()),
        P(out_v.data_ptr() if out_v is not None else 0), P(counts.data_ptr()), P(ws.data_ptr()), ws_bytes,
        P(s.cuda_stream))
    if rc != 0:
        _raise(rc, "pdq_bucket")
    return out_k, out_v, counts


def _local_sort(keys, values, config: SortConfig) -> None:
    if keys.numel():
        sort_device(keys, values, config)


def local_samples(keys, values, base: int, count: int):
    """``count`` rows of (raw key bits, payload, global index, valid) for one shard: evenly spaced
    samples, padded with invalid rows when the shard is shorter than ``count``."""
    import torch

    dev = keys.device
    n_local = keys.numel()
    pos = sample_positions(n_local, min(count, n_local))
    smp = torch.zeros((count, 4), dtype=torch.int64, device=dev)
    if pos.size:
        p = torch.from_numpy(pos).to(dev)
        raw = _raw_bits(keys)[p].to(torch.int64)
        if keys.element_size() == 4:
            raw = raw & 0xFFFFFFFF
        smp[: pos.size, 0] = raw
        if values is not None:
            smp[: pos.size, 1] = values.view(torch.int32)[p].to(torch.int64) & 0xFFFFFFFF
        smp[: pos.size, 2] = p + base
        smp[: pos.size, 3] = n_local  # valid; the shard size weights this rank's samples
    return smp


def valid_samples(rows: np.ndarray) -> np.ndarray:
    return rows[rows[:, 3] > 0][:, :3]


def sample_weights(rows: np.ndarray, per_rank: int) -> np.ndarray:
    """Weight of each valid gathered sample: its shard's size over its shard's sample count."""
    w = []
    for r in range(rows.shape[0] // per_rank):
        blk = rows[r * per_rank:(r + 1) * per_rank]
        v = blk[blk[:, 3] > 0]
        if v.shape[0]:
            w.append(np.full(v.shape[0], float(v[0, 3]) / v.shape[0]))
    return np.concatenate(w) if w else np.empty(0)


# ---- the collective ----------------------------------------------------------------------------

def sample_sort(keys, values=None, group=None, oversample: int = DEFAULT_OVERSAMPLE,
                config: SortConfig = DEFAULT_CONFIG) -> Tuple["torch.Tensor", Optional["torch.Tensor"]]:
    """Sort the array whose shards are the ranks' ``keys`` (+ optional uint32 ``values``).

    Collective over ``group`` (default: the world).  Returns this rank's slice of the sorted array
    as new tensors (its length is the number of elements that fall between this rank's splitters).
    The shards may have different lengths, including 0."""
    import torch
    import torch.distributed as dist

    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    if P > MAX_RANKS:
        raise ValueError(f"sample_sort supports up to {MAX_RANKS} ranks")
    if keys.dim() != 1 or not keys.is_contiguous():
        raise TypeError("keys must be a 1-D contiguous tensor")
    _dtype_code(keys.dtype)
    if values is not None and (values.shape != keys.shape or values.dtype not in (torch.int32, torch.uint32)):
        raise TypeError("values must be an int32/uint32 tensor of the keys' shape")
    dev = keys.device
    n_local = keys.numel()
    width = keys.element_size()
    is_float = keys.dtype in (torch.float32, torch.float64)

    # 1. global index base
    sizes = torch.zeros(P, dtype=torch.int64, device=dev)
    mine = torch.tensor([n_local], dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(sizes, mine, group=group)
    sizes_h = sizes.cpu().tolist()
    base = int(sum(sizes_h[:r]))

    # 2. samples -> splitters (identical on every rank)
    S = oversample * P
    smp = local_samples(keys, values, base, S)
    allsmp = torch.empty((P * S, 4), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allsmp, smp, group=group)
    rows = allsmp.cpu().numpy()
    g = valid_samples(rows)
    splitters = choose_splitters(g, P, width, is_float, sample_weights(rows, S))
    if splitters.shape[0] < P - 1:  # empty input everywhere: all buckets empty
        splitters = np.zeros((P - 1, 3), dtype=np.int64)

    # 3. bucket the shard
    bk, bv, counts = _bucket(keys, values, base, splitters)

    # 4. exchange sizes, then elements
    recv_counts = torch.empty_like(counts)
    dist.all_to_all_single(recv_counts, counts, group=group)
    send = counts.cpu().tolist()
    recv = recv_counts.cpu().tolist()
    total = int(sum(recv))
    out_k = torch.empty(total, dtype=keys.dtype, device=dev)
    dist.all_to_all_single(_raw_bits(out_k), _raw_bits(bk), output_split_sizes=recv, input_split_sizes=send,
                           group=group)
    out_v = None
    if values is not None:
        out_v = torch.empty(total, dtype=values.dtype, device=dev)
        dist.all_to_all_single(out_v.view(torch.int32), bv.view(torch.int32), output_split_sizes=recv,
                               input_split_sizes=send, group=group)  # payload bits as int32 (any backend)

    # 5. local sort of the received slice
    _local_sort(out_k, out_v, config)
    return out_k, out_v
