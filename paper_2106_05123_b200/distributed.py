"""Multi-GPU sample sort: one process per GPU, one exchange step.

The reference is single-process (its sort is `driver.py:267-292` on one sequence); this is the
scale-out the survey plans for arrays larger than one GPU's HBM or sorts spread over a node:

1. every rank draws ``oversample · P`` evenly spaced samples of its shard, each tagged with its
   global position key ``rank << 40 | local index`` (the global index order, without exchanging
   shard sizes first) and its shard's size;
2. one all-gather of the samples; every rank orders the same P · S samples on the device by
   (key, payload, position) and picks the same P − 1 splitters at the quantiles of the samples
   weighted by their shards' sizes (a short shard counts for little);
3. ``pdq_bucket`` (CUDA, csrc/pdq_bucket.cuh) splits the local shard into P buckets by those
   splitters, ties broken by position so even an all-equal input spreads evenly;
4. an all-to-all of the bucket sizes (the one host round trip: NCCL's all-to-all takes its split
   sizes on the host), then one all-to-all of keys (and payload): rank r receives bucket r of every
   rank;
5. the received elements are sorted in place by the single-GPU sort (``sort_device``).

Rank r's output is the r-th slice of the global sort; the concatenation over ranks in rank order is
the whole array sorted.  Equal elements are bit-identical (keys) or identical pairs, so the result
is the unique sorted array and parity with the single-GPU sort is bit-exact.

Device work (sampling, splitter choice, bucketing, exchange, local sort) runs in CUDA and NCCL;
``choose_splitters`` is the numpy statement of the splitter rule the device code follows (tests).
There is no CPU fallback: the bucketing and the local sort raise without the CUDA library.
"""

from __future__ import annotations

import ctypes
from typing import Optional, Tuple

import numpy as np

from . import _lib
from .driver import DEFAULT_CONFIG, SortConfig, _dtype_code, _raise, sort_device

DEFAULT_OVERSAMPLE = 256
MAX_RANKS = 64  # buckets per pdq_bucket call
POS_SHIFT = 40  # global position key of an element: rank << POS_SHIFT | local index


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
    if isinstance(splitters, np.ndarray):
        splitters = torch.from_numpy(np.ascontiguousarray(splitters, dtype=np.int64)).to(dev)
    sp = splitters.to(device=dev, dtype=torch.int64)
    if width == 4:  # raw 32-bit patterns held in the low half of int64
        sk = (sp[:, 0] & 0xFFFFFFFF).to(torch.int32) if sp.shape[0] else torch.empty(0, dtype=torch.int32, device=dev)
        sk = sk.contiguous().view(keys.dtype)
    else:
        sk = sp[:, 0].contiguous().view(keys.dtype)
    sv = (sp[:, 1] & 0xFFFFFFFF).to(torch.int32).contiguous()
    sg = sp[:, 2].contiguous()
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


def sortable_i64(raw, width: int, is_float: bool):
    """int64 tensor whose signed order is the sort's key order, for raw bit patterns given as int64
    (4-byte keys in the low 32 bits): the device twin of ``ordered_image``."""
    import torch

    if width == 4:
        x = raw & 0xFFFFFFFF
        if is_float:
            return torch.where(x >= 0x80000000, (~x) & 0xFFFFFFFF, x ^ 0x80000000)
        return x ^ 0x80000000
    if is_float:  # IEEE total order: negatives reversed
        return torch.where(raw < 0, raw ^ 0x7FFFFFFFFFFFFFFF, raw)
    return raw


def device_splitters(rows, nranks: int, per_rank: int, width: int, is_float: bool):
    """The P − 1 splitters (rows of (raw key bits, payload, position key), int64, on the device) from
    the gathered sample rows (raw, payload, position, shard size; shard size 0 = padding): the rule of
    ``choose_splitters`` with weights = shard size / the shard's sample count, computed without
    leaving the device.  Padding rows sort last with weight 0, so they are never picked while any
    sample is valid."""
    import torch

    if nranks <= 1:
        return torch.empty((0, 3), dtype=torch.int64, device=rows.device)
    valid = rows[:, 3] > 0
    big = torch.iinfo(torch.int64).max
    skey = torch.where(valid, sortable_i64(rows[:, 0], width, is_float), torch.full_like(rows[:, 0], big))
    pay = torch.where(valid, rows[:, 1], torch.full_like(rows[:, 1], big))
    pos = torch.where(valid, rows[:, 2], torch.full_like(rows[:, 2], big))
    # weight of a sample: its shard's size over its shard's count of valid samples
    per = valid.view(nranks, per_rank).sum(dim=1, keepdim=True).clamp(min=1)
    w = torch.where(valid.view(nranks, per_rank), rows[:, 3].view(nranks, per_rank).double() / per.double(),
                    torch.zeros((nranks, per_rank), dtype=torch.float64, device=rows.device)).view(-1)
    order = torch.sort(pos, stable=True).indices
    order = order[torch.sort(pay[order], stable=True).indices]
    order = order[torch.sort(skey[order], stable=True).indices]
    ws = w[order]
    cum = torch.cumsum(ws, 0)
    excl = cum - ws
    tot = cum[-1]
    targets = torch.arange(1, nranks, device=rows.device, dtype=torch.float64) * (tot / nranks) * (1 + 1e-12)
    picks = (torch.searchsorted(excl.contiguous(), targets, right=True) - 1).clamp(min=0)
    return rows[order[picks]][:, :3].contiguous()


def local_samples(keys, values, base: int, count: int):
    """``count`` rows of (raw key bits, payload, global position, shard size) for one shard: evenly
    spaced samples, padded with rows of shard size 0 when the shard is shorter than ``count``."""
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
    if n_local >= 1 << POS_SHIFT:
        raise ValueError(f"shards of up to 2^{POS_SHIFT} elements")
    width = keys.element_size()
    is_float = keys.dtype in (torch.float32, torch.float64)

    # 1-2. samples -> splitters on the device (identical on every rank); positions are
    # rank << POS_SHIFT | local index, ordered like global indices without a size exchange
    base = r << POS_SHIFT
    S = oversample * P
    smp = local_samples(keys, values, base, S)
    allsmp = torch.empty((P * S, 4), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allsmp, smp, group=group)
    splitters = device_splitters(allsmp, P, S, width, is_float)

    # 3. bucket the shard
    bk, bv, counts = _bucket(keys, values, base, splitters)

    # 4. exchange sizes (the one host round trip), then elements
    recv_counts = torch.empty_like(counts)
    dist.all_to_all_single(recv_counts, counts, group=group)
    both = torch.stack([counts, recv_counts]).cpu()
    send = both[0].tolist()
    recv = both[1].tolist()
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
