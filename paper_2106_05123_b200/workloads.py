"""Seeded synthetic inputs for the five BASELINE configs and the roofline input.

The reference ships no datasets for this path: BASELINE.json defines its
configs as formulas, and SURVEY.md §8(d) fixes the recipes below.  Every
generator is a pure function of (config, n) through numpy's PCG64 so the
GPU path, the CPU oracle and the Python reference see identical bytes on
any host.  The organ-pipe shape follows the reference's own formula
(pkg/src/pdqsort/datagen.py:121-123); asc/desc follow datagen.py:107-110.

Returned arrays are host numpy arrays.  KV configs return ``(keys, values)``.
"""

from __future__ import annotations

import numpy as np

SEED = 210605123

C2_KINDS = ("asc", "desc", "organ", "asc_tail", "asc_swaps")
C3_KS = (1, 2, 16, 256, 65536)
C4_KINDS = ("normal", "normal_half10")

FULL_N = {"C1": 1 << 20, "C2": 1 << 24, "C3": 1 << 26, "C4": 1 << 26, "C5": 1 << 28, "R": 1 << 28}


def _rng(offset: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED + offset))


def uniform_i32(n: int, offset: int = 1) -> np.ndarray:
    """C1 / R: i.i.d. uniform over the full int32 range (INT32_MIN included)."""
    return _rng(offset).integers(-(2**31), 2**31, n, dtype=np.int64).astype(np.int32)


def c1(n: int = FULL_N["C1"]) -> np.ndarray:
    return uniform_i32(n, 1)


def roofline_input(n: int = FULL_N["R"]) -> np.ndarray:
    return uniform_i32(n, 6)


def c2(kind: str, n: int = FULL_N["C2"]) -> np.ndarray:
    """C2 pattern set, int32, keys-only."""
    rng = _rng(2)
    if kind == "asc":
        return np.arange(n, dtype=np.int32)
    if kind == "desc":
        return np.arange(n, dtype=np.int32)[::-1].copy()
    if kind == "organ":  # datagen.py:121-123
        up = (n + 1) // 2
        return np.concatenate(
            [np.arange(up, dtype=np.int32), np.arange(n - up - 1, -1, -1, dtype=np.int32)]
        )
    if kind == "asc_tail":
        a = np.arange(n, dtype=np.int32)
        t = n // 100
        if t:
            a[n - t :] = rng.integers(-(2**31), 2**31, t, dtype=np.int64).astype(np.int32)
        return a
    if kind == "asc_swaps":
        a = np.arange(n, dtype=np.int32)
        pairs = rng.integers(0, max(n, 1), (n // 100, 2))
        for i, j in pairs.tolist():  # sequential swaps, order matters
            a[i], a[j] = a[j], a[i]
        return a
    raise ValueError(f"unknown C2 kind {kind!r}")


def c3(k: int, n: int = FULL_N["C3"]) -> np.ndarray:
    """C3: k distinct uniform int32 values, then n uniform draws among them."""
    rng = _rng(3)
    uniq = np.unique(rng.integers(-(2**31), 2**31, 2 * k + 64, dtype=np.int64))
    while uniq.size < k:  # pragma: no cover - astronomically unlikely
        uniq = np.unique(np.concatenate([uniq, rng.integers(-(2**31), 2**31, k, dtype=np.int64)]))
    vals = uniq[rng.permutation(uniq.size)[:k]].astype(np.int32)
    return vals[rng.integers(0, k, n)]


def c4(kind: str, n: int = FULL_N["C4"]) -> np.ndarray:
    """C4: float32 N(0,1), exact zeros -> 1e-30 (no -0.0, no NaN); variant
    with n//10 distinct positions set to 0.5."""
    rng = _rng(4)
    x = rng.standard_normal(n, dtype=np.float32)
    x[x == 0] = np.float32(1e-30)
    if kind == "normal":
        return x
    if kind == "normal_half10":
        idx = rng.choice(n, n // 10, replace=False)
        x[idx] = np.float32(0.5)
        return x
    raise ValueError(f"unknown C4 kind {kind!r}")


def c5(n: int = FULL_N["C5"]):
    """C5: distinct int64 keys (permutation * 2^20 + low offset) carrying a
    uint32 payload equal to the original index."""
    rng = _rng(5)
    keys = rng.permutation(n).astype(np.int64) * (1 << 20) + rng.integers(0, 1 << 20, n)
    vals = np.arange(n, dtype=np.uint32)
    return keys, vals


def cases(scale_shift: int = 0):
    """All parity cases as (name, keys, values-or-None) at FULL_N >> scale_shift."""
    def sz(c):
        return max(FULL_N[c] >> scale_shift, 1)

    yield "C1", c1(sz("C1")), None
    for kind in C2_KINDS:
        yield f"C2.{kind}", c2(kind, sz("C2")), None
    for k in C3_KS:
        yield f"C3.k{k}", c3(k, sz("C3")), None
    for kind in C4_KINDS:
        yield f"C4.{kind}", c4(kind, sz("C4")), None
    k, v = c5(sz("C5"))
    yield "C5", k, v


def stratified_adversary(n: int, seed: int = 7) -> np.ndarray:
    """A permutation of 0..n-1 (int32) against the root's pivot rule (K1): the positions the root
    samples -- (2i + 1) n / (2 S), S = 256 for n >= 2^20, else 64 -- hold the S smallest values, so the
    root's pivot is the (S/2)-th smallest key and its partition is bad (min(L, R) < n / 8).  Deeper
    segments cannot be targeted from the input: a partition places its tiles' runs in the order their
    reservations arrive, so a child's sample positions hold keys no input layout controls (the
    reference's deterministic adversary, instrumentation.adversary_input, has no GPU analogue)."""
    ns = 256 if n >= (1 << 20) else 64
    rng = _rng(seed)
    out = np.empty(n, dtype=np.int64)
    pos = ((2 * np.arange(ns, dtype=np.int64) + 1) * n) // (2 * ns)
    mask = np.ones(n, dtype=bool)
    mask[pos] = False
    out[pos] = np.arange(ns)
    out[mask] = ns + rng.permutation(n - ns)
    return out.astype(np.int32)


def make(name: str, n: int):
    """Build one named case (as listed by :func:`cases`) at size n."""
    if name == "C1":
        return c1(n), None
    if name == "R":
        return roofline_input(n), None
    if name.startswith("C2."):
        return c2(name[3:], n), None
    if name.startswith("C3.k"):
        return c3(int(name[4:]), n), None
    if name.startswith("C4."):
        return c4(name[3:], n), None
    if name == "C5":
        return c5(n)
    raise ValueError(name)


def expected(keys: np.ndarray, values=None):
    """The unique sorted output: np.sort for keys-only, lexicographic
    (key, payload) order for KV -- exactly what the reference's
    ``sort(list(zip(keys, values)))`` produces (tuples compare
    lexicographically)."""
    if values is None:
        return np.sort(keys, kind="stable"), None
    order = np.lexsort((values, keys))
    return keys[order], values[order]
