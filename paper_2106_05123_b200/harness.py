"""Harness integration: the reference's benchmark table and `gen` files
on the B200 sort path.

What a user of the reference's harness gets here:

* ``GPU_ALGORITHM`` — a ``(run, instrumented)`` pair with the exact shape of an entry of the
  reference's algorithm table (``_ALGORITHMS`` in R/pkg/src/pdqsort/bench.py:133-138).  Adding
  ``_ALGORITHMS["gpu"] = GPU_ALGORITHM`` to the reference gives side-by-side CPU/GPU rows in its
  own CSV.  ``run`` is the drop-in ``sort`` on the harness's list;
  ``instrumented`` returns a ``DeviceMetrics`` whose ``counter_values()`` fills the reference's
  ten counter columns from the device counters.
* ``generate`` / ``DistributionSpec`` — the reference's twelve input distributions
  (datagen.py:17-30, 115-146), restated with numpy so that 2^20-element cells generate in
  milliseconds, bit-identical to the reference's lists (pinned by
  tests/golden/datagen_digests.json), plus the GPU element types int32 / float32 / float64.
* ``read_array`` / ``write_array`` — the `gen` file format (datagen.py:164-168): a
  ``# kind n type seed`` header, one value per line.
* ``run_benchmark`` and ``main`` — the reference's ``bench`` / ``gen`` commands
  (cli.py:82-150, bench.py:158-197) for the ``gpu`` algorithm, writing the reference's CSV
  schema unchanged (golden header test_cli.py:10-15).

The product path is the same ``sort`` as everywhere else: CUDA kernels behind the C ABI, no CPU
fallback.  String element types (``str``, ``bigstr``) are out of scope.
"""

from __future__ import annotations

import argparse
import array
import csv
import hashlib
import math
import sys
import time
from dataclasses import dataclass
from typing import IO, Iterable, Optional, Sequence

import numpy as np

from .driver import DEFAULT_CONFIG, sort_device

# ---- schema (bench.py:30-40, instrumentation.py:20-31) ------------------------------------------

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
CSV_COLUMNS = ("algo", "kind", "element_type", "n", "seed", "iterations", "total_ns", "ns_per_nlog2n",
               "input_hash") + METRIC_FIELDS
TIMING_COLUMNS = ("iterations", "total_ns", "ns_per_nlog2n")

DISTRIBUTION_KINDS = ("uniform", "dupsq", "dup8", "mod8", "ones", "sort50", "sort90", "sort99", "organ",
                      "merge", "asc", "desc")
# int64 is the reference's numeric type; the others are the element types the device path sorts
ELEMENT_TYPES = ("int64", "int32", "float32", "float64")
REFERENCE_STRING_TYPES = ("str", "bigstr")

DEFAULT_SIZES = "1024..1048576:4"
DEFAULT_SEED = 0xDE5C


class UsageError(ValueError):
    """Bad harness arguments (unknown algorithm, kind, element type, size or duration)."""


# ---- datagen restatement ------------------------------------------------------------------------

_M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_SHUFFLED = ("uniform", "dupsq", "dup8", "mod8")
_SORTED_PCT = {"sort50": 50, "sort90": 90, "sort99": 99}


def _mix(z: int) -> int:
    """splitmix64 finaliser on a Python int (datagen.py:42-45)."""
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _mix_vec(z: np.ndarray) -> np.ndarray:
    """The same finaliser on a uint64 vector (numpy wraps modulo 2^64)."""
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def stream_seed(seed: int, kind: str, n: int) -> int:
    """Per-(seed, kind, n) generator seed (datagen.py:62-66)."""
    s = _mix((seed + _GOLDEN * (DISTRIBUTION_KINDS.index(kind) + 1)) & _M64)
    return _mix((s + _GOLDEN * (n + 1)) & _M64)


def shuffle_indices(n: int, seed: int) -> np.ndarray:
    """The swap partner of every Fisher-Yates step i = n-1 .. 1 (datagen.py:69-72).

    The generator's k-th draw is mix(seed + k·golden) (datagen.py:54-56), independent of the
    swaps, so all draws are computed at once; ``j[t]`` partners position ``n-1-t``."""
    if n < 2:
        return np.empty(0, np.int64)
    k = np.arange(1, n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        draws = _mix_vec(k * np.uint64(_GOLDEN) + np.uint64(seed & _M64))
    bounds = np.arange(n, 1, -1, dtype=np.uint64)
    return (draws % bounds).astype(np.int64)


def _fisher_yates(values: list, seed: int) -> None:
    j = shuffle_indices(len(values), seed).tolist()
    i = len(values) - 1
    for jj in j:
        values[i], values[jj] = values[jj], values[i]
        i -= 1


def _base(kind: str, n: int) -> np.ndarray:
    """Unshuffled values of each kind (datagen.py:115-137)."""
    i = np.arange(n, dtype=np.int64)
    if kind in ("uniform", "asc") or kind in _SORTED_PCT:
        return i
    if kind == "desc":
        return i[::-1].copy()
    if kind == "dupsq":
        return i % math.isqrt(n)
    if kind == "dup8":
        if n > 1 << 32:  # i*i would leave uint64
            return np.array([(pow(v, 8, n) + n // 2) % n for v in range(n)], dtype=np.int64)
        x = i.astype(np.uint64)
        m = np.uint64(n)
        for _ in range(3):
            x = (x * x) % m
        return ((x + np.uint64(n // 2)) % m).astype(np.int64)
    if kind == "mod8":
        return i % 8
    if kind == "ones":
        return np.ones(n, dtype=np.int64)
    if kind == "organ":
        up = (n + 1) // 2
        return np.concatenate([np.arange(up), np.arange(n - up - 1, -1, -1)]).astype(np.int64)
    if kind == "merge":
        up = (n + 1) // 2
        return np.concatenate([np.arange(up), np.arange(n - up)]).astype(np.int64)
    raise ValueError(f"unknown distribution kind: {kind!r}")


@dataclass(frozen=True)
class DistributionSpec:
    """One input recipe (datagen.py:75-112) over the numeric element types."""

    kind: str
    n: int
    element_type: str = "int64"
    seed: int = 0

    def __post_init__(self):
        if self.kind not in DISTRIBUTION_KINDS:
            raise ValueError(f"unknown distribution kind: {self.kind!r}")
        if self.element_type in REFERENCE_STRING_TYPES:
            raise ValueError(f"element type {self.element_type!r}: string keys are not on the device sort path")
        if self.element_type not in ELEMENT_TYPES:
            raise ValueError(f"unknown element type: {self.element_type!r}")
        if self.n < 0:
            raise ValueError("n must be >= 0")
        if self.element_type == "int32" and self.n > 1 << 31:
            raise ValueError("int32 element type needs n <= 2^31")


def generate_values(spec: DistributionSpec) -> np.ndarray:
    """The spec's values as int64, identical to the reference's ``generate`` (datagen.py:140-157)."""
    n = spec.n
    if n == 0:
        return np.empty(0, np.int64)
    vals = _base(spec.kind, n)
    if spec.kind in _SHUFFLED or spec.kind in _SORTED_PCT:
        seed = stream_seed(spec.seed, spec.kind, n)
        lst = vals.tolist()
        _fisher_yates(lst, seed)
        vals = np.array(lst, dtype=np.int64)
        if spec.kind in _SORTED_PCT:
            k = _SORTED_PCT[spec.kind] * n // 100
            vals[:k].sort()
    return vals


def encode(vals: np.ndarray, element_type: str):
    """The container the harness sorts: a list of Python ints for int64 (the reference's own
    type), ``array.array`` for the 4-byte types, a list of floats for float64."""
    if element_type == "int64":
        return vals.tolist()
    if element_type == "int32":
        return array.array("i", vals.astype(np.int32).tobytes())
    if element_type == "float32":
        return array.array("f", vals.astype(np.float32).tobytes())
    if element_type == "float64":
        return vals.astype(np.float64).tolist()
    raise ValueError(f"unknown element type: {element_type!r}")


def generate(spec: DistributionSpec):
    """``datagen.generate`` for the numeric element types."""
    return encode(generate_values(spec), spec.element_type)


def array_digest(values: Iterable) -> str:
    """sha256 over the newline-joined ``str`` of every value (datagen.py:160-163)."""
    return hashlib.sha256("\n".join(str(v) for v in values).encode("utf-8")).hexdigest()


def write_array(out: IO[str], spec: DistributionSpec, values) -> None:
    """The `gen` file format (datagen.py:164-168)."""
    out.write(f"# {spec.kind} {spec.n} {spec.element_type} {spec.seed}\n")
    for v in values:
        out.write(f"{v}\n")


def read_array(src: IO[str]):
    """Parse a `gen` file (from this module or the reference's ``pdqsort gen``) into its spec and
    container.  Numeric element types only."""
    header = src.readline()
    parts = header.split()
    if len(parts) != 5 or parts[0] != "#":
        raise ValueError(f"not a gen file header: {header.rstrip()!r}")
    kind, n, etype, seed = parts[1], int(parts[2]), parts[3], int(parts[4])
    spec = DistributionSpec(kind, n, etype, seed)
    lines = [ln for ln in (l.strip() for l in src) if ln]
    if len(lines) != n:
        raise ValueError(f"gen file declares {n} values, holds {len(lines)}")
    if etype in ("int64", "int32"):
        vals = np.array([int(x) for x in lines], dtype=np.int64)
        return spec, encode(vals, etype)
    f = np.array([float(x) for x in lines], dtype=np.float64)
    if etype == "float32":
        return spec, array.array("f", f.astype(np.float32).tobytes())
    return spec, f.tolist()


# ---- the gpu algorithm entry (bench.py:86-138 shape) ---------------------------------------------


@dataclass
class DeviceMetrics:
    """The reference's ``Metrics`` columns filled from the device counters (pdq_stats).

    ``comparisons``, ``element_moves``, ``exchanges`` and the partial-insertion counters describe
    scalar operations the device path does not perform one by one (a tile classifies 4096 keys at
    once; the sortedness check K4 replaces partial insertion); they are reported as 0.
    ``heapsort_fallbacks`` counts the K5 radix-exchange fallbacks that stand where heapsort does
    (DESIGN.md §3)."""

    comparisons: int = 0
    element_moves: int = 0
    exchanges: int = 0
    partition_right_calls: int = 0
    partition_left_calls: int = 0
    bad_partitions: int = 0
    heapsort_fallbacks: int = 0
    partial_insertion_attempts: int = 0
    partial_insertion_aborts: int = 0
    max_depth: int = 0

    def counter_values(self) -> tuple:
        return tuple(getattr(self, f) for f in METRIC_FIELDS)

    @classmethod
    def from_stats(cls, st: Optional[dict]) -> "DeviceMetrics":
        if not st:
            return cls()
        return cls(partition_right_calls=st["partition_right_calls"],
                   partition_left_calls=st["partition_left_calls"],
                   bad_partitions=st["bad_partitions"], heapsort_fallbacks=st["radix_fallbacks"],
                   max_depth=st["max_depth"])


_NP_OF = {"i": np.int32, "l": np.int64, "q": np.int64, "f": np.float32, "d": np.float64}


def _to_numpy(values) -> np.ndarray:
    if isinstance(values, array.array):
        return np.frombuffer(values, dtype=_NP_OF[values.typecode]).copy()
    if values and isinstance(values[0], float):
        return np.array(values, dtype=np.float64)
    return np.array(values, dtype=np.int64)


def _sort_with_stats(values) -> dict:
    """Device sort of the harness's container in place, returning the device counters."""
    import torch

    if len(values) == 0:
        return {}
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 sort path has no CPU fallback")
    host = _to_numpy(values)
    dev = torch.from_numpy(host).cuda()
    st = sort_device(dev, None, DEFAULT_CONFIG)
    out = dev.cpu().numpy()
    if isinstance(values, array.array):
        values[:] = array.array(values.typecode, out.tobytes())
    else:
        values[:] = out.tolist()
    return st


def run_gpu(values) -> None:
    """Timed leg: the drop-in ``sort`` on the harness's container (driver.py:267)."""
    from .driver import sort

    sort(values)


def instrumented_gpu(values) -> DeviceMetrics:
    """Counter leg: the same device sort, its counters in the reference's columns."""
    return DeviceMetrics.from_stats(_sort_with_stats(values))


GPU_ALGORITHM = (run_gpu, instrumented_gpu)
_ALGORITHMS = {"gpu": GPU_ALGORITHM}


# ---- benchmark table (bench.py:49-197) ------------------------------------------------------------


@dataclass(frozen=True)
class BenchPolicy:
    min_time: float = 1.0
    min_iterations: int = 10


@dataclass
class BenchmarkRecord:
    algo: str
    kind: str
    element_type: str
    n: int
    seed: int
    iterations: int
    total_ns: int
    ns_per_nlog2n: float
    input_hash: str
    metrics: DeviceMetrics

    def row(self) -> list:
        return [self.algo, self.kind, self.element_type, self.n, self.seed, self.iterations, self.total_ns,
                f"{self.ns_per_nlog2n:.6f}", self.input_hash, *self.metrics.counter_values()]


def resolve_algo(name: str) -> str:
    if name not in _ALGORITHMS:
        raise UsageError(f"unknown algorithm: {name!r} (choose from {', '.join(_ALGORITHMS)})")
    return name


def run_benchmark(algos: Sequence[str], specs: Iterable[DistributionSpec],
                  policy: BenchPolicy = BenchPolicy(), verify: bool = True) -> list:
    """Every (spec, algo) cell in order, the reference's timing rule (bench.py:171-181): each
    iteration sorts a freshly generated input, until both floors are met; then one counter pass.
    ``verify`` checks every counter-pass output against numpy's sort of the same input."""
    names = [resolve_algo(a) for a in algos]
    for algo in names:  # one untimed call: CUDA context and library load are per process, not per cell
        _ALGORITHMS[algo][0]([2, 1])
    records = []
    for spec in specs:
        base = generate_values(spec)
        for algo in names:
            run, instr = _ALGORITHMS[algo]
            total_ns, iters = 0, 0
            floor_ns = int(policy.min_time * 1e9)
            while total_ns < floor_ns or iters < policy.min_iterations:
                vals = encode(base, spec.element_type)
                t0 = time.perf_counter_ns()
                run(vals)
                total_ns += time.perf_counter_ns() - t0
                iters += 1
            vals = encode(base, spec.element_type)
            digest = array_digest(vals)
            metrics = instr(vals)
            if verify:
                want = np.sort(_to_numpy(encode(base, spec.element_type)), kind="stable")
                if not np.array_equal(_to_numpy(vals), want):
                    raise RuntimeError(f"{algo} produced an unsorted output for {spec}")
            nl = spec.n * math.log2(spec.n) if spec.n >= 2 else 0.0
            records.append(BenchmarkRecord(algo, spec.kind, spec.element_type, spec.n, spec.seed, iters,
                                           total_ns, total_ns / (iters * nl) if nl else 0.0, digest, metrics))
    return records


def format_text_tables(records: Sequence[BenchmarkRecord]) -> str:
    """One ns/(n log2 n) table per (kind, element type), as bench.py:209-237 prints."""
    lines = []
    groups = list(dict.fromkeys((r.kind, r.element_type) for r in records))
    for kind, etype in groups:
        rows = [r for r in records if (r.kind, r.element_type) == (kind, etype)]
        algos = list(dict.fromkeys(r.algo for r in rows))
        widths = [12] + [max(18, len(a) + 2) for a in algos]
        lines.append(f"{kind} / {etype}  (ns per n log2 n)")
        lines.append("".join(f"{h:>{w}}" for h, w in zip(["n"] + algos, widths)))
        for n in sorted({r.n for r in rows}):
            cells = [f"{n:>{widths[0]}}"]
            for a, w in zip(algos, widths[1:]):
                hit = [r for r in rows if r.n == n and r.algo == a]
                cells.append(f"{hit[0].ns_per_nlog2n:>{w}.3f}" if hit else " " * w)
            lines.append("".join(cells))
        lines.append("")
    return "\n".join(lines)


# ---- command line (cli.py) -------------------------------------------------------------------------


def parse_list(text: str) -> list:
    return [p.strip() for p in text.split(",") if p.strip()]


def parse_sizes(text: str) -> list:
    """Comma list of sizes; ``A..B`` doubles, ``A..B:K`` multiplies by K (cli.py:45-66)."""
    out = []
    for part in parse_list(text):
        try:
            if ".." in part:
                span, _, factor = part.partition(":")
                lo_s, _, hi_s = span.partition("..")
                lo, hi, step = int(lo_s), int(hi_s), int(factor) if factor else 2
                if lo < 1 or hi < lo or step < 2:
                    raise UsageError(f"bad size range: {part!r}")
                v = lo
                while v <= hi:
                    out.append(v)
                    v *= step
            else:
                v = int(part)
                if v < 0:
                    raise UsageError(f"bad size: {part!r}")
                out.append(v)
        except ValueError as e:
            if isinstance(e, UsageError):
                raise
            raise UsageError(f"bad size: {part!r}") from None
    if not out:
        raise UsageError("no sizes given")
    return out


def parse_duration(text: str) -> float:
    t = text.strip()
    try:
        if t.endswith("ms"):
            return float(t[:-2]) / 1000.0
        return float(t[:-1]) if t.endswith("s") else float(t)
    except ValueError:
        raise UsageError(f"bad duration: {text!r}") from None


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1, as the reference's CLI (cli.py:33-38)
        self.print_usage(sys.stderr)
        self.exit(1, f"{self.prog}: error: {message}\n")


def _parser() -> _Parser:
    p = _Parser(prog="pdqsort-gpu", description=__doc__.splitlines()[0])
    sub = p.add_subparsers(dest="command", required=True)
    b = sub.add_parser("bench")
    b.add_argument("--algos", default="gpu")
    b.add_argument("--dists", default=",".join(DISTRIBUTION_KINDS))
    b.add_argument("--sizes", default=DEFAULT_SIZES)
    b.add_argument("--types", default="int64")
    b.add_argument("--seed", type=int, default=DEFAULT_SEED)
    b.add_argument("--min-time", default="1s")
    b.add_argument("--min-iters", type=int, default=10)
    b.add_argument("--out", default="-")
    b.add_argument("--tables", action="store_true")
    g = sub.add_parser("gen")
    g.add_argument("--kind", required=True)
    g.add_argument("--n", type=int, required=True)
    g.add_argument("--type", default="int64", dest="element_type")
    g.add_argument("--seed", type=int, default=DEFAULT_SEED)
    g.add_argument("--out", default="-")
    s = sub.add_parser("sort", help="sort a gen file on the GPU and write it back in the gen format")
    s.add_argument("path")
    s.add_argument("--out", default="-")
    return p


def _emit(path: str, fn) -> None:
    if path == "-":
        fn(sys.stdout)
    else:
        with open(path, "w", encoding="utf-8", newline="") as f:
            fn(f)


def _cmd_bench(a) -> int:
    specs = [DistributionSpec(k, n, t, a.seed) for t in parse_list(a.types) for k in parse_list(a.dists)
             for n in parse_sizes(a.sizes)]
    pol = BenchPolicy(parse_duration(a.min_time), a.min_iters)
    if pol.min_iterations < 1:
        raise UsageError("--min-iters must be >= 1")
    algos = [resolve_algo(x) for x in parse_list(a.algos)]
    recs = run_benchmark(algos, specs, pol)

    def write(out):
        w = csv.writer(out, lineterminator="\n")
        w.writerow(CSV_COLUMNS)
        for r in recs:
            w.writerow(r.row())

    _emit(a.out, write)
    if a.tables:
        sys.stdout.write(format_text_tables(recs))
    return 0


def _cmd_gen(a) -> int:
    spec = DistributionSpec(a.kind, a.n, a.element_type, a.seed)
    vals = generate(spec)
    _emit(a.out, lambda out: write_array(out, spec, vals))
    return 0


def _cmd_sort(a) -> int:
    with open(a.path, encoding="utf-8") as f:
        spec, vals = read_array(f)
    run_gpu(vals)
    _emit(a.out, lambda out: write_array(out, spec, vals))
    return 0


def main(argv=None) -> int:
    p = _parser()
    try:
        a = p.parse_args(argv)
    except SystemExit as e:
        return e.code if isinstance(e.code, int) else 1
    try:
        return {"bench": _cmd_bench, "gen": _cmd_gen, "sort": _cmd_sort}[a.command](a)
    except (UsageError, ValueError) as e:
        print(f"pdqsort-gpu: error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
