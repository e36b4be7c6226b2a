"""ctypes binding of the C ABI in include/pdq_b200.h (libpdq_b200.so, built in-tree).

There is no fallback: if the shared library is missing, every sort raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.environ.get("PDQ_LIB") or os.path.join(HERE, "libpdq_b200.so")
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")

PDQ_I32, PDQ_I64, PDQ_F32, PDQ_F64 = 0, 1, 2, 3

STATUS = {
    0: "PDQ_OK",
    -1: "PDQ_ERR_CONFIG",
    -2: "PDQ_ERR_DTYPE",
    -3: "PDQ_ERR_ALIGN",
    -4: "PDQ_ERR_WORKSPACE",
    -5: "PDQ_ERR_CUDA",
    -6: "PDQ_ERR_INTERNAL",
    -7: "PDQ_ERR_ARG",
}

# every symbol include/pdq_b200.h declares
EXPORTS = (
    "pdq_config_default",
    "pdq_config_validate",
    "pdq_workspace_bytes",
    "pdq_sort",
    "pdq_sort_ex",
    "pdq_sort_timed",
    "pdq_sort_finish",
    "pdq_last_error",
    "pdq_version",
    "pdq_bucket_workspace_bytes",
    "pdq_bucket",
    "pdq_host_sorter_create",
    "pdq_host_sorter_destroy",
    "pdq_host_sort",
    "pdq_host_sorter_error",
)


class PdqConfig(ctypes.Structure):
    """POD mirror of pdq_config (include/pdq_b200.h)."""

    _fields_ = [
        ("insertion_threshold", ctypes.c_int64),
        ("ninther_threshold", ctypes.c_int64),
        ("partial_insertion_budget", ctypes.c_int64),
        ("block_size", ctypes.c_int64),
        ("bad_partition_shift", ctypes.c_int64),
        ("use_block_partition", ctypes.c_int32),
        ("use_partition_left", ctypes.c_int32),
        ("use_break_patterns", ctypes.c_int32),
        ("use_partial_insertion", ctypes.c_int32),
        ("base_case_size", ctypes.c_int32),
        ("bad_budget", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 4),
    ]


STAT_FIELDS = (
    "partition_right_calls",
    "partition_left_calls",
    "bad_partitions",
    "radix_fallbacks",
    "base_cases",
    "max_depth",
    "tiles",
    "bytes_algorithmic",
    "check_result",
    "segments",
    "status",
    "bytes_check",
    "cycles_wait",
    "cycles_work",
    "cycles_base",
    "cycles_spawn",
    "sched_retire",
    "sched_claim",
    "sched_fetch",
    "sched_idle",
    "bytes_base",
    "sort_ns",
    "base_ns",
    "run_split",
)


class PdqStats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in STAT_FIELDS]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f in STAT_FIELDS}


NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
]

# One translation unit per element type (pdq_inst.cu compiled eight times) so the instantiations of the
# persistent sorter and the leaf kernels build in parallel; (object name, source, extra -D flags)
_INST = [
    ("i32", "launch_i32", "uint32_t", "false", "false"),
    ("i32_kv", "launch_i32_kv", "uint32_t", "false", "true"),
    ("f32", "launch_f32", "uint32_t", "true", "false"),
    ("f32_kv", "launch_f32_kv", "uint32_t", "true", "true"),
    ("i64", "launch_i64", "uint64_t", "false", "false"),
    ("i64_kv", "launch_i64_kv", "uint64_t", "false", "true"),
    ("f64", "launch_f64", "uint64_t", "true", "false"),
    ("f64_kv", "launch_f64_kv", "uint64_t", "true", "true"),
]
BUILD_DIR = os.path.join(HERE, "_build")


def translation_units(only_i32: bool = False):
    """(object stem, source file, -D flags) of every translation unit of libpdq_b200.so."""
    units = [("capi", "pdq_capi.cu", ["-DPDQ_ONLY_I32"] if only_i32 else []),
             ("host", "pdq_host.cu", []),
             ("bucket", "pdq_bucket_capi.cu", [])]
    for stem, name, u, fl, kv in (_INST[:1] if only_i32 else _INST):
        units.append((f"inst_{stem}", "pdq_inst.cu",
                      [f"-DPDQ_INST_NAME={name}", f"-DPDQ_INST_U={u}", f"-DPDQ_INST_FLOAT={fl}", f"-DPDQ_INST_KV={kv}"]))
    return units


_lock = threading.Lock()
_lib = None


def build(verbose: bool = False, out: str = None, extra_flags=(), only_i32: bool = False, jobs: int = 0) -> str:
    """Compile csrc/ into libpdq_b200.so for sm_100a (nvcc cross-compiles without a GPU): the
    translation units are compiled in parallel into _build/*.o (an object newer than every source and
    header, built with the same flags, is reused) and linked into one shared library."""
    from concurrent.futures import ThreadPoolExecutor

    nvcc = os.environ.get("NVCC", "nvcc")
    if not os.path.exists(nvcc) and os.path.exists("/usr/local/cuda/bin/nvcc"):
        nvcc = "/usr/local/cuda/bin/nvcc"
    out = out or LIB_PATH
    tag = "" if out == LIB_PATH else "_" + os.path.splitext(os.path.basename(out))[0]
    os.makedirs(BUILD_DIR, exist_ok=True)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)]
    newest = max(os.path.getmtime(f) for f in deps)
    flags = [*NVCC_FLAGS, *extra_flags] + (["-Xptxas=-v"] if verbose else [])

    def compile_one(unit):
        stem, src, defs = unit
        obj = os.path.join(BUILD_DIR, f"{stem}{tag}.o")
        cmd = [nvcc, *flags, *defs, "-I", INCLUDE, "-c", os.path.join(CSRC, src), "-o", obj]
        stamp = obj + ".cmd"
        line = " ".join(cmd)
        if (os.path.exists(obj) and os.path.getmtime(obj) >= newest and os.path.exists(stamp)
                and open(stamp).read() == line):
            return obj, ""
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src} ({stem}):\n{r.stdout}\n{r.stderr}")
        with open(stamp, "w") as f:
            f.write(line)
        return obj, r.stdout + r.stderr

    units = translation_units(only_i32)
    with ThreadPoolExecutor(max_workers=jobs or min(len(units), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, units))
    if verbose:
        for (stem, _, _), (_, log) in zip(units, results):
            if log:
                print(f"== {stem}\n{log}")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out,
                    *[obj for obj, _ in results]], check=True)
    return out


def lib() -> ctypes.CDLL:
    """Load the in-tree shared library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            P, I64, I, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
            L.pdq_config_default.argtypes = [ctypes.POINTER(PdqConfig)]
            L.pdq_config_default.restype = None
            L.pdq_config_validate.argtypes = [ctypes.POINTER(PdqConfig)]
            L.pdq_config_validate.restype = I
            L.pdq_workspace_bytes.argtypes = [I, I, I64]
            L.pdq_workspace_bytes.restype = SZ
            L.pdq_sort.argtypes = [P, I, P, I64, ctypes.POINTER(PdqConfig), P, SZ, P]
            L.pdq_sort.restype = I
            L.pdq_sort_ex.argtypes = [P, I, P, I64, ctypes.POINTER(PdqConfig), P, SZ, P, P, P]
            L.pdq_sort_ex.restype = I
            L.pdq_sort_timed.argtypes = [P, I, P, I64, ctypes.POINTER(PdqConfig), P, SZ, P, ctypes.POINTER(P)]
            L.pdq_sort_timed.restype = I
            L.pdq_sort_finish.argtypes = [P, ctypes.POINTER(PdqStats), P]
            L.pdq_sort_finish.restype = I
            L.pdq_bucket_workspace_bytes.argtypes = [I64, I]
            L.pdq_bucket_workspace_bytes.restype = SZ
            L.pdq_bucket.argtypes = [P, I, P, I64, I64, P, P, P, I, P, P, P, P, SZ, P]
            L.pdq_bucket.restype = I
            L.pdq_host_sorter_create.argtypes = [I, I]
            L.pdq_host_sorter_create.restype = P
            L.pdq_host_sorter_destroy.argtypes = [P]
            L.pdq_host_sorter_destroy.restype = None
            L.pdq_host_sort.argtypes = [P, P, I, P, I64, ctypes.POINTER(PdqConfig), ctypes.POINTER(PdqStats),
                                        ctypes.POINTER(ctypes.c_double)]
            L.pdq_host_sort.restype = I
            L.pdq_host_sorter_error.argtypes = [P]
            L.pdq_host_sorter_error.restype = ctypes.c_char_p
            L.pdq_last_error.argtypes = []
            L.pdq_last_error.restype = ctypes.c_char_p
            L.pdq_version.argtypes = []
            L.pdq_version.restype = ctypes.c_char_p
            _lib = L
    return _lib


def last_error() -> str:
    return lib().pdq_last_error().decode()
