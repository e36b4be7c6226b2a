"""Pattern-defeating quicksort, B200-native (sm_100a).

Drop-in for the reference's sort entry point (pkg/src/pdqsort/__init__.py:19-29,
driver.py:267-292): ``sort``, ``sort_with``, ``sort_with_config``,
``SortConfig``, ``DEFAULT_CONFIG``, ``is_bad_partition``.  The sort runs in
hand-written CUDA kernels behind the C ABI of include/pdq_b200.h; there is no
CPU fallback.
"""

from .driver import (
    DEFAULT_CONFIG,
    MIN_BREAK_SIZE,
    Metrics,
    DeviceSorter,
    FieldOrder,
    HostPipeline,
    HostSorter,
    SortConfig,
    by_field,
    host_sorter,
    instrumented_sort,
    is_bad_partition,
    sort,
    sort_device,
    sort_with,
    sort_with_config,
)

__version__ = "0.1.0"

__all__ = [
    "DEFAULT_CONFIG",
    "DeviceSorter",
    "FieldOrder",
    "HostPipeline",
    "HostSorter",
    "MIN_BREAK_SIZE",
    "Metrics",
    "SortConfig",
    "by_field",
    "host_sorter",
    "instrumented_sort",
    "is_bad_partition",
    "sort",
    "sort_device",
    "sort_with",
    "sort_with_config",
]
