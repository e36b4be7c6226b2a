/* pdq_b200.h — C ABI of the B200 (sm_100a) pattern-defeating-quicksort sort path.
 *
 * This library replaces the reference's sort entry point for flat numeric
 * keys: pkg/src/pdqsort/driver.py:267-270 (sort), :273-279 (sort_with),
 * :282-292 (sort_with_config), all of which funnel into _sort_range
 * (driver.py:167-264) with the built-in ordering `operator.lt`.  The
 * reference is pure Python and has no FFI; INTEGRATION.md shows the ctypes
 * binding a maintainer adds to driver.py to route `sort()` here.
 *
 * Ordering.  Keys are sorted ascending under '<'.  With a payload, elements
 * are (key, payload) pairs ordered lexicographically — exactly how the
 * reference orders the list of (key, payload) tuples it is handed for the KV
 * config (driver.py:267 on tuples).  Float keys are ordered by the IEEE total
 * order (-0.0 before +0.0; NaNs with the sign bit set first, others last);
 * for NaN-free input without mixed signed zeros this is identical to '<'.
 *
 * All calls are stream-ordered and asynchronous: pdq_sort() enqueues work on
 * `stream` and returns.  pdq_sort_finish() synchronises the stream and
 * returns the device-side status and counters.  No global mutable state: two
 * sorts may run concurrently on different streams with different workspaces.
 */
#ifndef PDQ_B200_H
#define PDQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Key dtypes.  The reference sorts Python ints/floats; the GPU path covers the
 * fixed-width numeric types of BASELINE.json plus float64. */
enum pdq_dtype { PDQ_I32 = 0, PDQ_I64 = 1, PDQ_F32 = 2, PDQ_F64 = 3 };

/* Return codes.  The Python layer maps them onto the reference's exception
 * types: config -> ValueError (driver.py:65-75), dtype/layout -> TypeError,
 * CUDA -> RuntimeError. */
enum pdq_status {
    PDQ_OK = 0,
    PDQ_ERR_CONFIG = -1,     /* SortConfig rule violated (driver.py:65-75) */
    PDQ_ERR_DTYPE = -2,      /* unsupported dtype */
    PDQ_ERR_ALIGN = -3,      /* keys/payload not 16-byte aligned */
    PDQ_ERR_WORKSPACE = -4,  /* workspace NULL or smaller than pdq_workspace_bytes() */
    PDQ_ERR_CUDA = -5,       /* a CUDA runtime call failed; see pdq_last_error() */
    PDQ_ERR_INTERNAL = -6,   /* device-side capacity/invariant failure (reported by finish) */
    PDQ_ERR_ARG = -7         /* bad argument (negative n, NULL keys with n > 0, ...) */
};

/* POD mirror of SortConfig (driver.py:47-78) plus the GPU tunables.
 * The first nine fields keep the reference's names, defaults and validation;
 * SURVEY.md §8(b) gives each one's GPU meaning. */
typedef struct pdq_config {
    int64_t insertion_threshold;      /* 24: validated only (>= 3)                     driver.py:55 */
    int64_t ninther_threshold;        /* 128: validated only (>= max(8, ins. thresh.)) driver.py:56 */
    int64_t partial_insertion_budget; /* 8: validated only (>= 0)                      driver.py:57 */
    int64_t block_size;               /* 64: validated only (>= 1)                     driver.py:58 */
    int64_t bad_partition_shift;      /* 3: bad iff min(L,R) < size >> shift           driver.py:59,116-124 */
    int32_t use_block_partition;      /* no-op: the GPU partition is always branchless driver.py:60 */
    int32_t use_partition_left;       /* enables the equal-key partition_left split    driver.py:61,222 */
    int32_t use_break_patterns;       /* perturb child pivot samples after a bad split driver.py:62,239 */
    int32_t use_partial_insertion;    /* enables the sortedness check (K4) exits       driver.py:63,244 */
    /* ---- GPU fields ---- */
    int32_t base_case_size;           /* K7 threshold, 1024..32768 (default 32768), clamped to each
                                         element type's base-case capacity: 24572 keys for 4-byte
                                         keys without payload, 4096 otherwise */
    int32_t bad_budget;               /* -1: floor(log2 n) (driver.py:263); >= 0 overrides (0 forces the
                                         radix fallback on the first big segment: test knob) */
    int32_t reserved[4];              /* reserved[0] > 0: profiling knob, stop descending at that
                                         depth (output NOT sorted); keep 0.
                                         reserved[1] > 0: smallest n for K4's two-run path (default 2^15;
                                         tests lower it) */
} pdq_config;

/* Device counters (the GPU analogue of Metrics, instrumentation.py:20-61). */
typedef struct pdq_stats {
    int64_t partition_right_calls;  /* segments partitioned with equals-go-right (K2) */
    int64_t partition_left_calls;   /* segments split with equals-go-left (K3) */
    int64_t bad_partitions;         /* driver.py:235-238 analogue */
    int64_t radix_fallbacks;        /* segments that exhausted the budget (K5) */
    int64_t base_cases;             /* K7 invocations */
    int64_t max_depth;              /* deepest segment generation */
    int64_t tiles;                  /* partition tiles processed */
    int64_t bytes_algorithmic;      /* SURVEY.md §8(d) byte model over the init + sorter kernels, summed
                                       over the segments they actually processed */
    int64_t check_result;           /* K4: bit0 a descent seen, bit1 an ascent seen, bit2 a descent in the
                                       first half, bit3 one in the second half (with bit1 the pass stops
                                       early); bits 4-6: the two-run path was taken: bits 4-5 the other run was
                                       1 ascending, 2 descending (reversed in place), 3 sorted by the partition
                                       tree; bit 6 the sorted run of at least half the array is the second one */
    int64_t segments;               /* descriptors allocated */
    int64_t status;                 /* 0 or a negative pdq_status */
    int64_t bytes_check;            /* bytes the K4 check kernel read */
    int64_t cycles_wait;            /* sorter SM cycles (summed over CTAs) waiting for a task */
    int64_t cycles_work;            /*   ... processing tasks (includes the two below) */
    int64_t cycles_base;            /*   ... in K7 base cases */
    int64_t cycles_spawn;           /*   ... sampling pivots and pushing child tiles */
    int64_t sched_retire;           /* scheduler-thread cycles retiring tiles (fence + counter) */
    int64_t sched_claim;            /*   ... claiming ring positions */
    int64_t sched_fetch;            /*   ... polling the ring, copying descriptors, issuing loads */
    int64_t sched_idle;             /*   ... sleeping with nothing to do */
    int64_t bytes_base;             /* algorithmic bytes of the K7 base-case kernel (not in bytes_algorithmic) */
    int64_t sort_ns;                /* device-timer span of the persistent sorter (first CTA start -> last end) */
    int64_t base_ns;                /*   ... of the base-case kernel (0 if it did not run) */
    int64_t run_split;              /* K4 two-run path: A[0, run_split) and A[run_split, n) were merged, one of
                                       them a sorted run of at least half the array (0: path not taken); the
                                       merge's bytes are in bytes_base */
} pdq_stats;

/* Fill `cfg` with the reference defaults (driver.py:55-63) and GPU defaults. */
void pdq_config_default(pdq_config *cfg);

/* 0 if valid, else PDQ_ERR_CONFIG (same rules as driver.py:65-75). */
int pdq_config_validate(const pdq_config *cfg);

/* Bytes of device workspace one sort of n elements needs (scratch ping-pong
 * buffer, segment descriptors, task ring, counters). */
size_t pdq_workspace_bytes(int dtype, int has_payload, int64_t n);

/* Sort n keys (and the optional uint32 payload) in place on the device.
 * keys / payload: device pointers, 16-byte aligned (torch/cudaMalloc
 * allocations are).  workspace: device memory of >= pdq_workspace_bytes().
 * stream: a cudaStream_t (NULL = legacy default stream).  Asynchronous. */
int pdq_sort(void *keys, int dtype, uint32_t *payload, int64_t n, const pdq_config *cfg,
             void *workspace, size_t workspace_bytes, void *stream);

/* pdq_sort() that also records two caller-owned CUDA events (cudaEvent_t, may be NULL) on
 * `stream` immediately before and after the persistent partition kernel (K6/K1-K5), so a
 * profiler-free caller can time the dominant kernel alone (bench.py's roofline figure). */
int pdq_sort_ex(void *keys, int dtype, uint32_t *payload, int64_t n, const pdq_config *cfg,
                void *workspace, size_t workspace_bytes, void *stream, void *event_sort_begin,
                void *event_sort_end);

/* pdq_sort() recording up to four caller-owned CUDA events (events[i] may be NULL, or events itself)
 * on `stream` at the kernel boundaries of one sort: [0] before the first operation (state memsets,
 * K4 check, init), [1] before the persistent partition kernel, [2] after it, [3] after the base-case
 * kernel (the end of the sort).  For per-kernel timing without a profiler (bench.py). */
int pdq_sort_timed(void *keys, int dtype, uint32_t *payload, int64_t n, const pdq_config *cfg,
                   void *workspace, size_t workspace_bytes, void *stream, void *const *events);

/* Synchronise `stream`, copy the device counters of the last sort that used
 * `workspace` into *stats (may be NULL) and return its status. */
int pdq_sort_finish(void *workspace, pdq_stats *stats, void *stream);

/* ---- multi-GPU sample sort: bucketing one rank's shard ----
 * No reference counterpart (the reference is single-process); the host side is
 * paper_2106_05123_b200/distributed.py:sample_sort. */

/* Bytes of device workspace pdq_bucket() needs for n elements and nbuckets (<= 64) buckets. */
size_t pdq_bucket_workspace_bytes(int64_t n, int nbuckets);

/* Split the n elements (keys + optional uint32 payload) of a shard whose first element has global
 * index gidx_base into nbuckets = nsplit + 1 buckets.  Splitters are nsplit ascending
 * (key, payload, global index) triples in device memory (split_payload may be NULL without a
 * payload); element i goes to bucket b = number of splitters below (key_i, payload_i,
 * gidx_base + i), keys compared in the sort's order.  out_keys / out_payload (device, n elements)
 * (must not overlap the inputs) receive the elements grouped by bucket, stable within a bucket;
 * bucket_counts (device, int64[nbuckets]) each bucket's size.  Asynchronous on `stream`. */
int pdq_bucket(const void *keys, int dtype, const uint32_t *payload, int64_t n, int64_t gidx_base,
               const void *split_keys, const uint32_t *split_payload, const int64_t *split_gidx,
               int nsplit, void *out_keys, uint32_t *out_payload, int64_t *bucket_counts,
               void *workspace, size_t workspace_bytes, void *stream);

/* ---- host-buffer drop-in (the reference's sort() on a host sequence, driver.py:267-270) ----
 * The reference mutates the caller's host sequence in place.  A pdq_host_sorter owns device
 * buffers (grown on demand), pinned staging slots and a pool of host threads; pdq_host_sort()
 * copies the caller's keys (+ payload) to the device through the staging slots (T threads copy
 * into pinned memory while the DMA of earlier slots runs), sorts them with pdq_sort_ex() and
 * copies the result back into the same host buffers before it returns.  Synchronous; calls on one
 * sorter are serialised; distinct sorters are independent. */
typedef struct pdq_host_sorter pdq_host_sorter;

/* threads <= 0: $PDQ_HOST_THREADS, else min(8, hardware threads).  NULL on failure. */
pdq_host_sorter *pdq_host_sorter_create(int device, int threads);
void pdq_host_sorter_destroy(pdq_host_sorter *h);

/* keys / payload: HOST pointers (any alignment; payload may be NULL).  stats (may be NULL) receives
 * the device counters.  phase_ms (may be NULL, 4 doubles): host ms staging+H2D, host ms sort wait,
 * host ms D2H+copy-out, device ms of the sort alone.  Returns 0 or a negative pdq_status; on error
 * the caller's buffers hold their input unless the failure was in the copy back. */
int pdq_host_sort(pdq_host_sorter *h, void *keys, int dtype, uint32_t *payload, int64_t n, const pdq_config *cfg,
                  pdq_stats *stats, double *phase_ms);

/* Message for the last error of this sorter (CUDA failures; config/argument errors also set
 * pdq_last_error() of the calling thread). */
const char *pdq_host_sorter_error(const pdq_host_sorter *h);

/* Thread-local message for the last error returned on this thread. */
const char *pdq_last_error(void);

/* Library version string. */
const char *pdq_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PDQ_B200_H */
