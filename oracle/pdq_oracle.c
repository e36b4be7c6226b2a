/* ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's sort path (pattern-defeating
 * quicksort, /root/reference/pkg/src/pdqsort/{driver,partition,small_sorts}.py).
 * It is the CHECKER for the CUDA product path, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it.  The product (paper_2106_05123_b200) never
 * links, imports or calls anything under oracle/.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against
 * golden vectors produced by running the Python reference itself
 * (tests/golden/make_golden_vectors.py): exact output permutations of every
 * primitive and of full sorts, plus the reference's instrumentation counters
 * (comparisons, moves, exchanges, partition/fallback counts, max depth),
 * which only match if the same algorithm runs step for step.
 *
 * Element types: int32, int64, float32, float64 keys, and "kv" = (int64 key,
 * uint32 payload) pairs ordered lexicographically, which is how the reference
 * orders the Python tuples it is given for the KV config (driver.py:267 on a
 * list of (key, payload) tuples).
 */

#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t insertion_threshold;      /* driver.py:55 */
    int64_t ninther_threshold;        /* driver.py:56 */
    int64_t partial_insertion_budget; /* driver.py:57 */
    int64_t block_size;               /* driver.py:58 */
    int64_t bad_partition_shift;      /* driver.py:59 */
    int64_t use_block_partition;      /* driver.py:60 */
    int64_t use_partition_left;       /* driver.py:61 */
    int64_t use_break_patterns;       /* driver.py:62 */
    int64_t use_partial_insertion;    /* driver.py:63 */
} oracle_config;

/* instrumentation.py:20-61, METRIC_FIELDS order (:20-31) */
typedef struct {
    int64_t comparisons;
    int64_t element_moves;
    int64_t exchanges;
    int64_t partition_right_calls;
    int64_t partition_left_calls;
    int64_t bad_partitions;
    int64_t heapsort_fallbacks;
    int64_t partial_insertion_attempts;
    int64_t partial_insertion_aborts;
    int64_t max_depth;
} oracle_metrics;

/* partition.py:32-41 */
typedef struct {
    int64_t pivot_index;
    int64_t no_swaps;
} oracle_partition_result;

#define ORACLE_MIN_BREAK_SIZE 8 /* driver.py:44 */

static int64_t oracle_bit_length(int64_t n) {
    int64_t b = 0;
    while (n) {
        b++;
        n >>= 1;
    }
    return b;
}

/* driver.py:116-124 */
int oracle_is_bad_partition(int64_t left_size, int64_t right_size, int64_t total, const oracle_config *cfg) {
    int64_t threshold = total >> cfg->bad_partition_shift;
    return left_size < threshold || right_size < threshold;
}

/* driver.py:65-75: returns 0 if valid, else the index of the violated rule (1..5). */
int oracle_config_check(const oracle_config *cfg) {
    int64_t mx = cfg->insertion_threshold > 8 ? cfg->insertion_threshold : 8;
    if (cfg->insertion_threshold < 3) return 1;
    if (cfg->ninther_threshold < mx) return 2;
    if (cfg->partial_insertion_budget < 0) return 3;
    if (cfg->block_size < 1) return 4;
    if (cfg->bad_partition_shift < 1) return 5;
    return 0;
}

typedef struct {
    int64_t k;
    uint32_t v;
} oracle_kv;

#define T int32_t
#define SFX i32
#define LESS(a, b) ((a) < (b))
#include "pdq_oracle_impl.h"
#undef T
#undef SFX
#undef LESS

#define T int64_t
#define SFX i64
#define LESS(a, b) ((a) < (b))
#include "pdq_oracle_impl.h"
#undef T
#undef SFX
#undef LESS

/* The reference promotes float32 to Python float (double); the promotion is
 * exact, so float32 '<' orders identically for NaN-free input. */
#define T float
#define SFX f32
#define LESS(a, b) ((double)(a) < (double)(b))
#include "pdq_oracle_impl.h"
#undef T
#undef SFX
#undef LESS

#define T double
#define SFX f64
#define LESS(a, b) ((a) < (b))
#include "pdq_oracle_impl.h"
#undef T
#undef SFX
#undef LESS

/* Python tuple ordering: (k1, v1) < (k2, v2) lexicographically. */
#define T oracle_kv
#define SFX kv
#define LESS(a, b) ((a).k < (b).k || ((a).k == (b).k && (a).v < (b).v))
#include "pdq_oracle_impl.h"
#undef T
#undef SFX
#undef LESS

/* ---- flat entry points used by tests / bench (ctypes) ---------------------------- */

/* dtype codes match include/pdq_b200.h: 0 int32, 1 int64, 2 float32, 3 float64. */
int oracle_sort(void *keys, int dtype, int64_t n, const oracle_config *cfg, int use_block,
                oracle_metrics *m) {
    switch (dtype) {
        case 0: oracle_sort_range_i32((int32_t *)keys, 0, n, cfg, use_block, m); return 0;
        case 1: oracle_sort_range_i64((int64_t *)keys, 0, n, cfg, use_block, m); return 0;
        case 2: oracle_sort_range_f32((float *)keys, 0, n, cfg, use_block, m); return 0;
        case 3: oracle_sort_range_f64((double *)keys, 0, n, cfg, use_block, m); return 0;
        default: return -1;
    }
}

/* KV: int64 keys + uint32 payload, sorted as (key, payload) tuples. */
int oracle_sort_kv(int64_t *keys, uint32_t *vals, int64_t n, const oracle_config *cfg, int use_block,
                   oracle_metrics *m) {
    oracle_kv *tmp = (oracle_kv *)malloc(sizeof(oracle_kv) * (size_t)(n > 0 ? n : 1));
    if (!tmp) return -2;
    for (int64_t i = 0; i < n; i++) {
        tmp[i].k = keys[i];
        tmp[i].v = vals[i];
    }
    oracle_sort_range_kv(tmp, 0, n, cfg, use_block, m);
    for (int64_t i = 0; i < n; i++) {
        keys[i] = tmp[i].k;
        vals[i] = tmp[i].v;
    }
    free(tmp);
    return 0;
}

/* Primitive-level entry points over int64 data (the golden vectors use ints). */
void oracle_prim_insertion_sort(int64_t *d, int64_t b, int64_t e, oracle_metrics *m) {
    oracle_insertion_sort_i64(d, b, e, m);
}
void oracle_prim_unguarded_insertion_sort(int64_t *d, int64_t b, int64_t e, oracle_metrics *m) {
    oracle_unguarded_insertion_sort_i64(d, b, e, m);
}
int oracle_prim_partial_insertion_sort(int64_t *d, int64_t b, int64_t e, int64_t budget, oracle_metrics *m) {
    return oracle_partial_insertion_sort_i64(d, b, e, budget, m);
}
void oracle_prim_heapsort(int64_t *d, int64_t b, int64_t e, oracle_metrics *m) { oracle_heapsort_i64(d, b, e, m); }
void oracle_prim_sort3(int64_t *d, int64_t a, int64_t b, int64_t c, oracle_metrics *m) {
    oracle_sort3_i64(d, a, b, c, m);
}
void oracle_prim_partition_right(int64_t *d, int64_t b, int64_t e, oracle_metrics *m, oracle_partition_result *r) {
    *r = oracle_partition_right_i64(d, b, e, m);
}
void oracle_prim_partition_left(int64_t *d, int64_t b, int64_t e, oracle_metrics *m, oracle_partition_result *r) {
    *r = oracle_partition_left_i64(d, b, e, m);
}
void oracle_prim_block_partition_right(int64_t *d, int64_t b, int64_t e, int64_t block, oracle_metrics *m,
                                       oracle_partition_result *r) {
    *r = oracle_block_partition_right_i64(d, b, e, block, m);
}
void oracle_prim_choose_pivot(int64_t *d, int64_t b, int64_t e, const oracle_config *cfg, oracle_metrics *m) {
    oracle_choose_pivot_i64(d, b, e, cfg, m);
}
void oracle_prim_break_patterns(int64_t *d, int64_t b, int64_t e, const oracle_config *cfg, oracle_metrics *m) {
    oracle_break_patterns_i64(d, b, e, cfg, m);
}
