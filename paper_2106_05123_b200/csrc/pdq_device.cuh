// pdq_device.cuh — device-side building blocks of the B200 pdqsort path.
//
// Key representation.  Every kernel works on the *ordered* unsigned image of a
// key: signed ints flip the sign bit, floats use the IEEE total-order map.  The
// image is computed in registers when a key is classified and inverted when a
// key is written back, so HBM always holds the caller's original bits.  With a
// payload, elements compare as (ordered key, payload) pairs, lexicographically
// (the reference's tuple order, driver.py:267 on (key, payload) tuples).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <type_traits>

namespace pdq {

constexpr int THREADS = 256;          // threads per CTA in every kernel
constexpr int TILE = 4096;            // keys per partition tile (one "block" of partition.py:184)
constexpr int ITEMS = TILE / THREADS; // keys per thread per tile
#ifndef PDQ_BIG_BASE
#define PDQ_BIG_BASE 24576
#endif
constexpr int BIG_BASE = PDQ_BIG_BASE;  // base-case capacity for 4-byte keys-only sorts (k_base_big)
constexpr int SAMPLES = 256;          // K1 pivot samples per big segment
constexpr int WARPS = THREADS / 32;
constexpr int64_t INLINE_FILL = 16 * TILE;  // fills up to this size run inline in the finalizer

// ---- task ring --------------------------------------------------------------------
// A task is one 64-bit word carrying its own round tag, so publishing it is a
// single store:  [63:48] round tag | [47:45] type | [44:23] segment | [22:0] tile.
enum : uint32_t { T_PART = 1, T_FILL = 2, T_RHIST = 3, T_RSCAT = 4 };  // RHIST/RSCAT: K5 digit passes
__host__ __device__ inline uint64_t task_word(uint64_t pos, int log_q, uint32_t type, uint32_t seg,
                                              uint32_t tile) {
    return ((pos >> log_q) & 0xFFFFull) << 48 | (uint64_t)(type & 7) << 45 |
           (uint64_t)(seg & 0x3FFFFF) << 23 | (uint64_t)(tile & 0x7FFFFF);
}
constexpr uint32_t MAX_SEGS = 0x3FFFFF;
constexpr uint32_t MAX_TILES = 0x7FFFFF;

// ---- segment descriptor ------------------------------------------------------------
// info bits
enum : uint32_t {
    I_SRC_B = 1u << 0,    // segment data lives in the scratch buffer B (else in the caller's A)
    I_LEFT = 1u << 1,     // equals-go-left split (partition_left, partition.py:128-181)
    I_HAS_LB = 1u << 2,   // `lb` is a valid lower bound = the reference's predecessor (driver.py:222)
    I_PERTURB = 1u << 3,  // sample positions perturbed (pattern breaking, driver.py:239-243)
    I_COUNT_EQ = 1u << 4, // the sample's low end repeats the pivot: count keys equal to it
    I_RADIX = 1u << 5,    // K5 fallback: radix exchange on composite bit `rbit` (threshold pivot)
    I_HAS_UB = 1u << 6,   // `ub` is a valid exclusive upper bound
    I_RADIX8 = 1u << 7,   // K5 fallback: digit pass on composite bits [rbit, rbit + pivot_v) (slot `rslot`)
};
constexpr int RDIG = 256;  // digits of a K5 radix pass

struct __align__(128) Seg {
    int64_t begin, end;   // [begin, end) in element indices
    uint64_t pivot;       // pivot key: raw bits for partition segments, ordered image for fills
    uint64_t lb;          // ordered lower bound (predecessor), valid iff I_HAS_LB
    uint32_t pivot_v, lb_v;
    uint32_t ntiles;
    uint32_t info;
    int32_t budget;       // remaining bad-partition budget (driver.py:209-213, 263)
    int32_t depth;
    unsigned long long cnt_left;   // atomics: keys reserved on the left side
    unsigned long long cnt_right;  //          keys reserved on the right side
    unsigned long long cnt_eq;     //          keys bitwise equal to the pivot (RIGHT mode)
    unsigned int tiles_done;
    unsigned int rbit;    // I_RADIX: the composite bit this split decides (0 = most significant)
    uint32_t ub_v;
    uint32_t rslot;       // I_RADIX8: the segment's 256-counter slot (histogram, then scatter cursors)
    uint64_t ub;          // exclusive upper bound (ordered), valid iff I_HAS_UB
    uint64_t pad1;
};
static_assert(sizeof(Seg) == 128, "Seg is one 128-byte line");

// ---- global state (in the workspace) -------------------------------------------------
struct __align__(128) State {
    unsigned long long q_head;     // consumer claim counter
    unsigned long long pad_a[15];
    unsigned long long q_tail;     // producer reservation counter
    unsigned long long pad_b[15];
    unsigned long long keys_final; // keys written to their final place in A
    unsigned int done;             // termination flag
    unsigned int seg_alloc;        // descriptor bump allocator
    int status;
    unsigned int check_bits;       // K4: 1 descent seen, 2 ascent seen
    unsigned int reverse;          // K4 decided the input is non-increasing
    unsigned int rslot_alloc;      // K5 radix-slot bump allocator
    // K4 run detection (exact whenever the check pass was not cut short): the smallest descent index
    // (stored inverted: a zeroed state and atomicMax give the minimum), the largest descent index + 1
    // and the largest ascent index + 1
    unsigned long long run_d1_inv, run_dl, run_la;
    unsigned long long run_split;  // > 0: A[0, run_split) and A[run_split, n) are merged after the sort
    unsigned int run_kind;         // the other run was 1 ascending, 2 descending (reversed), 3 sorted by the tree;
                                   // + 4 when the sorted run of at least half the array is the second one
    unsigned int pad_e;
    // merge epilogue of the leaf kernel (RunsMerge): progress counters instead of grid barriers, so a CTA
    // only ever waits for work that running CTAs have already claimed
    unsigned long long leaves_done;  // leaves finished (summed per CTA at the end of its leaf loop)
    unsigned long long merge_next;   // next unclaimed merge tile
    unsigned long long merge_done;   // merge tiles written to B
    unsigned long long run_fa_inv;   // K4: the smallest ascent index, stored inverted like run_d1_inv
    unsigned long long rev_begin, rev_end;  // the range the sorter's prologue reverses (K4)
    unsigned long long pad_d[1];
    // counters (pdq_stats order)
    unsigned long long leaf_count;  // queued base-case segments (K7 kernel input)
    unsigned long long leaf_next;   // K7 kernel claim counter
    unsigned long long c_part_right, c_part_left, c_bad, c_fallback, c_base, c_max_depth, c_tiles,
        c_bytes, c_bytes_check, c_bytes_base;
    unsigned long long c_cyc_wait, c_cyc_work, c_cyc_base, c_cyc_spawn;  // SM cycles by phase (thread 0)
    unsigned long long c_sch_retire, c_sch_claim, c_sch_fetch, c_sch_idle;  // scheduler-thread cycles
    // device-timer spans (%globaltimer ns) of the two big kernels, first CTA start (stored inverted, so
    // a zeroed state and atomicMax give the minimum) to last CTA end: per-kernel times without events
    // between the kernels (which would end their programmatic overlap)
    unsigned long long t_sort_b_inv, t_sort_e, t_base_b_inv, t_base_e;
};

struct Params {
    void *a_keys;          // caller's keys (final buffer)
    void *b_keys;          // scratch
    uint32_t *a_vals;      // caller's payload or nullptr
    uint32_t *b_vals;
    int64_t n;
    State *st;
    Seg *segs;
    uint64_t *ring;
    uint32_t seg_cap;
    int log_q;
    int bad_shift;
    int use_left;
    int use_break;
    int use_check;
    int base_size;
    int budget0;
    int debug_depth;   // > 0: segments at this depth are dropped unsorted (profiling only)
    int64_t runs_min;  // K4 merges two runs only for n >= runs_min
    uint64_t *leaves;  // queued leaves: begin << 16 | (size - 1) << 1 | in-B
    unsigned long long leaf_cap;
    uint32_t chunk;    // tiles per ring task
    unsigned long long *rslots;  // K5: rslot_cap slots of RDIG counters
    uint32_t rslot_cap;
};

// ---- key traits ----------------------------------------------------------------------
template <class U, bool FLOAT>
struct Ord {
    static constexpr U SIGN = (U)1 << (sizeof(U) * 8 - 1);
    __device__ __forceinline__ static U to(U x) {
        if (FLOAT) return (x & SIGN) ? (U)~x : (U)(x ^ SIGN);
        return x ^ SIGN;
    }
    __device__ __forceinline__ static U from(U x) {
        if (FLOAT) return (x & SIGN) ? (U)(x ^ SIGN) : (U)~x;
        return x ^ SIGN;
    }
};

template <bool KV>
__device__ __forceinline__ bool pless(uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
    if (KV) return ka < kb || (ka == kb && va < vb);
    return ka < kb;
}

// ---- PTX helpers -----------------------------------------------------------------------
__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned *p) {
    return *(const volatile unsigned *)p;
}
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}
// TMA bulk copy global -> shared (cp.async.bulk, SASS UBLKCP); 16-byte aligned, size % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void *sdst, const void *gsrc, unsigned bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
// TMA bulk copy shared -> global (bulk-group completion); 16-byte aligned, size % 16 == 0.
__device__ __forceinline__ void bulk_s2g(void *gdst, const void *ssrc, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_addr(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the shared-memory sources of every committed bulk store have been read (the buffer may be reused)
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// every committed bulk store has completed its global writes
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr uint64_t WATCHDOG_NS = 10ull * 1000 * 1000 * 1000;

// Debug builds (-DPDQ_DEBUG, tools/build_debug.sh): device-side bounds / invariant checks that trap
// with a message (compute-sanitizer is not available on the GPU pool).  Compiled out otherwise.
#ifdef PDQ_DEBUG
#define PDQ_CHECK(cond, what)                                                                        \
    do {                                                                                             \
        if (!(cond)) {                                                                               \
            printf("PDQ_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,    \
                   (int)blockIdx.x, (int)threadIdx.x);                                               \
            __trap();                                                                                \
        }                                                                                            \
    } while (0)
#else
#define PDQ_CHECK(cond, what) \
    do {                      \
    } while (0)
#endif

template <class U>
__device__ __forceinline__ U ldcg(const U *p) {
    return __ldcg(p);
}

}  // namespace pdq
