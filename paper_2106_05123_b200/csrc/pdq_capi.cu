// pdq_capi.cu — the C ABI (include/pdq_b200.h) over the sm_100a kernels.
//
// One pdq_sort() call = memset(state) + memset(ring) + K4 check + init + persistent sorter,
// all stream-ordered; no host synchronisation inside.  Replaces driver.py:267-292.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include <nvtx3/nvToolsExt.h>  // header-only; ranges are no-ops unless a profiler is attached

#include "../../include/pdq_b200.h"
#include "pdq_bucket.cuh"
#include "pdq_kernels.cuh"

using namespace pdq;

static thread_local char g_err[512];

static int set_err(int code, const char *fmt, const char *detail = "") {
    snprintf(g_err, sizeof(g_err), fmt, detail);
    return code;
}

extern "C" const char *pdq_last_error(void) { return g_err; }
extern "C" const char *pdq_version(void) { return "pdq_b200 0.1.0 (sm_100a)"; }

extern "C" void pdq_config_default(pdq_config *c) {
    memset(c, 0, sizeof(*c));
    c->insertion_threshold = 24;
    c->ninther_threshold = 128;
    c->partial_insertion_budget = 8;
    c->block_size = 64;
    c->bad_partition_shift = 3;
    c->use_block_partition = 1;
    c->use_partition_left = 1;
    c->use_break_patterns = 1;
    c->use_partial_insertion = 1;
    c->base_case_size = 32768;  // the largest leaf each element type's base-case kernel takes
    c->bad_budget = -1;
}

extern "C" int pdq_config_validate(const pdq_config *c) {
    // driver.py:65-75, same rules, same order
    if (c->insertion_threshold < 3)
        return set_err(PDQ_ERR_CONFIG, "insertion_threshold must be >= 3 (pivot selection needs three candidates)%s");
    int64_t mx = c->insertion_threshold > 8 ? c->insertion_threshold : 8;
    if (c->ninther_threshold < mx)
        return set_err(PDQ_ERR_CONFIG, "ninther_threshold must be >= max(8, insertion_threshold)%s");
    if (c->partial_insertion_budget < 0) return set_err(PDQ_ERR_CONFIG, "partial_insertion_budget must be >= 0%s");
    if (c->block_size < 1) return set_err(PDQ_ERR_CONFIG, "block_size must be >= 1%s");
    if (c->bad_partition_shift < 1) return set_err(PDQ_ERR_CONFIG, "bad_partition_shift must be >= 1%s");
    if (c->bad_partition_shift > 62) return set_err(PDQ_ERR_CONFIG, "bad_partition_shift must be <= 62%s");
    if (c->base_case_size < 1024 || c->base_case_size > 32768)  // clamped per element type at launch
        return set_err(PDQ_ERR_CONFIG, "base_case_size must be in [1024, 32768]%s");
    return PDQ_OK;
}

namespace {

constexpr int MIN_BASE = 1024;
#ifndef PDQ_CHUNK_MAX
#define PDQ_CHUNK_MAX 32  // tiles per ring task at most
#endif
#ifndef PDQ_RUNS_MIN
#define PDQ_RUNS_MIN (1 << 18)  // K4 takes the two-run path (sorted prefix of >= n/2 + merge) from this size
#endif
#ifndef PDQ_CHUNK_DIV
#define PDQ_CHUNK_DIV 2  // the root level gets about this many tasks per CTA
#endif

struct Layout {
    size_t b_keys, b_vals, state, segs, ring, leaves, rslots, total;
    uint32_t rslot_cap;
    uint64_t leaf_cap;
    uint32_t seg_cap;
    int log_q;
};

size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

int dtype_size(int dtype) {
    switch (dtype) {
        case PDQ_I32:
        case PDQ_F32: return 4;
        case PDQ_I64:
        case PDQ_F64: return 8;
        default: return 0;
    }
}

Layout layout(int dtype, int has_payload, int64_t n) {
    // State sits at offset 0 so pdq_sort_finish() can find it from the workspace pointer alone.
    Layout L;
    const size_t w = (size_t)dtype_size(dtype);
    size_t off = 0;
    L.state = off;
    off += a256(sizeof(State));
    L.b_keys = off;
    off += a256((size_t)n * w + 16);
    L.b_vals = off;
    if (has_payload) off += a256((size_t)n * 4 + 16);
    // descriptors ever allocated (with parent-slot reuse) <= terminal big segments + big fills
    uint64_t segs = (uint64_t)n / MIN_BASE + (uint64_t)n / INLINE_FILL + 256;
    L.seg_cap = (uint32_t)segs;
    L.segs = off;
    off += a256(segs * sizeof(Seg));
    // outstanding tasks <= tiles of live (disjoint) segments + claimed-but-unprocessed
    uint64_t q = (uint64_t)n / (TILE / 2) + 2 * ((uint64_t)n / MIN_BASE) + 2 * segs + 16384;  // tiles >= TILE/2
    int lq = 14;
    while ((1ull << lq) < q) ++lq;
    L.log_q = lq;
    L.ring = off;
    off += a256((size_t)(1ull << lq) * 8);
    // leaves are disjoint segments of more than 64 keys (smaller ones are sorted in place)
    L.leaf_cap = (uint64_t)n / 64 + 16;
    L.leaves = off;
    off += a256((size_t)L.leaf_cap * 8);
    // K5 digit passes: one slot of RDIG 64-bit counters per radix segment (bump-allocated; when they
    // run out a segment falls back to one-bit radix exchange, which needs none)
    L.rslot_cap = (uint32_t)((uint64_t)n / 32768 + 512);
    L.rslots = off;
    off += a256((size_t)L.rslot_cap * RDIG * 8);
    L.total = off;
    return L;
}

struct LaunchInfo {
    int sms = 0;
    int occ = 0;
    int occ_base = 0;
};

// 4-byte keys without payload: leaves of up to BIG_BASE - 4 (24572) keys sorted by k_base_big; 8-byte
// keys and key-value sorts: leaves of up to 8188 elements sorted by k_base_wide
template <class U, bool KV>
constexpr bool big_leaves() {
    return sizeof(U) == 4 && !KV;
}

template <class U, bool FLOAT, bool KV>
int smem_bytes() {
    return Bufs<U, KV>::bytes();
}

constexpr int MAX_DEVS = 64;

template <class U, bool FLOAT, bool KV>
cudaError_t prepare(LaunchInfo &li) {
    // per device and element type: kernel attributes set once, occupancy and SM count cached
    static std::mutex mu;
    static bool ready[MAX_DEVS] = {};
    static LaunchInfo cache[MAX_DEVS];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= MAX_DEVS) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> g(mu);
    LaunchInfo &cached = cache[dev];
    if (!ready[dev]) {
        const int sm = smem_bytes<U, FLOAT, KV>();
        if ((e = cudaFuncSetAttribute(k_sort<U, FLOAT, KV>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)) !=
            cudaSuccess)
            return e;
        if ((e = cudaFuncSetAttribute(k_init<U, FLOAT, KV>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)) !=
            cudaSuccess)
            return e;
        if constexpr (big_leaves<U, KV>()) {
            if ((e = cudaFuncSetAttribute(k_base_big<FLOAT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          BigLeaf<FLOAT>::bytes())) != cudaSuccess)
                return e;
            if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cached.occ_base, k_base_big<FLOAT>, BigLeaf<FLOAT>::BT,
                                                                   BigLeaf<FLOAT>::bytes())) != cudaSuccess)
                return e;
        } else {
            if ((e = cudaFuncSetAttribute(k_base_wide<U, FLOAT, KV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          WideLeaf<U, FLOAT, KV>::bytes())) != cudaSuccess)
                return e;
            cached.occ_base = 1;
        }
        if (cached.occ_base < 1) cached.occ_base = 1;
        if ((e = cudaDeviceGetAttribute(&cached.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cached.occ, k_sort<U, FLOAT, KV>, THREADS, sm)) !=
            cudaSuccess)
            return e;
        if (cached.occ < 1) cached.occ = 1;
        ready[dev] = true;
    }
    li = cached;
    return cudaSuccess;
}

// Programmatic dependent launch: the kernel may be scheduled while the previous kernel of the stream is
// still running (its CTAs wait in griddepcontrol.wait until that kernel has completed and its memory is
// visible), so the launch latency of each of the sort's kernels overlaps its predecessor's tail.
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                       bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <class U, bool FLOAT, bool KV>
int launch(Params &P, cudaStream_t s, const Layout &L, cudaEvent_t ev0, cudaEvent_t ev1, cudaEvent_t ev_end) {
    LaunchInfo li;
    // (k_base_big reads a leaf as 16-byte vectors from its aligned base: up to 3 slots of lead-in)
    const int base_max = big_leaves<U, KV>() ? BIG_BASE - 4 : WideLeaf<U, FLOAT, KV>::CAP - 4;
    if (P.base_size > base_max) P.base_size = base_max;
    cudaError_t e = prepare<U, FLOAT, KV>(li);
    if (e != cudaSuccess) return set_err(PDQ_ERR_CUDA, "setup: %s", cudaGetErrorString(e));
    const int sm = smem_bytes<U, FLOAT, KV>();
    {  // tiles per task: the largest power of two <= 32 giving the root ~2 tasks per CTA
        constexpr int TL = Sorter<U, FLOAT, KV>::TL;
        const int64_t per = ((P.n + TL - 1) / TL) / (PDQ_CHUNK_DIV * (int64_t)li.sms * li.occ);
        uint32_t c = 1;
        while (c < PDQ_CHUNK_MAX && (int64_t)(c * 2) <= per) c *= 2;
        P.chunk = c;
    }
    if (P.use_check && P.n > 1) {
        const int64_t ch = (int64_t)THREADS * ITEMS;
        int64_t blocks = (P.n + ch - 1) / ch;
        const int64_t cap = (int64_t)li.sms * 8;
        if (blocks > cap) blocks = cap;
        k_check<U, FLOAT, KV><<<(unsigned)blocks, THREADS, 0, s>>>(P);
    }
    // (an event between two kernels ends the programmatic overlap there: timed runs measure each kernel)
    e = launch_pdl(k_init<U, FLOAT, KV>, 1, THREADS, sm, s, P.use_check && P.n > 1, P);
    if (e == cudaSuccess && ev0) cudaEventRecord(ev0, s);
    if (e == cudaSuccess) e = launch_pdl(k_sort<U, FLOAT, KV>, (unsigned)(li.sms * li.occ), THREADS, sm, s, !ev0, P);
    if (e == cudaSuccess && ev1) cudaEventRecord(ev1, s);
    if (e == cudaSuccess) {
        if constexpr (big_leaves<U, KV>())
            e = launch_pdl(k_base_big<FLOAT>, (unsigned)(li.sms * li.occ_base), BigLeaf<FLOAT>::BT,
                           BigLeaf<FLOAT>::bytes(), s, !ev1, P);
        else
            e = launch_pdl(k_base_wide<U, FLOAT, KV>, (unsigned)li.sms, 1024, WideLeaf<U, FLOAT, KV>::bytes(), s, !ev1,
                           P);
    }
    if (e == cudaSuccess && ev_end) cudaEventRecord(ev_end, s);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(PDQ_ERR_CUDA, "launch: %s", cudaGetErrorString(e));
    return PDQ_OK;
}

}  // namespace

extern "C" size_t pdq_workspace_bytes(int dtype, int has_payload, int64_t n) {
    if (dtype_size(dtype) == 0 || n < 0) return 0;
    return layout(dtype, has_payload, n).total;
}

extern "C" int pdq_sort(void *keys, int dtype, uint32_t *payload, int64_t n, const pdq_config *cfg_in,
                        void *workspace, size_t ws_bytes, void *stream) {
    return pdq_sort_ex(keys, dtype, payload, n, cfg_in, workspace, ws_bytes, stream, nullptr, nullptr);
}

extern "C" int pdq_sort_ex(void *keys, int dtype, uint32_t *payload, int64_t n, const pdq_config *cfg_in,
                           void *workspace, size_t ws_bytes, void *stream, void *ev_begin, void *ev_end) {
    void *ev[4] = {nullptr, ev_begin, ev_end, nullptr};
    return pdq_sort_timed(keys, dtype, payload, n, cfg_in, workspace, ws_bytes, stream, ev);
}

extern "C" int pdq_sort_timed(void *keys, int dtype, uint32_t *payload, int64_t n, const pdq_config *cfg_in,
                              void *workspace, size_t ws_bytes, void *stream, void *const *events) {
    cudaEvent_t evs = events ? (cudaEvent_t)events[0] : nullptr, ev0 = events ? (cudaEvent_t)events[1] : nullptr,
                ev1 = events ? (cudaEvent_t)events[2] : nullptr, eve = events ? (cudaEvent_t)events[3] : nullptr;
    pdq_config cfg;
    if (cfg_in)
        cfg = *cfg_in;
    else
        pdq_config_default(&cfg);
    int rc = pdq_config_validate(&cfg);
    if (rc) return rc;
    if (dtype_size(dtype) == 0) return set_err(PDQ_ERR_DTYPE, "unsupported dtype code%s");
    if (n < 0) return set_err(PDQ_ERR_ARG, "n must be >= 0%s");
    if (n > ((int64_t)MAX_TILES - 2) * (TILE / 2)) return set_err(PDQ_ERR_ARG, "n too large for the task encoding%s");
    if (n > 0 && !keys) return set_err(PDQ_ERR_ARG, "keys is NULL%s");
    if (((uintptr_t)keys & 15) || ((uintptr_t)payload & 15))
        return set_err(PDQ_ERR_ALIGN, "keys and payload must be 16-byte aligned%s");
    const Layout L = layout(dtype, payload != nullptr, n);
    if (!workspace || ws_bytes < L.total) return set_err(PDQ_ERR_WORKSPACE, "workspace too small%s");
    if (((uintptr_t)workspace & 255)) return set_err(PDQ_ERR_ALIGN, "workspace must be 256-byte aligned%s");
    cudaStream_t s = (cudaStream_t)stream;
    unsigned char *ws = (unsigned char *)workspace;
    struct Range {  // NVTX range over the enqueue (SURVEY §5 tracing)
        Range() { nvtxRangePushA("pdq_sort"); }
        ~Range() { nvtxRangePop(); }
    } range;
    if (evs) cudaEventRecord(evs, s);
    cudaError_t e = cudaMemsetAsync(ws + L.state, 0, sizeof(State), s);
    // the ring is emptied by k_check when it runs (one fewer stream operation on the latency path)
    const bool check_kernel = cfg.use_partial_insertion && n > 1;
    if (e == cudaSuccess && !check_kernel) e = cudaMemsetAsync(ws + L.ring, 0xFF, (size_t)(1ull << L.log_q) * 8, s);
    if (e != cudaSuccess) return set_err(PDQ_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
    if (n == 0) {  // finish() reads a zeroed state: status 0
        if (ev0) cudaEventRecord(ev0, s);
        if (ev1) cudaEventRecord(ev1, s);
        if (eve) cudaEventRecord(eve, s);
        return PDQ_OK;
    }

    Params P;
    P.a_keys = keys;
    P.b_keys = ws + L.b_keys;
    P.a_vals = payload;
    P.b_vals = payload ? (uint32_t *)(ws + L.b_vals) : nullptr;
    P.n = n;
    P.st = (State *)(ws + L.state);
    P.segs = (Seg *)(ws + L.segs);
    P.ring = (uint64_t *)(ws + L.ring);
    P.seg_cap = L.seg_cap;
    P.log_q = L.log_q;
    P.bad_shift = (int)cfg.bad_partition_shift;
    P.use_left = cfg.use_partition_left ? 1 : 0;
    P.use_break = cfg.use_break_patterns ? 1 : 0;
    P.use_check = cfg.use_partial_insertion ? 1 : 0;
    P.base_size = cfg.base_case_size;
    P.budget0 = cfg.bad_budget;
    P.debug_depth = cfg.reserved[0];
    P.runs_min = cfg.reserved[1] > 0 ? (int64_t)cfg.reserved[1] : (int64_t)PDQ_RUNS_MIN;
    P.leaves = (uint64_t *)(ws + L.leaves);
    P.leaf_cap = L.leaf_cap;
    P.rslots = (unsigned long long *)(ws + L.rslots);
    P.rslot_cap = L.rslot_cap;


    const bool kv = payload != nullptr;
#ifdef PDQ_ONLY_I32  // profiling builds (tools/): int32 keys-only instantiation, fast to compile
    if (dtype == PDQ_I32 && !kv) return launch<uint32_t, false, false>(P, s, L, ev0, ev1, eve);
    return set_err(PDQ_ERR_DTYPE, "this profiling build sorts int32 keys only%s");
#else
    switch (dtype) {
        case PDQ_I32: return kv ? launch<uint32_t, false, true>(P, s, L, ev0, ev1, eve) : launch<uint32_t, false, false>(P, s, L, ev0, ev1, eve);
        case PDQ_F32: return kv ? launch<uint32_t, true, true>(P, s, L, ev0, ev1, eve) : launch<uint32_t, true, false>(P, s, L, ev0, ev1, eve);
        case PDQ_I64: return kv ? launch<uint64_t, false, true>(P, s, L, ev0, ev1, eve) : launch<uint64_t, false, false>(P, s, L, ev0, ev1, eve);
        case PDQ_F64: return kv ? launch<uint64_t, true, true>(P, s, L, ev0, ev1, eve) : launch<uint64_t, true, false>(P, s, L, ev0, ev1, eve);
    }
#endif
    return set_err(PDQ_ERR_DTYPE, "unsupported dtype code%s");
}

extern "C" int pdq_sort_finish(void *workspace, pdq_stats *out, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!workspace) return set_err(PDQ_ERR_ARG, "workspace is NULL%s");
    State st;
    cudaError_t e = cudaMemcpyAsync(&st, workspace, sizeof(State), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return set_err(PDQ_ERR_CUDA, "finish: %s", cudaGetErrorString(e));
    if (out) {
        memset(out, 0, sizeof(*out));
        out->partition_right_calls = (int64_t)st.c_part_right;
        out->partition_left_calls = (int64_t)st.c_part_left;
        out->bad_partitions = (int64_t)st.c_bad;
        out->radix_fallbacks = (int64_t)st.c_fallback;
        out->base_cases = (int64_t)st.c_base;
        out->max_depth = (int64_t)st.c_max_depth;
        out->tiles = (int64_t)st.c_tiles;
        out->bytes_algorithmic = (int64_t)st.c_bytes;
        out->check_result = (int64_t)(st.check_bits | st.run_kind << 4);
        out->run_split = (int64_t)st.run_split;
        out->segments = (int64_t)st.seg_alloc;
        out->status = (int64_t)st.status;
        out->bytes_check = (int64_t)st.c_bytes_check;
        out->bytes_base = (int64_t)st.c_bytes_base;
        out->cycles_wait = (int64_t)st.c_cyc_wait;
        out->cycles_work = (int64_t)st.c_cyc_work;
        out->cycles_base = (int64_t)st.c_cyc_base;
        out->cycles_spawn = (int64_t)st.c_cyc_spawn;
        out->sched_retire = (int64_t)st.c_sch_retire;
        out->sched_claim = (int64_t)st.c_sch_claim;
        out->sched_fetch = (int64_t)st.c_sch_fetch;
        out->sched_idle = (int64_t)st.c_sch_idle;
        out->sort_ns = st.t_sort_e && st.t_sort_b_inv ? (int64_t)(st.t_sort_e - ~st.t_sort_b_inv) : 0;
        out->base_ns = st.t_base_e && st.t_base_b_inv ? (int64_t)(st.t_base_e - ~st.t_base_b_inv) : 0;
    }
    if (st.status == -8) return set_err(PDQ_ERR_INTERNAL, "device watchdog: the task queue stalled for 10 s%s");
    if (st.status) return set_err(PDQ_ERR_INTERNAL, "device-side failure (descriptor capacity)%s");
    return PDQ_OK;
}

// ---- sample-sort bucketing ----------------------------------------

extern "C" size_t pdq_bucket_workspace_bytes(int64_t n, int nbuckets) {
    if (n < 0 || nbuckets < 1 || nbuckets > BK_MAX) return 0;
    return a256((size_t)nbuckets * (size_t)BK_MAX_CTAS * sizeof(int64_t));  // any element type's grid
}

__global__ void k_set_i64(int64_t *p, int64_t v) { *p = v; }

namespace {
template <class U, bool FLOAT, bool KV, int LT>
int launch_bucket(const void *keys, const uint32_t *vals, int64_t n, int64_t gidx_base, const void *sk,
                  const uint32_t *sv, const int64_t *sg, int ns, void *ok, uint32_t *ov, int64_t *bucket_counts,
                  int64_t *cnt, cudaStream_t s) {
    const BucketGeom g = bucket_geom(n, BkShape<U, KV>::TILE, BkShape<U, KV>::CTAS);
    const int nb = ns + 1;
    const size_t hist = (size_t)nb * BK_THREADS * sizeof(uint32_t);
    const size_t sc = sizeof(ScatterSmem<U, KV>) + hist;
    cudaError_t ea = cudaFuncSetAttribute(k_bucket_count<U, FLOAT, KV, LT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(BK_MAX * BK_THREADS * sizeof(uint32_t)));
    if (ea == cudaSuccess)
        ea = cudaFuncSetAttribute(k_bucket_scatter<U, FLOAT, KV, LT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(ScatterSmem<U, KV>) + BK_MAX * BK_THREADS * sizeof(uint32_t)));
    if (ea != cudaSuccess) return set_err(PDQ_ERR_CUDA, "bucket setup: %s", cudaGetErrorString(ea));
    k_bucket_count<U, FLOAT, KV, LT><<<g.ctas, BK_THREADS, hist, s>>>((const U *)keys, vals, n, gidx_base,
                                                                         (const U *)sk, sv, sg, ns, cnt, g);
    k_bucket_scan<<<1, BK_SCAN_THREADS, 0, s>>>(cnt, (int64_t)nb * g.ctas, nb, g.ctas, bucket_counts);
    k_bucket_scatter<U, FLOAT, KV, LT><<<g.ctas, BK_THREADS, sc, s>>>(
        (const U *)keys, vals, n, gidx_base, (const U *)sk, sv, sg, ns, cnt, (U *)ok, ov, g);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(PDQ_ERR_CUDA, "bucket launch: %s", cudaGetErrorString(e));
    return PDQ_OK;
}

template <class U, bool FLOAT, bool KV>
int launch_bucket_nb(const void *keys, const uint32_t *vals, int64_t n, int64_t gidx_base, const void *sk,
                     const uint32_t *sv, const int64_t *sg, int ns, void *ok, uint32_t *ov, int64_t *bucket_counts,
                     int64_t *cnt, cudaStream_t s) {
    // up to 8 buckets (one NVLink node): per-thread counts packed in registers, the splitter search
    // unrolled to its depth
#define PDQ_LB(LT) launch_bucket<U, FLOAT, KV, LT>(keys, vals, n, gidx_base, sk, sv, sg, ns, ok, ov, bucket_counts, cnt, s)
    switch (bucket_log2(ns + 1)) {
        case 0: return PDQ_LB(0);
        case 1: return PDQ_LB(1);
        case 2: return PDQ_LB(2);
        case 3: return PDQ_LB(3);
        default: return PDQ_LB(-1);
    }
#undef PDQ_LB
}
}  // namespace

extern "C" int pdq_bucket(const void *keys, int dtype, const uint32_t *payload, int64_t n, int64_t gidx_base,
                          const void *split_keys, const uint32_t *split_payload, const int64_t *split_gidx,
                          int nsplit, void *out_keys, uint32_t *out_payload, int64_t *bucket_counts,
                          void *workspace, size_t ws_bytes, void *stream) {
    if (dtype_size(dtype) == 0) return set_err(PDQ_ERR_DTYPE, "unsupported dtype code%s");
    if (n < 0) return set_err(PDQ_ERR_ARG, "n must be >= 0%s");
    if (nsplit < 0 || nsplit + 1 > BK_MAX) return set_err(PDQ_ERR_ARG, "nsplit must be in [0, 63]%s");
    if (!bucket_counts) return set_err(PDQ_ERR_ARG, "bucket_counts is NULL%s");
    if (n > 0 && (!keys || !out_keys)) return set_err(PDQ_ERR_ARG, "keys / out_keys is NULL%s");
    if ((payload == nullptr) != (out_payload == nullptr))
        return set_err(PDQ_ERR_ARG, "payload and out_payload must both be given or both be NULL%s");
    if (nsplit > 0 && (!split_keys || !split_gidx || (payload && !split_payload)))
        return set_err(PDQ_ERR_ARG, "splitter arrays are NULL%s");
    const size_t need = pdq_bucket_workspace_bytes(n, nsplit + 1);
    if (!workspace || ws_bytes < need) return set_err(PDQ_ERR_WORKSPACE, "bucket workspace too small%s");
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) {
        cudaError_t e = cudaMemsetAsync(bucket_counts, 0, (size_t)(nsplit + 1) * sizeof(int64_t), s);
        return e == cudaSuccess ? PDQ_OK : set_err(PDQ_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
    }
    if (((uintptr_t)keys & 15) || ((uintptr_t)payload & 15))
        return set_err(PDQ_ERR_ALIGN, "keys and payload must be 16-byte aligned%s");
    if (nsplit == 0) {  // one bucket: a copy
        const int64_t cn = n;
        cudaError_t e = cudaMemcpyAsync(out_keys, keys, (size_t)n * dtype_size(dtype), cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess && payload)
            e = cudaMemcpyAsync(out_payload, payload, (size_t)n * 4, cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess) {  // the one bucket's size, written by the device (no host staging)
            k_set_i64<<<1, 1, 0, s>>>(bucket_counts, cn);
            e = cudaGetLastError();
        }
        return e == cudaSuccess ? PDQ_OK : set_err(PDQ_ERR_CUDA, "bucket copy: %s", cudaGetErrorString(e));
    }
    int64_t *cnt = (int64_t *)workspace;
    const bool kv = payload != nullptr;
#define PDQ_BK(U, F) \
    (kv ? launch_bucket_nb<U, F, true>(keys, payload, n, gidx_base, split_keys, split_payload, split_gidx, nsplit, \
                                    out_keys, out_payload, bucket_counts, cnt, s)                              \
        : launch_bucket_nb<U, F, false>(keys, payload, n, gidx_base, split_keys, split_payload, split_gidx, nsplit, \
                                     out_keys, out_payload, bucket_counts, cnt, s))
    switch (dtype) {
        case PDQ_I32: return PDQ_BK(uint32_t, false);
        case PDQ_F32: return PDQ_BK(uint32_t, true);
        case PDQ_I64: return PDQ_BK(uint64_t, false);
        case PDQ_F64: return PDQ_BK(uint64_t, true);
    }
#undef PDQ_BK
    return set_err(PDQ_ERR_DTYPE, "unsupported dtype code%s");
}
