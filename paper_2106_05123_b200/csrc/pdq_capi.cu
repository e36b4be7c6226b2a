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
#include "pdq_device.cuh"
#include "pdq_err.h"

using namespace pdq;

static thread_local char g_err[512];

int pdq::set_err(int code, const char *fmt, const char *detail) {
    snprintf(g_err, sizeof(g_err), fmt, detail);
    return code;
}

extern "C" const char *pdq_last_error(void) { return g_err; }
extern "C" const char *pdq_version(void) { return "pdq_b200 0.2.0 (sm_100a)"; }

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
#ifndef PDQ_RUNS_MIN
// K4 takes the two-run path (sorted prefix of >= n/2 + merge) from this size: below it one or two leaves sort
// the array as fast (tools/runs_prof.py: organ 42 vs 59 us at 2^15, 43 vs 44 us at 2^14)
#define PDQ_RUNS_MIN (1 << 15)
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
    // at least 2^17 entries (1 MiB): ring positions only grow during a sort, and a degenerate sort of a few
    // million elements (tiny segments taking many one-tile digit passes) issues tens of thousands of them
    int lq = 17;
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
    if (dtype == PDQ_I32 && !kv) return launch_i32(P, s, ev0, ev1, eve);
    return set_err(PDQ_ERR_DTYPE, "this profiling build sorts int32 keys only%s");
#else
    switch (dtype) {
        case PDQ_I32: return kv ? launch_i32_kv(P, s, ev0, ev1, eve) : launch_i32(P, s, ev0, ev1, eve);
        case PDQ_F32: return kv ? launch_f32_kv(P, s, ev0, ev1, eve) : launch_f32(P, s, ev0, ev1, eve);
        case PDQ_I64: return kv ? launch_i64_kv(P, s, ev0, ev1, eve) : launch_i64(P, s, ev0, ev1, eve);
        case PDQ_F64: return kv ? launch_f64_kv(P, s, ev0, ev1, eve) : launch_f64(P, s, ev0, ev1, eve);
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

