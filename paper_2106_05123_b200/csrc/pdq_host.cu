// pdq_host.cu — host-buffer entry of the C ABI (include/pdq_b200.h: pdq_host_*).
//
// The reference's sort(data) (driver.py:267-270) mutates a HOST sequence in place and returns.
// pdq_host_sort() is that call for flat numeric host arrays: the caller's keys (+ payload) are
// copied to the device, sorted by pdq_sort_ex() and copied back into the same host buffers before
// the call returns.
//
// Transfers.  A pageable buffer cannot be DMA'd directly; the CUDA driver's own pageable path
// stages it through a small bounce buffer with one CPU thread.  Here T worker threads each own
// two pinned staging slots and one stream: a worker copies its chunk of the caller's buffer into a
// slot (memcpy, all T in parallel) while the DMA of its previous slot runs, so the host-side copies
// of T threads overlap the PCIe transfer.  D2H is the mirror image (DMA into a slot, then memcpy
// out of it while the next chunk's DMA runs).
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/pdq_b200.h"

#include <nvtx3/nvToolsExt.h>  // header-only; ranges are no-ops unless a profiler is attached

#if defined(__x86_64__)
#include <emmintrin.h>
#endif

namespace {

// memcpy with non-temporal (streaming) stores: the destination (a pinned slot about to be DMA'd, or
// the caller's buffer) is not read back by this CPU, so streaming stores skip the read-for-ownership
// of every destination line -- a third of the host memory traffic of a staged copy.
// $PDQ_HOST_NT=0 uses plain memcpy.
bool g_nt = true;
void copy_nt(unsigned char *dst, const unsigned char *src, size_t n) {
#if defined(__x86_64__)
    if (g_nt && n >= 4096) {
        size_t h = (16 - ((uintptr_t)dst & 15)) & 15;
        memcpy(dst, src, h);
        dst += h;
        src += h;
        n -= h;
        size_t i = 0;
        for (; i + 64 <= n; i += 64) {
            const __m128i a = _mm_loadu_si128((const __m128i *)(src + i));
            const __m128i b = _mm_loadu_si128((const __m128i *)(src + i + 16));
            const __m128i c = _mm_loadu_si128((const __m128i *)(src + i + 32));
            const __m128i d = _mm_loadu_si128((const __m128i *)(src + i + 48));
            _mm_stream_si128((__m128i *)(dst + i), a);
            _mm_stream_si128((__m128i *)(dst + i + 16), b);
            _mm_stream_si128((__m128i *)(dst + i + 32), c);
            _mm_stream_si128((__m128i *)(dst + i + 48), d);
        }
        _mm_sfence();
        memcpy(dst + i, src + i, n - i);
        return;
    }
#endif
    memcpy(dst, src, n);
}

constexpr size_t CHUNK_DEFAULT = 4u << 20;  // bytes per staging slot ($PDQ_HOST_CHUNK_KB overrides; tools/host_sweep.py)
constexpr int MAX_SLOTS = 8;               // staging slots per worker ($PDQ_HOST_SLOTS, default 2)

struct Seg1 {  // one array to transfer: host <-> device, `bytes` long
    unsigned char *host;
    unsigned char *dev;
    size_t bytes;
};

struct Worker {
    std::thread th;
    cudaStream_t stream = nullptr;
    unsigned char *slot[MAX_SLOTS] = {};
    cudaEvent_t ev[MAX_SLOTS] = {};
    cudaEvent_t done = nullptr;
    int rc = 0;
};

}  // namespace

struct pdq_host_sorter {
    int device = 0;
    cudaStream_t stream = nullptr;  // the sort's stream
    cudaEvent_t ev_h2d = nullptr, ev_sort = nullptr, ev_k0 = nullptr, ev_k1 = nullptr, ev_t0 = nullptr;
    unsigned char *d_keys = nullptr, *d_vals = nullptr, *d_ws = nullptr;
    size_t cap_keys = 0, cap_vals = 0, cap_ws = 0;
    int nthreads = 1;
    size_t chunk = CHUNK_DEFAULT;
    int nslots = 2;
    std::vector<Worker> w;
    // job dispatch to the worker pool
    std::mutex mu;
    std::condition_variable cv, cv_done;
    uint64_t gen = 0;
    int pending = 0;
    bool quit = false;
    std::function<void(int)> job;
    std::mutex call_mu;  // one sort at a time per sorter
    char err[256] = {0};
};

namespace {

int fail(pdq_host_sorter *h, const char *what, cudaError_t e) {
    snprintf(h->err, sizeof(h->err), "%s: %s", what, cudaGetErrorString(e));
    return PDQ_ERR_CUDA;
}

void worker_main(pdq_host_sorter *h, int id) {
    cudaSetDevice(h->device);
    uint64_t seen = 0;
    for (;;) {
        std::function<void(int)> f;
        {
            std::unique_lock<std::mutex> lk(h->mu);
            h->cv.wait(lk, [&] { return h->quit || h->gen != seen; });
            if (h->quit) return;
            seen = h->gen;
            f = h->job;
        }
        f(id);
        {
            std::lock_guard<std::mutex> lk(h->mu);
            if (--h->pending == 0) h->cv_done.notify_all();
        }
    }
}

// run f(worker id) on every worker and wait for all of them
void run_all(pdq_host_sorter *h, std::function<void(int)> f) {
    {
        std::lock_guard<std::mutex> lk(h->mu);
        h->job = std::move(f);
        h->pending = h->nthreads;
        ++h->gen;
    }
    h->cv.notify_all();
    std::unique_lock<std::mutex> lk(h->mu);
    h->cv_done.wait(lk, [&] { return h->pending == 0; });
}

// chunk c of the concatenated segments -> (segment, offset, bytes)
struct ChunkRef {
    const Seg1 *s;
    size_t off, bytes;
};
// Chunks of `chunk` bytes, except that the first and the last `workers` chunks of the whole transfer
// ramp up from / taper down to chunk / 8 (three rounds each): the first DMA starts after a short host
// copy instead of a full slot, and the last host copy-out after the final DMA is short
// ($PDQ_HOST_RAMP=0: equal chunks).
bool g_ramp = true;
std::vector<ChunkRef> chunk_list(const std::vector<Seg1> &segs, size_t chunk, int workers) {
    std::vector<ChunkRef> out;
    size_t total = 0;
    for (const Seg1 &s : segs) total += s.bytes;
    const size_t gran = 64u << 10;
    const bool ramp = g_ramp && chunk >= 8 * gran && total >= (size_t)workers * chunk * 8;
    size_t done = 0;  // bytes of the whole transfer before the current position
    const size_t edge = ramp ? (size_t)workers * (chunk / 8 + chunk / 4 + chunk / 2) : 0;
    auto size_at = [&](size_t pos) -> size_t {  // size of the chunk that starts `pos` bytes into the transfer
        if (!ramp) return chunk;
        const size_t w = (size_t)workers;
        const size_t d = std::min(pos, total - pos - 1);  // distance from the nearer end (the tail mirrors the head)
        if (d < w * (chunk / 8)) return chunk / 8;
        if (d < w * (chunk / 8 + chunk / 4)) return chunk / 4;
        if (d < edge) return chunk / 2;
        return chunk;
    };
    for (const Seg1 &s : segs) {
        for (size_t off = 0; off < s.bytes;) {
            const size_t c = std::min(size_at(done + off), s.bytes - off);
            out.push_back({&s, off, c});
            off += c;
        }
        done += s.bytes;
    }
    return out;
}

// H2D: worker id takes chunks id, id + T, ...; memcpy into slot k while the DMAs of its other slots run
void h2d_worker(pdq_host_sorter *h, int id, const std::vector<ChunkRef> &ch) {
    Worker &w = h->w[id];
    int k = 0;
    bool used[MAX_SLOTS] = {};
    for (size_t c = id; c < ch.size(); c += h->nthreads) {
        const ChunkRef &r = ch[c];
        if (used[k]) {
            cudaError_t e = cudaEventSynchronize(w.ev[k]);  // the slot's previous DMA has read it
            if (e != cudaSuccess) { w.rc = fail(h, "h2d slot wait", e); return; }
        }
        copy_nt(w.slot[k], r.s->host + r.off, r.bytes);
        cudaError_t e = cudaMemcpyAsync(r.s->dev + r.off, w.slot[k], r.bytes, cudaMemcpyHostToDevice, w.stream);
        if (e == cudaSuccess) e = cudaEventRecord(w.ev[k], w.stream);
        if (e != cudaSuccess) { w.rc = fail(h, "h2d copy", e); return; }
        used[k] = true;
        k = (k + 1) % h->nslots;
    }
    cudaError_t e = cudaEventRecord(w.done, w.stream);
    if (e != cudaSuccess) w.rc = fail(h, "h2d done", e);
}

// D2H: DMAs of the next chunks run into the other slots while chunk i is copied out of its slot
void d2h_worker(pdq_host_sorter *h, int id, const std::vector<ChunkRef> &ch) {
    Worker &w = h->w[id];
    const int S = h->nslots;
    cudaError_t e = cudaStreamWaitEvent(w.stream, h->ev_sort, 0);
    if (e != cudaSuccess) { w.rc = fail(h, "d2h wait", e); return; }
    std::vector<size_t> mine;
    for (size_t c = id; c < ch.size(); c += h->nthreads) mine.push_back(c);
    auto issue = [&](size_t i) -> cudaError_t {
        const ChunkRef &r = ch[mine[i]];
        cudaError_t e2 = cudaMemcpyAsync(w.slot[i % S], r.s->dev + r.off, r.bytes, cudaMemcpyDeviceToHost, w.stream);
        if (e2 == cudaSuccess) e2 = cudaEventRecord(w.ev[i % S], w.stream);
        return e2;
    };
    for (size_t i = 0; i < mine.size() && i + 1 < (size_t)S; ++i)
        if ((e = issue(i)) != cudaSuccess) { w.rc = fail(h, "d2h copy", e); return; }
    for (size_t i = 0; i < mine.size(); ++i) {
        if (i + S - 1 < mine.size() && (e = issue(i + S - 1)) != cudaSuccess) { w.rc = fail(h, "d2h copy", e); return; }
        if ((e = cudaEventSynchronize(w.ev[i % S])) != cudaSuccess) { w.rc = fail(h, "d2h slot wait", e); return; }
        const ChunkRef &r = ch[mine[i]];
        copy_nt(r.s->host + r.off, w.slot[i % S], r.bytes);
    }
}

int ensure(pdq_host_sorter *h, unsigned char *&p, size_t &cap, size_t need) {
    if (cap >= need) return 0;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = need + need / 8;  // grow with slack
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
        e = cudaMalloc(&p, need);
        if (e != cudaSuccess) return fail(h, "device buffer", e);
        want = need;
    }
    cap = want;
    return 0;
}

int dsize(int dtype) { return (dtype == PDQ_I32 || dtype == PDQ_F32) ? 4 : (dtype == PDQ_I64 || dtype == PDQ_F64) ? 8 : 0; }

}  // namespace

extern "C" pdq_host_sorter *pdq_host_sorter_create(int device, int threads) {
    pdq_host_sorter *h = new pdq_host_sorter();
    h->device = device;
    if (threads <= 0) {
        const char *env = getenv("PDQ_HOST_THREADS");
        threads = env ? atoi(env) : 0;
        if (threads <= 0) {
            unsigned hw = std::thread::hardware_concurrency();
            threads = (int)std::min(16u, std::max(1u, hw));
        }
    }
    h->nthreads = std::min(threads, 64);
    if (const char *nt = getenv("PDQ_HOST_NT")) g_nt = atoi(nt) != 0;
    if (const char *rp = getenv("PDQ_HOST_RAMP")) g_ramp = atoi(rp) != 0;
    if (const char *sl = getenv("PDQ_HOST_SLOTS")) h->nslots = std::max(2, std::min(MAX_SLOTS, atoi(sl)));
    if (const char *ck = getenv("PDQ_HOST_CHUNK_KB")) {
        const long kb = atol(ck);
        if (kb >= 64 && kb <= (256l << 10)) h->chunk = (size_t)kb << 10;
    }
    bool ok = cudaSetDevice(device) == cudaSuccess && cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) == cudaSuccess;
    for (cudaEvent_t *e : {&h->ev_h2d, &h->ev_sort, &h->ev_k0, &h->ev_k1, &h->ev_t0})
        ok = ok && cudaEventCreate(e) == cudaSuccess;
    h->w.resize(h->nthreads);
    for (Worker &w : h->w) {
        ok = ok && cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking) == cudaSuccess;
        for (int k = 0; k < h->nslots; ++k) {
            ok = ok && cudaHostAlloc((void **)&w.slot[k], h->chunk, cudaHostAllocPortable) == cudaSuccess;
            ok = ok && cudaEventCreateWithFlags(&w.ev[k], cudaEventDisableTiming) == cudaSuccess;
        }
        ok = ok && cudaEventCreateWithFlags(&w.done, cudaEventDisableTiming) == cudaSuccess;
    }
    if (!ok) {
        cudaGetLastError();
        pdq_host_sorter_destroy(h);
        return nullptr;
    }
    for (int i = 0; i < h->nthreads; ++i) h->w[i].th = std::thread(worker_main, h, i);
    return h;
}

extern "C" void pdq_host_sorter_destroy(pdq_host_sorter *h) {
    if (!h) return;
    {
        std::lock_guard<std::mutex> lk(h->mu);
        h->quit = true;
    }
    h->cv.notify_all();
    for (Worker &w : h->w)
        if (w.th.joinable()) w.th.join();
    cudaSetDevice(h->device);
    for (Worker &w : h->w) {
        if (w.stream) cudaStreamSynchronize(w.stream), cudaStreamDestroy(w.stream);
        for (int k = 0; k < MAX_SLOTS; ++k) {
            if (w.slot[k]) cudaFreeHost(w.slot[k]);
            if (w.ev[k]) cudaEventDestroy(w.ev[k]);
        }
        if (w.done) cudaEventDestroy(w.done);
    }
    if (h->stream) cudaStreamSynchronize(h->stream), cudaStreamDestroy(h->stream);
    for (cudaEvent_t e : {h->ev_h2d, h->ev_sort, h->ev_k0, h->ev_k1, h->ev_t0})
        if (e) cudaEventDestroy(e);
    for (unsigned char *p : {h->d_keys, h->d_vals, h->d_ws})
        if (p) cudaFree(p);
    delete h;
}

extern "C" const char *pdq_host_sorter_error(const pdq_host_sorter *h) { return h ? h->err : "NULL sorter"; }

extern "C" int pdq_host_sort(pdq_host_sorter *h, void *keys, int dtype, uint32_t *payload, int64_t n,
                             const pdq_config *cfg, pdq_stats *stats, double *phase_ms) {
    if (!h) return PDQ_ERR_ARG;
    std::lock_guard<std::mutex> call(h->call_mu);
    h->err[0] = 0;
    const int w = dsize(dtype);
    if (w == 0) { snprintf(h->err, sizeof(h->err), "unsupported dtype code"); return PDQ_ERR_DTYPE; }
    if (n < 0 || (n > 0 && !keys)) { snprintf(h->err, sizeof(h->err), "bad keys / n"); return PDQ_ERR_ARG; }
    if (stats) memset(stats, 0, sizeof(*stats));
    if (phase_ms) phase_ms[0] = phase_ms[1] = phase_ms[2] = phase_ms[3] = 0.0;
    if (n <= 1) return PDQ_OK;
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) return fail(h, "set device", e);
    const auto t0 = std::chrono::steady_clock::now();
    const size_t kb = (size_t)n * w, vb = payload ? (size_t)n * 4 : 0;
    const size_t wsb = pdq_workspace_bytes(dtype, payload != nullptr, n);
    int rc = ensure(h, h->d_keys, h->cap_keys, kb);
    if (!rc && payload) rc = ensure(h, h->d_vals, h->cap_vals, vb);
    if (!rc) rc = ensure(h, h->d_ws, h->cap_ws, wsb);
    if (rc) return rc;

    std::vector<Seg1> segs{{(unsigned char *)keys, h->d_keys, kb}};
    if (payload) segs.push_back({(unsigned char *)payload, h->d_vals, vb});
    // chunks: the slot size, or smaller so that a small array still spreads over every worker
    size_t ck = (kb + vb + h->nthreads - 1) / h->nthreads;
    ck = std::max<size_t>(64u << 10, std::min(h->chunk, (ck + (64u << 10) - 1) & ~(size_t)((64u << 10) - 1)));
    const std::vector<ChunkRef> ch = chunk_list(segs, ck, h->nthreads);
    for (Worker &wk : h->w) wk.rc = 0;

    // 1. H2D through the pinned slots (all workers)
    if ((e = cudaEventRecord(h->ev_t0, h->stream)) != cudaSuccess) return fail(h, "event", e);
    for (Worker &wk : h->w)  // worker streams start after anything earlier on the sort stream
        if ((e = cudaStreamWaitEvent(wk.stream, h->ev_t0, 0)) != cudaSuccess) return fail(h, "stream wait", e);
    nvtxRangePushA("pdq_host_sort h2d");
    run_all(h, [&](int id) { h2d_worker(h, id, ch); });
    nvtxRangePop();
    for (Worker &wk : h->w) {
        if (wk.rc) return wk.rc;
        if ((e = cudaStreamWaitEvent(h->stream, wk.done, 0)) != cudaSuccess) return fail(h, "join h2d", e);
    }
    if ((e = cudaEventRecord(h->ev_h2d, h->stream)) != cudaSuccess) return fail(h, "event", e);
    const auto t1 = std::chrono::steady_clock::now();

    // 2. sort (stream-ordered), then the status: nothing is copied back from a failed sort
    rc = pdq_sort(h->d_keys, dtype, payload ? (uint32_t *)h->d_vals : nullptr, n, cfg, h->d_ws, h->cap_ws,
                  h->stream);
    if (rc) return rc;
    if ((e = cudaEventRecord(h->ev_sort, h->stream)) != cudaSuccess) return fail(h, "event", e);
    rc = pdq_sort_finish(h->d_ws, stats, h->stream);  // synchronises the sort stream
    if (rc) return rc;
    const auto t2 = std::chrono::steady_clock::now();

    // 3. D2H through the pinned slots into the caller's buffers
    nvtxRangePushA("pdq_host_sort d2h");
    run_all(h, [&](int id) { d2h_worker(h, id, ch); });
    nvtxRangePop();
    for (Worker &wk : h->w)
        if (wk.rc) return wk.rc;
    const auto t3 = std::chrono::steady_clock::now();
    if (phase_ms) {
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        float ksort = 0.f;
        cudaEventElapsedTime(&ksort, h->ev_h2d, h->ev_sort);
        phase_ms[0] = ms(t0, t1) + 0.0;  // host: staging + H2D issue (completion is in phase 1's wait)
        phase_ms[1] = ms(t1, t2);        // host: wait for H2D tail + sort
        phase_ms[2] = ms(t2, t3);        // host: D2H + copy-out
        phase_ms[3] = ksort;             // device: the sort alone (events)
    }
    return PDQ_OK;
}
