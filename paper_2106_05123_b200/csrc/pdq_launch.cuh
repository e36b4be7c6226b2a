// pdq_launch.cuh — launching one sort's kernels for one element type (included by pdq_inst.cu, which is
// compiled once per element type so the eight instantiations build in parallel).
#pragma once

#include <cuda_runtime.h>

#include <mutex>

#include "../../include/pdq_b200.h"
#include "pdq_err.h"
#include "pdq_kernels.cuh"

namespace pdq {

#ifndef PDQ_CHUNK_MAX
#define PDQ_CHUNK_MAX 32  // tiles per ring task at most
#endif
#ifndef PDQ_CHUNK_DIV
#define PDQ_CHUNK_DIV 2  // the root level gets about this many tasks per CTA
#endif

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
int launch(Params &P, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1, cudaEvent_t ev_end) {
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


}  // namespace pdq
