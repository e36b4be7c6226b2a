// pdq_bucket_capi.cu — C ABI of the sample-sort bucketing kernels (include/pdq_b200.h: pdq_bucket*).
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include "../../include/pdq_b200.h"
#include "pdq_bucket.cuh"
#include "pdq_err.h"

using namespace pdq;

namespace {
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
}  // namespace

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
