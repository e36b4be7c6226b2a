// pdq_bucket.cuh — bucketing one rank's shard for the multi-GPU sample sort (SURVEY.md §8(e),
// row f3).  No reference counterpart: the reference is single-process.
//
// Given nsplit ascending splitters — (ordered key, payload, global index) triples — element i of
// the shard (global index gidx_base + i) belongs to bucket b = #splitters < (key, payload, gidx).
// Ties between equal elements are broken by global index, so even an all-equal input spreads
// evenly over the ranks; equal elements are bit-identical, so the order this induces is
// invisible in the output.
//
// Three stream-ordered launches, HBM-bound (w+p bytes read in pass 1, read + written in pass 3):
//   k_bucket_count   every warp owns a contiguous range of the shard and counts its elements per
//                    bucket (one ballot per bucket per 32 elements, counts held in lanes);
//   k_bucket_scan    one CTA turns the bucket-major (bucket, warp) counts into exclusive offsets
//                    and per-bucket totals;
//   k_bucket_scatter every warp walks its range again in order and writes each element at its
//                    bucket's offset + its rank among the warp's earlier elements of that bucket,
//                    so the output is stable within a bucket.
#pragma once

#include "pdq_device.cuh"

namespace pdq {

constexpr int BK_THREADS = 256;
constexpr int BK_WARPS = BK_THREADS / 32;
constexpr int BK_UNROLL = 8;                  // elements per lane per warp step (256 per step)
constexpr int BK_STEP = 32 * BK_UNROLL;
constexpr int BK_MAX = 64;                    // buckets (ranks) per call
constexpr int BK_MAX_CTAS = 148 * 8;
constexpr int BK_SCAN_THREADS = 1024;

struct BucketGeom {
    int ctas;        // CTAs of the count / scatter kernels
    int64_t per_warp;  // elements per warp range (a multiple of BK_STEP)
    __host__ __device__ int warps() const { return ctas * BK_WARPS; }
};

__host__ __device__ inline BucketGeom bucket_geom(int64_t n) {
    BucketGeom g;
    int64_t steps = (n + BK_STEP - 1) / BK_STEP;
    int64_t want = (steps + BK_WARPS - 1) / BK_WARPS;  // one step per warp at the least
    g.ctas = (int)(want < 1 ? 1 : (want > BK_MAX_CTAS ? BK_MAX_CTAS : want));
    int64_t w = (int64_t)g.ctas * BK_WARPS;
    g.per_warp = ((steps + w - 1) / w) * BK_STEP;
    return g;
}

template <class U, bool FLOAT, bool KV>
struct Bucketer {
    struct Smem {
        U sk[BK_MAX - 1];
        uint32_t sv[BK_MAX - 1];
        int64_t sg[BK_MAX - 1];
    };

    __device__ static void load_splitters(Smem &s, const U *k, const uint32_t *v, const int64_t *g, int ns) {
        for (int i = threadIdx.x; i < ns; i += blockDim.x) {
            s.sk[i] = Ord<U, FLOAT>::to(k[i]);
            s.sv[i] = KV ? v[i] : 0u;
            s.sg[i] = g[i];
        }
        __syncthreads();
    }

    // number of splitters strictly below (k, v, g)
    __device__ __forceinline__ static int bucket_of(const Smem &s, int ns, U k, uint32_t v, int64_t g) {
        int lo = 0, hi = ns;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            U a = s.sk[mid];
            bool below = a < k || (a == k && (KV ? (s.sv[mid] < v || (s.sv[mid] == v && s.sg[mid] < g)) : s.sg[mid] < g));
            lo = below ? mid + 1 : lo;
            hi = below ? hi : mid;
        }
        return lo;
    }
};

// Pass 1: per-warp bucket counts, stored bucket-major: cnt[b * warps + warp].
template <class U, bool FLOAT, bool KV>
__global__ void __launch_bounds__(BK_THREADS) k_bucket_count(const U *keys, const uint32_t *vals, int64_t n,
                                                             int64_t gidx_base, const U *sk, const uint32_t *sv,
                                                             const int64_t *sg, int ns, int64_t *cnt,
                                                             BucketGeom geom) {
    using B = Bucketer<U, FLOAT, KV>;
    __shared__ typename B::Smem s;
    B::load_splitters(s, sk, sv, sg, ns);
    const int lane = threadIdx.x & 31;
    const int warp = blockIdx.x * BK_WARPS + (threadIdx.x >> 5);
    const int nb = ns + 1;
    const int64_t lo = (int64_t)warp * geom.per_warp;
    const int64_t hi = lo + geom.per_warp < n ? lo + geom.per_warp : n;
    int64_t c0 = 0, c1 = 0;  // lane q counts bucket q (c0) and bucket q + 32 (c1)
    for (int64_t base = lo; base < hi; base += BK_STEP) {
        U k[BK_UNROLL];
        uint32_t v[BK_UNROLL];
#pragma unroll
        for (int u = 0; u < BK_UNROLL; ++u) {
            int64_t e = base + u * 32 + lane;
            k[u] = e < hi ? ldcg(keys + e) : (U)0;
            v[u] = (KV && e < hi) ? ldcg(vals + e) : 0u;
        }
#pragma unroll
        for (int u = 0; u < BK_UNROLL; ++u) {
            int64_t e = base + u * 32 + lane;
            int b = e < hi ? B::bucket_of(s, ns, Ord<U, FLOAT>::to(k[u]), v[u], gidx_base + e) : -1;
            for (int q = 0; q < nb; ++q) {
                unsigned m = __ballot_sync(0xffffffffu, b == q);
                if (q < 32) {
                    if (lane == q) c0 += __popc(m);
                } else if (lane == q - 32) {
                    c1 += __popc(m);
                }
            }
        }
    }
    const int W = geom.warps();
    if (lane < nb) cnt[(int64_t)lane * W + warp] = c0;
    if (lane + 32 < nb) cnt[(int64_t)(lane + 32) * W + warp] = c1;
}

// Pass 2: exclusive scan of the m = nb * warps counts in place; bucket totals.
__global__ void __launch_bounds__(BK_SCAN_THREADS) k_bucket_scan(int64_t *cnt, int64_t m, int nb, int warps,
                                                                 int64_t *bucket_counts) {
    __shared__ int64_t part[BK_SCAN_THREADS];
    const int t = threadIdx.x;
    const int64_t per = (m + BK_SCAN_THREADS - 1) / BK_SCAN_THREADS;
    const int64_t a = t * per, b = a + per < m ? a + per : m;
    int64_t sum = 0;
    for (int64_t i = a; i < b; ++i) sum += cnt[i];
    part[t] = sum;
    __syncthreads();
    for (int d = 1; d < BK_SCAN_THREADS; d <<= 1) {  // Hillis-Steele inclusive scan of the partials
        int64_t x = t >= d ? part[t - d] : 0;
        __syncthreads();
        part[t] += x;
        __syncthreads();
    }
    int64_t run = part[t] - sum;
    for (int64_t i = a; i < b; ++i) {
        int64_t c = cnt[i];
        cnt[i] = run;
        run += c;
    }
    __syncthreads();  // the block's global writes are visible to the block after the barrier
    if (t < nb) {
        int64_t start = cnt[(int64_t)t * warps];
        int64_t end = t + 1 < nb ? cnt[(int64_t)(t + 1) * warps] : part[BK_SCAN_THREADS - 1];
        bucket_counts[t] = end - start;
    }
}

// Pass 3: stable scatter to the bucket offsets.
template <class U, bool FLOAT, bool KV>
__global__ void __launch_bounds__(BK_THREADS) k_bucket_scatter(const U *keys, const uint32_t *vals, int64_t n,
                                                               int64_t gidx_base, const U *sk, const uint32_t *sv,
                                                               const int64_t *sg, int ns, const int64_t *off,
                                                               U *out_keys, uint32_t *out_vals, BucketGeom geom) {
    using B = Bucketer<U, FLOAT, KV>;
    __shared__ typename B::Smem s;
    B::load_splitters(s, sk, sv, sg, ns);
    const int lane = threadIdx.x & 31;
    const int warp = blockIdx.x * BK_WARPS + (threadIdx.x >> 5);
    const int nb = ns + 1;
    const int W = geom.warps();
    const int64_t lo = (int64_t)warp * geom.per_warp;
    const int64_t hi = lo + geom.per_warp < n ? lo + geom.per_warp : n;
    int64_t o0 = lane < nb ? off[(int64_t)lane * W + warp] : 0;  // lane q: next slot of bucket q
    int64_t o1 = lane + 32 < nb ? off[(int64_t)(lane + 32) * W + warp] : 0;
    const unsigned lt = lanemask_lt();
    for (int64_t base = lo; base < hi; base += BK_STEP) {
        U k[BK_UNROLL];
        uint32_t v[BK_UNROLL];
#pragma unroll
        for (int u = 0; u < BK_UNROLL; ++u) {
            int64_t e = base + u * 32 + lane;
            k[u] = e < hi ? ldcg(keys + e) : (U)0;
            v[u] = (KV && e < hi) ? ldcg(vals + e) : 0u;
        }
#pragma unroll
        for (int u = 0; u < BK_UNROLL; ++u) {
            int64_t e = base + u * 32 + lane;
            int b = e < hi ? B::bucket_of(s, ns, Ord<U, FLOAT>::to(k[u]), v[u], gidx_base + e) : -1;
            int64_t pos = 0;
            for (int q = 0; q < nb; ++q) {
                unsigned m = __ballot_sync(0xffffffffu, b == q);
                if (!m) continue;
                int64_t at = __shfl_sync(0xffffffffu, q < 32 ? o0 : o1, q & 31);
                if (b == q) pos = at + __popc(m & lt);
                if (q < 32) {
                    if (lane == q) o0 += __popc(m);
                } else if (lane == q - 32) {
                    o1 += __popc(m);
                }
            }
            if (b >= 0) {
                out_keys[pos] = k[u];
                if (KV) out_vals[pos] = v[u];
            }
        }
    }
}

}  // namespace pdq
