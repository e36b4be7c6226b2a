// pdq_bucket.cuh — bucketing one rank's shard for the multi-GPU sample sort (SURVEY.md §8(e),
// row f3).  No reference counterpart: the reference is single-process.
//
// Given nsplit ascending splitters — (ordered key, payload, global index) triples — element i of
// the shard (global index gidx_base + i) belongs to bucket b = #splitters < (key, payload, gidx).
// Ties between equal elements are broken by global index, so even an all-equal input spreads
// evenly over the ranks; equal elements are bit-identical, so the order this induces is
// invisible in the output.
//
// Three stream-ordered launches, HBM-bound ((w+p) bytes read in pass 1, read + written in pass 3):
//   k_bucket_count   every CTA owns a contiguous range of whole 4096-element tiles; each thread
//                    counts its elements per bucket in its own shared-memory column (no atomics);
//                    the CTA's per-bucket totals are stored bucket-major, cnt[b * ctas + cta];
//   k_bucket_scan    one CTA turns them into exclusive offsets and per-bucket totals;
//   k_bucket_scatter every CTA walks its tiles again: per-thread column counts, one block scan
//                    (bucket-major) gives every element its slot in a shared-memory staging tile
//                    grouped by bucket, and the staged runs leave with coalesced stores at the
//                    CTA's running bucket cursors — stable within a bucket, deterministic.
// The bucket of an element is a branch-free binary search over the splitters (padded with +inf
// sentinels to a power of two) in shared memory.
#pragma once

#include "pdq_device.cuh"

namespace pdq {

constexpr int BK_THREADS = 256;
constexpr int BK_MAX = 64;                       // buckets (ranks) per call
constexpr int BK_MAX_CTAS = 148 * 16;            // upper bound of every element type's grid

// Per element type: elements per thread per tile (4-byte keys: 16, wider elements: 8, which keeps
// them in registers without spilling) and the CTAs per SM the registers allow.
template <class U, bool KV>
struct BkShape {
    static constexpr int IPT = (sizeof(U) == 4 && !KV) ? 16 : 8;
    static constexpr int TILE = BK_THREADS * IPT;
#ifndef PDQ_BK_MINB16
#define PDQ_BK_MINB16 3
#endif
    static constexpr int MINB = IPT == 16 ? PDQ_BK_MINB16 : 4;
#ifndef PDQ_BK_WAVES
#define PDQ_BK_WAVES 4
#endif
    static constexpr int CTAS = 148 * PDQ_BK_WAVES * MINB;
    static_assert(CTAS <= BK_MAX_CTAS, "the count workspace is sized for BK_MAX_CTAS CTAs");
};
constexpr int BK_SCAN_THREADS = 1024;

struct BucketGeom {
    int ctas;           // CTAs of the count / scatter kernels
    int64_t per_cta;    // elements per CTA range (whole tiles)
};

__host__ __device__ inline BucketGeom bucket_geom(int64_t n, int tile, int max_ctas) {
    BucketGeom g;
    int64_t tiles = (n + tile - 1) / tile;
    g.ctas = (int)(tiles < 1 ? 1 : (tiles > max_ctas ? max_ctas : tiles));
    g.per_cta = ((tiles + g.ctas - 1) / g.ctas) * tile;
    return g;
}

__host__ __device__ inline int bucket_log2(int nb) {  // splitter table of 2^L - 1 entries, L >= 0
    int l = 0;
    while ((1 << l) < nb) ++l;
    return l;
}

template <class U, bool FLOAT, bool KV>
struct Bucketer {
    static constexpr int BK_IPT = BkShape<U, KV>::IPT;
    static constexpr int BK_TILE = BkShape<U, KV>::TILE;
    struct Split {
        U sk[BK_MAX];
        uint32_t sv[BK_MAX];
        int64_t sg[BK_MAX];
    };

    // splitters in ordered images; entries ns .. 2^L - 2 are +inf sentinels (above every element)
    __device__ static void load_splitters(Split &s, const U *k, const uint32_t *v, const int64_t *g, int ns, int L) {
        for (int i = threadIdx.x; i < (1 << L) - 1; i += blockDim.x) {
            bool real = i < ns;
            s.sk[i] = real ? Ord<U, FLOAT>::to(k[i]) : ~(U)0;
            s.sv[i] = real && KV ? v[i] : 0xFFFFFFFFu;
            s.sg[i] = real ? g[i] : INT64_MAX;
        }
    }

    // number of splitters strictly below (k, v, g): branch-free search over the 2^L - 1 table on the
    // key alone (L <= 6, unrolled; independent elements overlap their shared-memory latencies); an
    // element that meets a splitter with an equal key repeats the search with the full
    // (key, payload, global index) comparison
    __device__ __noinline__ static int bucket_tie(const Split &s, int L, U k, uint32_t v, int64_t g) {
        int pos = 0;
        for (int step = (1 << L) >> 1; step > 0; step >>= 1) {
            const int i = pos + step - 1;
            const U a = s.sk[i];
            bool below = a < k;
            if (a == k) below = KV ? (s.sv[i] < v || (s.sv[i] == v && s.sg[i] < g)) : s.sg[i] < g;
            pos += below ? step : 0;
        }
        return pos;
    }
    // buckets of this thread's BK_IPT elements (0xFF for the `valid`-th and later ones).  LT >= 0: the
    // table depth is a compile-time constant (the search unrolls to LT compare-and-select steps);
    // LT < 0: runtime depth L <= 6
    template <int LT>
    __device__ __forceinline__ static void buckets(const Split &s, int L, const U (&k)[BK_IPT],
                                                   const uint32_t (&v)[BK_IPT], int64_t g0, int valid,
                                                   uint8_t (&b)[BK_IPT]) {
        unsigned ties = 0;
        int pos[BK_IPT];
#pragma unroll
        for (int j = 0; j < BK_IPT; ++j) {
            const U x = Ord<U, FLOAT>::to(k[j]);
            int p = 0;
            bool tie = false;
            if (LT >= 0) {
#pragma unroll
                for (int i = 0; i < (LT > 0 ? LT : 0); ++i) {
                    const int step = 1 << (LT - 1 - i);
                    const U a = s.sk[p + step - 1];
                    tie |= a == x;
                    p += a < x ? step : 0;
                }
            } else {
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    if (i < L) {
                        const int step = 1 << (L - 1 - i);
                        const U a = s.sk[p + step - 1];
                        tie |= a == x;
                        p += a < x ? step : 0;
                    }
                }
            }
            pos[j] = p;
            ties |= (tie && j < valid ? 1u : 0u) << j;
        }
        if (ties) {  // rare: an element whose key equals a splitter's is placed by (key, payload, index)
#pragma unroll
            for (int j = 0; j < BK_IPT; ++j)
                if (ties >> j & 1) pos[j] = bucket_tie(s, L, Ord<U, FLOAT>::to(k[j]), v[j], g0 + j);
        }
#pragma unroll
        for (int j = 0; j < BK_IPT; ++j) b[j] = j < valid ? (uint8_t)pos[j] : (uint8_t)0xFF;
    }

    // per-thread bucket counts of one tile packed in 8-bit fields (nb <= 8, <= 16 elements)
    __device__ __forceinline__ static uint64_t packed_counts(const uint8_t (&b)[BK_IPT]) {
        uint64_t pk = 0;
#pragma unroll
        for (int j = 0; j < BK_IPT; ++j) pk += b[j] != 0xFF ? 1ull << (8 * b[j]) : 0ull;
        return pk;
    }

    // this thread's BK_IPT consecutive elements of the tile at `t0` (guarded by `hi`)
    __device__ __forceinline__ static void load(const U *keys, const uint32_t *vals, int64_t t0, int64_t hi,
                                                U (&k)[BK_IPT], uint32_t (&v)[BK_IPT]) {
        const int64_t e0 = t0 + (int64_t)threadIdx.x * BK_IPT;
        if (e0 + BK_IPT <= hi) {
            constexpr int PER = 16 / sizeof(U);
#pragma unroll
            for (int j = 0; j < BK_IPT; j += PER) {
                uint4 x = __ldg((const uint4 *)(keys + e0 + j));
                if (sizeof(U) == 4) {
                    k[j] = (U)x.x, k[j + 1] = (U)x.y, k[j + 2] = (U)x.z, k[j + 3] = (U)x.w;
                } else {
                    k[j] = (U)(((uint64_t)x.y << 32) | x.x), k[j + 1] = (U)(((uint64_t)x.w << 32) | x.z);
                }
            }
            if (KV) {
#pragma unroll
                for (int j = 0; j < BK_IPT; j += 4) {
                    uint4 y = __ldg((const uint4 *)(vals + e0 + j));
                    v[j] = y.x, v[j + 1] = y.y, v[j + 2] = y.z, v[j + 3] = y.w;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < BK_IPT; ++j) {
                const bool in = e0 + j < hi;
                k[j] = in ? __ldg(keys + e0 + j) : (U)0;
                v[j] = (KV && in) ? __ldg(vals + e0 + j) : 0u;
            }
        }
    }
};

// Pass 1: per-CTA bucket counts, stored bucket-major: cnt[b * ctas + cta].
template <class U, bool FLOAT, bool KV, int LT>
__global__ void __launch_bounds__(BK_THREADS, (BkShape<U, KV>::MINB)) k_bucket_count(const U *keys, const uint32_t *vals, int64_t n,
                                                             int64_t gidx_base, const U *sk, const uint32_t *sv,
                                                             const int64_t *sg, int ns, int64_t *cnt,
                                                             BucketGeom geom) {
    using B = Bucketer<U, FLOAT, KV>;
    constexpr bool SMALL = LT >= 0;  // <= 8 buckets: per-thread counts packed in registers
    constexpr int BK_IPT = B::BK_IPT, BK_TILE = B::BK_TILE;
    __shared__ typename B::Split s;
    extern __shared__ __align__(16) unsigned char dyn[];
    uint32_t *hist = reinterpret_cast<uint32_t *>(dyn);  // [nb][BK_THREADS]: one column per thread
    const int nb = ns + 1, L = bucket_log2(nb), t = threadIdx.x;
    B::load_splitters(s, sk, sv, sg, ns, L);
    if (!SMALL)
        for (int q = 0; q < nb; ++q) hist[q * BK_THREADS + t] = 0;
    __syncthreads();
    const int64_t lo = (int64_t)blockIdx.x * geom.per_cta;
    const int64_t hi = lo + geom.per_cta < n ? lo + geom.per_cta : n;
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // SMALL: this thread's counts per bucket
    for (int64_t t0 = lo; t0 < hi; t0 += BK_TILE) {
        U k[BK_IPT];
        uint32_t v[BK_IPT];
        uint8_t b[BK_IPT];
        B::load(keys, vals, t0, hi, k, v);
        const int64_t e0 = t0 + (int64_t)t * BK_IPT;
        const int valid = hi - e0 >= BK_IPT ? BK_IPT : (hi > e0 ? (int)(hi - e0) : 0);
        B::template buckets<LT>(s, L, k, v, gidx_base + e0, valid, b);
        if (SMALL) {
            const uint64_t pk = B::packed_counts(b);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] += (uint32_t)(pk >> (8 * q)) & 0xFFu;
        } else {
#pragma unroll
            for (int j = 0; j < BK_IPT; ++j)
                if (b[j] != 0xFF) ++hist[b[j] * BK_THREADS + t];
        }
    }
    if (SMALL) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (q < nb) hist[q * BK_THREADS + t] = acc[q];
    }
    __syncthreads();
    const int warp = t >> 5, lane = t & 31;
    for (int q = warp; q < nb; q += BK_THREADS / 32) {
        uint32_t x = 0;
        for (int i = lane; i < BK_THREADS; i += 32) x += hist[q * BK_THREADS + i];
        x = __reduce_add_sync(0xffffffffu, x);
        if (lane == 0) cnt[(int64_t)q * geom.ctas + blockIdx.x] = x;
    }
}

// Pass 2: exclusive scan of the m = nb * ctas counts in place; bucket totals.
__global__ void __launch_bounds__(BK_SCAN_THREADS) k_bucket_scan(int64_t *cnt, int64_t m, int nb, int ctas,
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
        int64_t start = cnt[(int64_t)t * ctas];
        int64_t end = t + 1 < nb ? cnt[(int64_t)(t + 1) * ctas] : part[BK_SCAN_THREADS - 1];
        bucket_counts[t] = end - start;
    }
}

// Pass 3: stable scatter through a shared-memory staging tile grouped by bucket.
// Staging slots are padded so that the 32 lanes of a warp, whose slots sit BK_IPT apart while a
// bucket's run is filled, hit distinct banks: element slot p lives at p + p / BK_IPT, its bucket
// byte at p + 4 (p / BK_IPT).
template <int BK_IPT>
__device__ __forceinline__ int pad_w(int p) { return p + p / BK_IPT; }
template <int BK_IPT>
__device__ __forceinline__ int pad_b(int p) { return p + 4 * (p / BK_IPT); }

template <class U, bool KV>
struct ScatterSmem {
    static constexpr int BK_IPT = BkShape<U, KV>::IPT, BK_TILE = BkShape<U, KV>::TILE;
    U sk[BK_TILE + BK_TILE / BK_IPT];
    uint32_t sv[KV ? BK_TILE + BK_TILE / BK_IPT : 1];
    uint8_t sb[BK_TILE + 4 * BK_TILE / BK_IPT];
    int32_t tstart[BK_MAX + 1];
    int64_t cur[BK_MAX];
    int64_t delta[BK_MAX];  // cur - tstart: global position of staging slot 0's bucket run
    int64_t part[BK_THREADS / 32];
    uint64_t wp[2][2][BK_THREADS / 32];  // <= 8 buckets: per-warp 16-bit-field count totals, by tile parity
};

template <class U, bool FLOAT, bool KV, int LT>
__global__ void __launch_bounds__(BK_THREADS, (BkShape<U, KV>::MINB)) k_bucket_scatter(const U *keys, const uint32_t *vals, int64_t n,
                                                               int64_t gidx_base, const U *sk, const uint32_t *sv,
                                                               const int64_t *sg, int ns, const int64_t *off,
                                                               U *out_keys, uint32_t *out_vals, BucketGeom geom) {
    using B = Bucketer<U, FLOAT, KV>;
    constexpr bool SMALL = LT >= 0;
    constexpr int BK_IPT = B::BK_IPT, BK_TILE = B::BK_TILE;
    __shared__ typename B::Split s;
    extern __shared__ __align__(16) unsigned char dyn[];
    ScatterSmem<U, KV> &st = *reinterpret_cast<ScatterSmem<U, KV> *>(dyn);
    uint32_t *hist = reinterpret_cast<uint32_t *>(dyn + sizeof(ScatterSmem<U, KV>));  // [nb][BK_THREADS]
    const int nb = ns + 1, L = bucket_log2(nb), t = threadIdx.x, lane = t & 31, warp = t >> 5;
    B::load_splitters(s, sk, sv, sg, ns, L);
    if (t < nb) st.cur[t] = off[(int64_t)t * geom.ctas + blockIdx.x];
    __syncthreads();  // splitter table ready
    const int64_t lo = (int64_t)blockIdx.x * geom.per_cta;
    const int64_t hi = lo + geom.per_cta < n ? lo + geom.per_cta : n;
    int par = 0;
    for (int64_t t0 = lo; t0 < hi; t0 += BK_TILE, par ^= 1) {
        U k[BK_IPT];
        uint32_t v[BK_IPT];
        uint8_t b[BK_IPT];
        B::load(keys, vals, t0, hi, k, v);
        const int64_t e0 = t0 + (int64_t)t * BK_IPT;
        const int valid = hi - e0 >= BK_IPT ? BK_IPT : (hi > e0 ? (int)(hi - e0) : 0);
        B::template buckets<LT>(s, L, k, v, gidx_base + e0, valid, b);
        // (4-byte keys with <= 4 buckets keep the per-thread column pass below: cheaper at that size)
        if constexpr (SMALL && (LT == 3 || BK_IPT == 8)) {
            // Counts as 16-bit fields (buckets 0-3 in c0, 4-7 in c1; a tile holds <= 4096 elements), one
            // warp scan of the packed words, per-warp totals through shared memory (double-buffered by
            // tile parity), field-wise prefix sums by multiplication: no per-bucket shared-memory pass.
            uint64_t c0 = 0, c1 = 0;
#pragma unroll
            for (int j = 0; j < BK_IPT; ++j) {
                const uint64_t one = 1ull << (16 * (b[j] & 3));
                if (b[j] < 4) c0 += one;
                else if (b[j] != 0xFF) c1 += one;
            }
            uint64_t i0 = c0, i1 = c1;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint64_t y0 = __shfl_up_sync(0xffffffffu, i0, d), y1 = __shfl_up_sync(0xffffffffu, i1, d);
                if (lane >= d) i0 += y0, i1 += y1;
            }
            if (lane == 31) st.wp[par][0][warp] = i0, st.wp[par][1][warp] = i1;
            __syncthreads();  // (also: the previous tile's output loop is done with st.sk / sb / delta)
            uint64_t w0 = 0, w1 = 0, T0 = 0, T1 = 0;
#pragma unroll
            for (int w = 0; w < BK_THREADS / 32; ++w) {
                const uint64_t a = st.wp[par][0][w], a1 = st.wp[par][1][w];
                if (w < warp) w0 += a, w1 += a1;
                T0 += a, T1 += a1;
            }
            constexpr uint64_t M = 0x0001000100010001ull;  // field k of x * M = sum of fields 0..k of x
            const uint64_t s0 = T0 * M - T0, s1 = T1 * M - T1 + ((T0 * M) >> 48) * M;  // tile bucket starts
            uint64_t base0 = s0 + w0 + i0 - c0, base1 = s1 + w1 + i1 - c1;  // this thread's first slots
            if (t < nb) {
                const int f = 16 * (t & 3);
                st.delta[t] = st.cur[t] - (int64_t)(((t < 4 ? s0 : s1) >> f) & 0xFFFFu);
                st.cur[t] += (int64_t)(((t < 4 ? T0 : T1) >> f) & 0xFFFFu);
            }
#pragma unroll
            for (int j = 0; j < BK_IPT; ++j) {
                if (b[j] != 0xFF) {
                    const int f = 16 * (b[j] & 3);
                    const bool lo4 = b[j] < 4;
                    const int p = (int)(((lo4 ? base0 : base1) >> f) & 0xFFFFu);
                    if (lo4) base0 += 1ull << f;
                    else base1 += 1ull << f;
                    st.sk[pad_w<BK_IPT>(p)] = k[j];
                    if (KV) st.sv[pad_w<BK_IPT>(p)] = v[j];
                    st.sb[pad_b<BK_IPT>(p)] = b[j];
                }
            }
            __syncthreads();
            const int tn = (int)(hi - t0 < BK_TILE ? hi - t0 : BK_TILE);
            for (int p = t; p < tn; p += BK_THREADS) {
                const int64_t g = st.delta[st.sb[pad_b<BK_IPT>(p)]] + p;
                out_keys[g] = st.sk[pad_w<BK_IPT>(p)];
                if (KV) out_vals[g] = st.sv[pad_w<BK_IPT>(p)];
            }
            continue;
        }
        __syncthreads();  // the previous tile's readers of st / hist are done
        {
            for (int q = 0; q < nb; ++q) hist[q * BK_THREADS + t] = 0;
#pragma unroll
            for (int j = 0; j < BK_IPT; ++j)
                if (b[j] != 0xFF) ++hist[b[j] * BK_THREADS + t];
        }
        __syncthreads();
        // exclusive scan of hist in bucket-major order: thread t owns entries [t*nb, (t+1)*nb)
        uint32_t sum = 0;
        for (int i = 0; i < nb; ++i) sum += hist[t * nb + i];
        uint32_t inc = sum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += y;
        }
        if (lane == 31) st.part[warp] = inc;
        __syncthreads();
        uint32_t wbase = 0;
        for (int w = 0; w < warp; ++w) wbase += (uint32_t)st.part[w];
        uint32_t run = wbase + inc - sum;
        for (int i = 0; i < nb; ++i) {
            const int f = t * nb + i;
            uint32_t c = hist[f];
            hist[f] = run;
            if ((f & (BK_THREADS - 1)) == 0) st.tstart[f / BK_THREADS] = (int32_t)run;  // entry (q, thread 0)
            run += c;
        }
        if (t == 0) st.tstart[nb] = (int32_t)(hi - t0 < BK_TILE ? hi - t0 : BK_TILE);
        __syncthreads();
        if (t < nb) st.delta[t] = st.cur[t] - st.tstart[t];
        // stage: this thread's elements go to its slots, in order (stable)
        uint64_t seen = 0;
#pragma unroll
        for (int j = 0; j < BK_IPT; ++j) {
            if (b[j] != 0xFF) {
                int p;
                if (SMALL) {
                    p = (int)hist[b[j] * BK_THREADS + t] + (int)((seen >> (8 * b[j])) & 0xFF);
                    seen += 1ull << (8 * b[j]);
                } else {
                    p = (int)hist[b[j] * BK_THREADS + t]++;
                }
                st.sk[pad_w<BK_IPT>(p)] = k[j];
                if (KV) st.sv[pad_w<BK_IPT>(p)] = v[j];
                st.sb[pad_b<BK_IPT>(p)] = b[j];
            }
        }
        __syncthreads();
        const int tn = st.tstart[nb];
        for (int p = t; p < tn; p += BK_THREADS) {
            const int64_t g = st.delta[st.sb[pad_b<BK_IPT>(p)]] + p;
            out_keys[g] = st.sk[pad_w<BK_IPT>(p)];
            if (KV) out_vals[g] = st.sv[pad_w<BK_IPT>(p)];
        }
        if (t < nb) st.cur[t] += st.tstart[t + 1] - st.tstart[t];
    }
}

}  // namespace pdq
