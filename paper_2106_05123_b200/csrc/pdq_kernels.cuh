// pdq_kernels.cuh — the seven kernels of the B200 pdqsort path.
//
//   K1 sample pivot          spawn(): 64 (256 for >= 2^20 keys) stratified samples, warp/CTA
//                            bitonic, median (generalises choose_pivot, driver.py:81-113)
//   K2 partition_right       part_tile(): TMA bulk tile -> classify -> per-warp counts -> one packed
//                            reservation atomic per tile for both sides -> warp-ballot compaction in
//                            shared memory -> TMA bulk stores (block_partition_right, partition.py:184-301)
//   K3 partition_left        part_tile() in I_LEFT mode (partition.py:128-181, driver.py:222-225)
//   K4 sortedness check      k_check(): adjacent-compare reduction; k_sort prologue reverses
//                            non-increasing input (partial_insertion_sort path, driver.py:244-250)
//   K5 bad-partition budget  finalize_part(): is_bad_partition (driver.py:116-124), budget,
//                            sample perturbation (break_patterns, driver.py:127-156); an exhausted
//                            budget switches the segment to radix exchange (heapsort's role)
//   K6 segment queue         k_sort(): persistent CTAs claim chunks of up to 32 tiles from a device ring
//                            of 64-bit task words, keep two TMA tile loads in flight, retire chunks
//                            with one bulk-store wait + fence + counter; the last chunk's CTA
//                            finalizes the segment and spawns its children (driver.py:198-260)
//   K7 base case             k_base_big (4-byte keys, leaves <= 24572) / k_base_wide (8-byte keys and
//                            key-value sorts, leaves <= 8188): bucket placement + in-bucket ranking in
//                            shared memory, tiny segments by one warp in registers (insertion_sort /
//                            unguarded_insertion_sort, small_sorts.py:16-73)
#pragma once

#include "pdq_device.cuh"
#include "pdq_networks.cuh"

namespace pdq {

// A ring task is a chunk of P.chunk consecutive tiles of one segment (one claim, one descriptor read,
// one retire).  The host picks the chunk from the sort size: the largest power of two <= 32 that still
// gives the top level ~2 tasks per CTA (32 tiles for 2^28 keys, 8 for 2^26).  A task word carries its
// first tile.
__device__ __forceinline__ uint32_t seg_ntasks(uint32_t N, uint32_t chunk) { return (N + chunk - 1) / chunk; }
__device__ __forceinline__ uint32_t task_end_tile(uint32_t first, uint32_t N, uint32_t chunk) {
    return min(first + chunk, N);
}
#ifndef PDQ_NST
#define PDQ_NST 1
#endif
constexpr int NST = PDQ_NST;
#ifndef PDQ_SLEEP_CAP
#define PDQ_SLEEP_CAP 256  // ns: the longest back-off of a CTA polling the ring for its next task
#endif
#ifndef PDQ_PAIR
#define PDQ_PAIR 1  // spawn both children of a partition with one ring reservation (spawn_pair)
#endif            // TMA stages: tile loads run up to NST tiles ahead of compute
// CTA barrier (named barrier 1, all THREADS threads)
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(THREADS) : "memory"); }
__device__ __forceinline__ int csync_or(int p) {
    int r;
    asm volatile(
        "{\n .reg .pred a, b;\n setp.ne.s32 a, %1, 0;\n bar.red.or.pred b, 1, %2, a;\n selp.s32 %0, 1, 0, b;\n}\n"
        : "=r"(r)
        : "r"(p), "n"(THREADS)
        : "memory");
    return r;
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t *bar, unsigned phase) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}

struct Shared {
    uint64_t bar[4];         // TMA stage barriers (Bufs::NSTAGE used)
    uint64_t task;           // current ring task word (0 = exit)
    Seg seg;                 // its descriptor
    uint64_t ntask;          // prefetched next task (0 = none / not yet published)
    Seg nseg;
    unsigned long long npos; // ring position claimed for the next task
    uint64_t lf[2];          // K7: descriptors of the current and the next leaf
    uint64_t lq[2];          // K7 (k_base_big): current and next leaf descriptors
    long long lc0;           // K7: cycle stamp of the current leaf (counters)
    int nstate;              // 0 none, 1 claimed (unpublished), 2 ready, 3 exit
    // load cursor (thread 0): tiles issued so far, and which task/tile is the next to load
    unsigned li;             // loads issued (stage li % NST)
    unsigned ci;             // tiles consumed by the compute side (mirrors the per-thread counter)
    int lslot;               // 0: the load cursor is in the current task, 1: in the next task
    uint32_t ltile;          // next tile index to load within that task
    int wl[WARPS], weq[WARPS];
    long long L, R, lOff, rOff, fL, fE;
    int aL, aR;  // kc positions of the current tile's left / right runs
    int rl_tiny, rl_seq;     // K5 finalizer: children sorted by warps / handled by the whole CTA
    unsigned long long push_pos;
    uint32_t new_sid;
    int last;
    uint64_t red_min[WARPS], red_max[WARPS];
    unsigned red_a[WARPS], red_b[WARPS];
    uint32_t scan[WARPS];
    // per-CTA counters, flushed once at exit
    unsigned long long s_part_right, s_part_left, s_bad, s_fallback, s_base, s_tiles, s_bytes;
    long long s_max_depth;
    unsigned long long s_cyc_wait, s_cyc_work, s_cyc_base, s_cyc_spawn;
    unsigned long long s_sch_retire, s_sch_claim, s_sch_fetch, s_sch_idle;
};

// Per-CTA shared state and the dynamic shared buffer are namespace-scope so every helper
// (inlined or not) addresses them as shared memory (LDS/STS, never generic LD/ST).
__shared__ Shared g_sh;
extern __shared__ __align__(128) unsigned char g_dsm[];

// programmatic dependent launch (launch_pdl in pdq_capi.cu): wait for the stream's previous kernel /
// let the next kernel of the stream be scheduled
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint32_t mix32(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return (uint32_t)x;
}

// Dynamic shared memory of the persistent sorter: NSTAGE TMA stages and the compaction buffer kc
// (keys, then payloads for KV).  Every pointer is computed arithmetically from the extern shared
// symbol so the compiler emits LDS/STS, never generic LD/ST.  kc holds a tile's left and right runs,
// each placed at the 16-byte phase of its global destination (so the run bodies leave by TMA bulk
// stores): KC_PAD elements of slack.  4-byte keys without payload use two stages (4 CTAs/SM), wider
// elements one (their occupancy is bounded by shared memory already).
// (Measured on 2^28 int32 and not kept: three stages with the tile compacted in place in its own
// stage, and a software pipeline issuing tile t+1's reservation before tile t is compacted.)
constexpr int KC_PAD = 16;
template <class U, bool KV>
struct Bufs {
    static constexpr int TLB = (sizeof(U) + (KV ? 4 : 0)) > 4 ? TILE / 2 : TILE;  // elements per tile
    static constexpr int NSTAGE = 2;
    static constexpr int SLOT = TLB + KC_PAD;
    static constexpr int KEY_BYTES = (NSTAGE + 1) * SLOT * (int)sizeof(U);
    static constexpr int VAL_BYTES = KV ? (NSTAGE + 1) * SLOT * 4 : 0;
    __device__ __forceinline__ static U *stage(int i) { return reinterpret_cast<U *>(g_dsm) + i * SLOT; }
    __device__ __forceinline__ static U *kc() { return reinterpret_cast<U *>(g_dsm) + NSTAGE * SLOT; }
    __device__ __forceinline__ static uint32_t *vstage(int i) {
        return reinterpret_cast<uint32_t *>(g_dsm + KEY_BYTES) + i * SLOT;
    }
    __device__ __forceinline__ static uint32_t *vc() {
        return reinterpret_cast<uint32_t *>(g_dsm + KEY_BYTES) + NSTAGE * SLOT;
    }
    // pivot samples alias kc (free whenever samples are taken)
    __device__ __forceinline__ static uint64_t *samp_k() { return reinterpret_cast<uint64_t *>(kc()); }
    __device__ __forceinline__ static uint32_t *samp_v() {
        return reinterpret_cast<uint32_t *>(reinterpret_cast<unsigned char *>(samp_k()) + SAMPLES * 8);
    }
    __host__ __device__ static constexpr int bytes() { return KEY_BYTES + VAL_BYTES; }
};

template <class U, bool FLOAT, bool KV>
struct Sorter {
    using O = Ord<U, FLOAT>;
    using B = Bufs<U, KV>;
    static constexpr int VEC = 16 / sizeof(U);
    static constexpr int AL = KV ? 4 : VEC;  // element alignment making both key and payload 16 B aligned
    static constexpr int ELEM_BYTES = sizeof(U) + (KV ? 4 : 0);
    // partition tile: 4096 elements of 4 bytes, 2048 of wider elements (16-24 KB per TMA stage, so the
    // persistent sorter keeps two stages and 3-4 CTAs per SM for every element type)
    static constexpr int TL = B::TLB, IT = TL / THREADS;
    using SU = typename std::conditional<sizeof(U) == 4, int32_t, int64_t>::type;
    
    // Tiles are relative to the segment: tile i covers [base + i TL, base + (i + 1) TL) from the segment's
    // 16-byte-aligned base, so a segment of m elements has ceil(m / TL) tiles plus at most one (from the
    // <= AL - 1 elements of lead-in) -- globally aligned tiles gave deep-level segments two partial tiles.
    __device__ __forceinline__ static int64_t tile_base(int64_t b, uint32_t tile) {
        return (b & ~(int64_t)(AL - 1)) + (int64_t)tile * TL;
    }
    __device__ __forceinline__ static uint32_t tiles_of(int64_t b, int64_t e) {
        return (uint32_t)((e - (b & ~(int64_t)(AL - 1)) + TL - 1) / TL);
    }

    static constexpr int KBITS = 8 * (int)sizeof(U);
    static constexpr int NBITS = KBITS + (KV ? 32 : 0);  // bits of the (ordered key, payload) composite
    __device__ __forceinline__ static bool tile_task(uint32_t type) {
        return type == T_PART || type == T_RHIST || type == T_RSCAT;
    }

    // Bounds known for a segment: every element e satisfies lb <= e (has_lb) and e < ub (has_ub),
    // in the (ordered key, payload) order.  lb is the reference's predecessor (driver.py:222).
    struct Bnd {
        uint64_t lb, ub;
        uint32_t lbv, ubv;
        bool has_lb, has_ub;
    };

    // strict order on raw key bits (+ payload): ints compare signed, floats by total order
    __device__ __forceinline__ static bool lt_raw(U a, uint32_t va, U b, uint32_t vb) {
        if (FLOAT) {
            const U oa = O::to(a), ob = O::to(b);
            if (KV) return oa < ob || (oa == ob && va < vb);
            return oa < ob;
        }
        if (KV) return (SU)a < (SU)b || (a == b && va < vb);
        return (SU)a < (SU)b;
    }

    // ---- vectorised contiguous store of `len` elements produced by get(i) -----------
    template <class T, class F>
    __device__ __forceinline__ static void store_run(T *g, int len, F get) {
        constexpr int V = 16 / sizeof(T);
        const int tid = threadIdx.x;
        const int mis = (int)(((uintptr_t)g / sizeof(T)) & (V - 1));
        int h = mis ? V - mis : 0;
        if (h > len) h = len;
        if (tid < h) g[tid] = get(tid);
        const int nb = (len - h) / V;
        uint4 *gv = reinterpret_cast<uint4 *>(g + h);
        for (int b = tid; b < nb; b += THREADS) {
            union {
                T t[V];
                uint4 u;
            } pk;
#pragma unroll
            for (int q = 0; q < V; ++q) pk.t[q] = get(h + b * V + q);
            gv[b] = pk.u;
        }
        const int t0 = h + nb * V;
        if (t0 + tid < len) g[t0 + tid] = get(t0 + tid);
    }

    // ---- CTA bitonic sort of a power-of-two array in shared memory (pivot samples) -----
    __device__ static void bitonic_samples(uint64_t *k, uint32_t *v, int P) {
        const int tid = threadIdx.x;
        for (int kk = 2; kk <= P; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
                const int lj = __ffs(j) - 1;
                const bool mirror = (j == (kk >> 1));
                for (int p = tid; p < (P >> 1); p += THREADS) {
                    const int i = ((p >> lj) << (lj + 1)) | (p & (j - 1));
                    const int q = mirror ? (i ^ (kk - 1)) : (i + j);
                    const uint64_t a = k[i], b = k[q];
                    const uint32_t va = KV ? v[i] : 0, vb = KV ? v[q] : 0;
                    if (pless<KV>(b, vb, a, va)) {
                        k[i] = b;
                        k[q] = a;
                        if (KV) {
                            v[i] = vb;
                            v[q] = va;
                        }
                    }
                }
                csync();
            }
        }
    }

    // Warp-level bitonic sort of 32*PL (key, payload) pairs held PL per lane (lane l owns
    // elements [PL*l, PL*l + PL)); no block barriers.
    template <int PL>
    __device__ __forceinline__ static void warp_bitonic(uint64_t (&x)[PL], uint32_t (&y)[PL]) {
        const int lane = threadIdx.x & 31;
        constexpr int S = 32 * PL;
#pragma unroll
        for (int k = 2; k <= S; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                const bool mirror = (j == (k >> 1));
                if (j < PL && (!mirror || k <= PL)) {
#pragma unroll
                    for (int i = 0; i < PL; ++i) {
                        const int p = mirror ? (i ^ (k - 1)) : (i ^ j);
                        if (p > i && pless<KV>(x[p], y[p], x[i], y[i])) {
                            const uint64_t t = x[i];
                            x[i] = x[p];
                            x[p] = t;
                            const uint32_t u = y[i];
                            y[i] = y[p];
                            y[p] = u;
                        }
                    }
                } else {
                    // partner lives in another lane: element e ^ j (or the mirror e ^ (k-1))
                    const int lmask = mirror ? ((k - 1) / PL) : (j / PL);
                    const bool lower = mirror ? ((lane & ((k >> 1) / PL)) == 0) : ((lane & (j / PL)) == 0);
                    uint64_t ox[PL];
                    uint32_t oy[PL];
#pragma unroll
                    for (int i = 0; i < PL; ++i) {
                        const int src = mirror ? (PL - 1 - i) : i;
                        ox[i] = __shfl_xor_sync(0xffffffffu, x[src], lmask);
                        oy[i] = KV ? __shfl_xor_sync(0xffffffffu, y[src], lmask) : 0u;
                    }
#pragma unroll
                    for (int i = 0; i < PL; ++i) {
                        const bool olt = pless<KV>(ox[i], oy[i], x[i], y[i]);
                        if (lower == olt) {
                            x[i] = ox[i];
                            y[i] = oy[i];
                        }
                    }
                }
            }
        }
    }

    __device__ static void finish_keys(const Params &P, unsigned long long cnt) {
        // single thread; callers fence their data writes first
        unsigned long long old = atomicAdd(&P.st->keys_final, cnt);
        if (old + cnt == (unsigned long long)P.n) {
            __threadfence();
            atomicExch(&P.st->done, 1u);
        }
    }

    __device__ static void fail(const Params &P, int code) {
        atomicCAS(&P.st->status, 0, code);
        __threadfence();
        atomicExch(&P.st->done, 1u);
    }

    __device__ __forceinline__ static int clz_u(U x) {
        if (sizeof(U) == 4) return __clz((uint32_t)x);
        return __clzll((long long)x);
    }

    // <= 64 keys: warp 0 sorts them in registers (2 per lane, bitonic over shuffles) straight into A.
    // Padding elements are the maximum (key, payload); a real element equal to the padding is the
    // same bits, so whichever lands in the first m slots is correct.
    __device__ static void tiny_sort(const Params &P, bool srcB, int64_t b, int m) {
        const int tid = threadIdx.x;
        if (tid < 32) {
            const U *src = (const U *)(srcB ? P.b_keys : P.a_keys);
            const uint32_t *srcv = srcB ? P.b_vals : P.a_vals;
            uint64_t x[2];
            uint32_t y[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int i = 2 * tid + q;
                x[q] = i < m ? (uint64_t)O::to(ldcg(src + b + i)) : ~0ull;
                y[q] = (KV && i < m) ? ldcg(srcv + b + i) : 0xFFFFFFFFu;
            }
            warp_bitonic<2>(x, y);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int i = 2 * tid + q;
                if (i < m) {
                    ((U *)P.a_keys)[b + i] = O::from((U)x[q]);
                    if (KV) P.a_vals[b + i] = y[q];
                }
            }
            __threadfence();
            __syncwarp();
            if (tid == 0) {
                g_sh.s_base++;
                g_sh.s_bytes += 2ull * ELEM_BYTES * m;
                finish_keys(P, (unsigned long long)m);
            }
        }
    }

    // T_PART: the segment's guided tasks (word = first tile); T_FILL: one task per tile
    __device__ static void push_tasks(const Params &P, uint32_t type, uint32_t sid, uint32_t ntiles) {
        Shared &sh = g_sh;
        const unsigned long long pos = sh.push_pos;
        const uint64_t mask = (1ull << P.log_q) - 1;
        const bool chunked = tile_task(type);
        const uint32_t nt = chunked ? seg_ntasks(ntiles, P.chunk) : ntiles;
        for (uint32_t t = threadIdx.x; t < nt; t += THREADS)
            *(volatile uint64_t *)&P.ring[(pos + t) & mask] =
                task_word(pos + t, P.log_q, type, sid, chunked ? t * P.chunk : t);
    }

    // ---- write [b, e) of A with the pivot (equal-key runs are bitwise identical under the
    // total order, so a fill is exact).  Returns true if it took the reusable descriptor. ---
    __device__ static bool fill_final(const Params &P, int64_t b, int64_t e, uint64_t piv,
                                      uint32_t pv, int reuse_sid) {
        Shared &sh = g_sh;
        const int tid = threadIdx.x;
        const int64_t m = e - b;
        if (m <= 0) return false;
        if (m <= INLINE_FILL) {
            const U raw = O::from((U)piv);
            store_run<U>((U *)P.a_keys + b, (int)m, [&](int) { return raw; });
            if (KV) store_run<uint32_t>(P.a_vals + b, (int)m, [&](int) { return pv; });
            __threadfence();
            csync();
            if (tid == 0) {
                sh.s_bytes += (unsigned long long)ELEM_BYTES * m;
                finish_keys(P, m);
            }
            csync();
            return false;
        }
        const uint32_t ntiles = tiles_of(b, e);
        if (tid == 0) {
            uint32_t sid = reuse_sid >= 0 ? (uint32_t)reuse_sid : atomicAdd(&P.st->seg_alloc, 1u);
            sh.new_sid = sid;
            if (sid >= P.seg_cap) {
                fail(P, -6);
            } else {
                Seg *s = &P.segs[sid];
                s->begin = b;
                s->end = e;
                s->pivot = piv;
                s->pivot_v = pv;
                s->ntiles = ntiles;
                s->info = 0;
                __threadfence();
                sh.push_pos = atomicAdd(&P.st->q_tail, (unsigned long long)ntiles);
            }
        }
        csync();
        if (sh.new_sid < P.seg_cap) push_tasks(P, T_FILL, sh.new_sid, ntiles);
        csync();
        return reuse_sid >= 0;
    }

    // ---- K5 radix exchange: split [b, e) on composite bit `bit` (0 = most significant) ---------------
    // Every element shares the prefix (pk, pv) above `bit`; the threshold prefix|bit sends elements
    // with a 0 bit left.  Returns true iff the reusable descriptor was consumed.
    __device__ static bool radix_split(const Params &P, int64_t b, int64_t e, bool srcB, int bit, uint64_t pk,
                                       uint32_t pv, int depth, int reuse_sid) {
        Shared &sh = g_sh;
        const int tid = threadIdx.x;
        const int64_t m = e - b;
        if (m <= 0) return false;
        if (bit >= NBITS || m == 1) {  // every bit decided: the elements are identical
            finish_constant(P, b, e, srcB);
            return false;
        }
        if (m <= P.base_size) {
            Bnd nb{};
            return spawn(P, b, e, srcB, nb, 1, depth, false, reuse_sid);  // leaf
        }
        uint64_t tk = pk;
        uint32_t tv = pv;
        if (bit < KBITS)
            tk |= (uint64_t)((U)1 << (KBITS - 1 - bit));
        else
            tv |= 1u << (31 - (bit - KBITS));
        const uint32_t ntiles = tiles_of(b, e);
        if (tid == 0) {
            const uint32_t sid = reuse_sid >= 0 ? (uint32_t)reuse_sid : atomicAdd(&P.st->seg_alloc, 1u);
            sh.new_sid = sid;
            if (sid >= P.seg_cap) {
                fail(P, -6);
            } else {
                Seg *s = &P.segs[sid];
                s->begin = b;
                s->end = e;
                s->pivot = (uint64_t)O::from((U)tk);  // raw bits: tiles compare raw keys
                s->pivot_v = tv;
                s->lb = pk;
                s->lb_v = pv;
                s->ntiles = ntiles;
                s->info = (srcB ? I_SRC_B : 0) | I_RADIX;
                s->rbit = (unsigned)bit;
                s->budget = 0;
                s->depth = depth;
                s->cnt_left = 0;
                s->cnt_right = 0;
                s->cnt_eq = 0;
                s->tiles_done = 0;
                __threadfence();
                sh.push_pos = atomicAdd(&P.st->q_tail, (unsigned long long)seg_ntasks(ntiles, P.chunk));
            }
        }
        csync();
        if (sh.new_sid < P.seg_cap) push_tasks(P, T_PART, sh.new_sid, ntiles);
        csync();
        if (depth > sh.s_max_depth && tid == 0) sh.s_max_depth = depth;
        return reuse_sid >= 0;
    }

    // ---- K1 + segment creation ------------------------------------------------------------
    // Creates the child segment [b, e) whose data lives in buffer srcB.  Small children are
    // finished right here (K7); big ones get a sampled pivot and their tiles are pushed.
    // Returns true iff the reusable descriptor `reuse_sid` was consumed.
    __device__ static bool spawn(const Params &P, int64_t b, int64_t e, bool srcB, const Bnd &bd, int budget,
                                 int depth, bool perturb, int reuse_sid) {
        const bool has_lb = bd.has_lb;
        const uint64_t lb = bd.lb;
        const uint32_t lbv = bd.lbv;
        Shared &sh = g_sh;
        const int tid = threadIdx.x;
        const int64_t m = e - b;
        if (m <= 0) return false;
        if (tid == 0 && depth > sh.s_max_depth) sh.s_max_depth = depth;
        if (P.debug_depth && depth >= P.debug_depth) {  // profiling knob: stop descending (unsorted!)
            if (tid == 0) finish_keys(P, (unsigned long long)m);
            csync();
            return false;
        }
        if (m == 1) {
            if (tid == 0) {
                if (srcB) {
                    ((U *)P.a_keys)[b] = ldcg((const U *)P.b_keys + b);
                    if (KV) P.a_vals[b] = ldcg(P.b_vals + b);
                    sh.s_bytes += 2 * ELEM_BYTES;
                    __threadfence();
                }
                finish_keys(P, 1);
            }
            csync();
            return false;
        }
        if (m <= P.base_size) {
            // K7 leaf: tiny ones are sorted right here by one warp, the rest are queued for the
            // base-case kernel that runs after this one
            if (m <= 64) {
                tiny_sort(P, srcB, b, (int)m);
            } else if (tid == 0) {
                const unsigned long long pos = atomicAdd(&P.st->leaf_count, 1ull);
                if (pos < P.leaf_cap)
                    P.leaves[pos] = (uint64_t)b << 16 | (uint64_t)(m - 1) << 1 | (srcB ? 1u : 0u);
                else
                    fail(P, -6);
                finish_keys(P, (unsigned long long)m);
            }
            csync();
            return false;
        }
        // K5: the bad-partition budget is spent (driver.py:209-213, heapsort in the reference): the
        // segment leaves quicksort for radix exchange, i.e. it is split on its most significant
        // undecided bit by the same partition kernel; the work is bounded by the key width.
        if (budget <= 0) {
            if (tid == 0) sh.s_fallback++;
            int bit = 0;
            uint64_t pk = 0;
            uint32_t pv = 0;
            if (bd.has_lb && bd.has_ub) {  // lb <= e < ub: the common prefix of lb and ub is fixed
                if (bd.lb != bd.ub) {
                    bit = clz_u((U)(bd.lb ^ bd.ub));
                    pk = bit ? (bd.lb & ~((uint64_t)(~(U)0) >> bit)) : 0;
                } else {
                    bit = KBITS + (KV ? (bd.lbv != bd.ubv ? __clz(bd.lbv ^ bd.ubv) : 32) : 0);
                    pk = bd.lb;
                    pv = (KV && bit > KBITS) ? (bit - KBITS >= 32 ? bd.lbv : (bd.lbv & ~(0xFFFFFFFFu >> (bit - KBITS)))) : 0u;
                }
            }
            return radix8_start(P, b, e, srcB, bit, pk, pv, depth, reuse_sid);
        }
        // K1: stratified samples (64, or SAMPLES for segments of 2^20+ keys) sorted by warp 0; perturbed
        // strata after a bad partition.  The median of the sorted sample is the pivot.
        const long long c0 = clock64();
        if (tid < 32) warp_sample(P, b, m, srcB, perturb, depth, 0);
        csync();
        const uint32_t ntiles = tiles_of(b, e);
        if (tid == 0) {
            const uint32_t sid = reuse_sid >= 0 ? (uint32_t)reuse_sid : atomicAdd(&P.st->seg_alloc, 1u);
            sh.new_sid = sid;
            if (sid >= P.seg_cap) {
                fail(P, -6);
            } else {
                write_part_seg(P, sid, b, e, srcB, bd, budget, depth, perturb, 0);
                __threadfence();
                sh.push_pos = atomicAdd(&P.st->q_tail, (unsigned long long)seg_ntasks(ntiles, P.chunk));
            }
        }
        csync();
        if (sh.new_sid < P.seg_cap) push_tasks(P, T_PART, sh.new_sid, ntiles);
        csync();
        if (tid == 0) sh.s_cyc_spawn += clock64() - c0;
        return reuse_sid >= 0;
    }

    // One warp: stratified samples of [b, b + m) (64, or SAMPLES = 256 for 2^20+ keys; perturbed strata
    // after a bad partition, break_patterns' role) sorted in registers by a warp bitonic network; the
    // median goes to sample slot `slot` (samp_k/samp_v[2 slot]), the smallest sample to samp_k[2 slot + 1].
    __device__ static void warp_sample(const Params &P, int64_t b, int64_t m, bool srcB, bool perturb, int depth,
                                       int slot) {
        Shared &sh = g_sh;
        const int lane = threadIdx.x & 31;
        const U *src = (const U *)(srcB ? P.b_keys : P.a_keys);
        const uint32_t *srcv = srcB ? P.b_vals : P.a_vals;
        const int ns = m >= (1 << 20) ? SAMPLES : 64;
        auto sample_at = [&](int i) -> int64_t {
            if (perturb)
                return ((int64_t)i * m +
                        (int64_t)(mix32((uint64_t)b * 0x9E3779B97F4A7C15ull ^ (uint64_t)(depth * 977 + i)) %
                                  (uint64_t)m)) /
                       ns;
            return ((int64_t)(2 * i + 1) * m) / (2 * ns);
        };
        auto run = [&](auto pl_c) {
            constexpr int PL = decltype(pl_c)::value;
            uint64_t x[PL];
            uint32_t y[PL];
#pragma unroll
            for (int q = 0; q < PL; ++q) {
                const int64_t off = sample_at(PL * lane + q);
                x[q] = (uint64_t)O::to(ldcg(src + b + off));
                y[q] = KV ? ldcg(srcv + b + off) : 0u;
            }
            warp_bitonic<PL>(x, y);
            if (lane == 16) {  // element 16 PL (the median) = lane 16, register 0
                B::samp_k()[2 * slot] = x[0];
                B::samp_v()[2 * slot] = y[0];
            }
            if (lane == 0) B::samp_k()[2 * slot + 1] = x[0];  // the smallest sample
        };
        if (ns == 64)
            run(std::integral_constant<int, 2>());
        else
            run(std::integral_constant<int, SAMPLES / 32>());
        if (lane == 0) atomicAdd(&sh.s_bytes, (unsigned long long)ns * ELEM_BYTES);
    }

    // thread 0: the descriptor of partition segment [b, e) (buffer srcB) with the pivot of sample slot
    // `slot`: partition_left when the predecessor equals the pivot (driver.py:222), equal counting when
    // the sample's low end repeats the pivot
    __device__ static void write_part_seg(const Params &P, uint32_t sid, int64_t b, int64_t e, bool srcB,
                                          const Bnd &bd, int budget, int depth, bool perturb, int slot) {
        const uint64_t piv = B::samp_k()[2 * slot], lo_sample = B::samp_k()[2 * slot + 1];
        const uint32_t pv = B::samp_v()[2 * slot];
        const bool dup_heavy = lo_sample == piv;  // the low end of the sample repeats the pivot
        const bool left = P.use_left && bd.has_lb && !pless<KV>(bd.lb, bd.lbv, piv, pv);
        Seg *s = &P.segs[sid];
        s->begin = b;
        s->end = e;
        s->pivot = (uint64_t)O::from((U)piv);  // raw bits: tiles compare raw keys
        s->pivot_v = pv;
        s->lb = bd.lb;
        s->lb_v = bd.lbv;
        s->ntiles = tiles_of(b, e);
        s->info = (srcB ? I_SRC_B : 0) | (left ? I_LEFT : 0) | (bd.has_lb ? I_HAS_LB : 0) |
                  (bd.has_ub ? I_HAS_UB : 0) | (perturb ? I_PERTURB : 0) | (dup_heavy ? I_COUNT_EQ : 0);
        s->budget = budget > 0 ? budget : 0;
        s->depth = depth;
        s->ub = bd.ub;
        s->ub_v = bd.ubv;
        s->cnt_left = 0;
        s->cnt_right = 0;
        s->cnt_eq = 0;
        s->tiles_done = 0;
    }

    // Both children of a partition are big partition segments: warps 0 and 1 sample them at once and
    // one ring reservation publishes both (halves the finalize -> first-tile latency of a tree level).
    // Returns false (nothing done) when the pair does not qualify; spawn() then handles each child.
    __device__ static bool spawn_pair(const Params &P, int64_t b, int64_t mid, int64_t e, bool srcB,
                                      const Bnd &lbd, const Bnd &rbd, int budget, int depth, bool perturb,
                                      int reuse_sid) {
        Shared &sh = g_sh;
        const int tid = threadIdx.x, warp = tid >> 5;
        if (!PDQ_PAIR || budget <= 0 || P.debug_depth || mid - b <= P.base_size || e - mid <= P.base_size ||
            reuse_sid < 0)
            return false;
        const long long c0 = clock64();
        if (warp < 2) warp_sample(P, warp ? mid : b, warp ? e - mid : mid - b, srcB, perturb, depth, warp);
        csync();
        const uint32_t ntL = tiles_of(b, mid), ntR = tiles_of(mid, e);
        const uint32_t nkL = seg_ntasks(ntL, P.chunk), nkR = seg_ntasks(ntR, P.chunk);
        if (tid == 0) {
            const uint32_t sidL = (uint32_t)reuse_sid, sidR = atomicAdd(&P.st->seg_alloc, 1u);
            sh.new_sid = sidR;
            if (sidR >= P.seg_cap) {
                fail(P, -6);
            } else {
                write_part_seg(P, sidL, b, mid, srcB, lbd, budget, depth, perturb, 0);
                write_part_seg(P, sidR, mid, e, srcB, rbd, budget, depth, perturb, 1);
                __threadfence();
                sh.push_pos = atomicAdd(&P.st->q_tail, (unsigned long long)(nkL + nkR));
            }
            if (depth > sh.s_max_depth) sh.s_max_depth = depth;
        }
        csync();
        if (sh.new_sid < P.seg_cap) {
            const unsigned long long pos = sh.push_pos;
            const uint64_t mask = (1ull << P.log_q) - 1;
            for (uint32_t t = tid; t < nkL + nkR; t += THREADS) {
                const bool r = t >= nkL;
                const uint32_t k = r ? t - nkL : t;
                *(volatile uint64_t *)&P.ring[(pos + t) & mask] =
                    task_word(pos + t, P.log_q, T_PART, r ? sh.new_sid : (uint32_t)reuse_sid, k * P.chunk);
            }
        }
        csync();
        if (tid == 0) sh.s_cyc_spawn += clock64() - c0;
        return true;
    }

    // ---- K5 + K6: the last tile of a segment decides its children ----------------------------
    // `sg` is the parent's descriptor (copied when the task was claimed; immutable while it lived).
    __device__ __noinline__ static void finalize_part(const Params &P, const Seg &sg,
                                                      uint32_t sid) {
        Shared &sh = g_sh;
        const int tid = threadIdx.x;
        if (tid == 0) {
            Seg *gs = &P.segs[sid];
            const unsigned long long c = __ldcg(&gs->cnt_left);
            sh.fL = sg.end - sg.begin < (1ll << 32) ? (long long)(c & 0xFFFFFFFFull) : (long long)c;
            sh.fE = (long long)__ldcg(&gs->cnt_eq);
        }
        csync();
        const int64_t b = sg.begin, e = sg.end, m = e - b, L = sh.fL;
        PDQ_CHECK(L >= 0 && L <= m, "finalized left count");
        const bool srcB = sg.info & I_SRC_B, dstB = !srcB;
        const uint64_t piv_ord = (uint64_t)O::to((U)sg.pivot);
        if (sg.info & I_RADIX) {
            // K5 radix exchange: both sides continue on the next bit
            if (tid == 0) sh.s_part_right++;
            const int bit = (int)sg.rbit;
            bool used = radix_split(P, b, b + L, dstB, bit + 1, sg.lb, sg.lb_v, sg.depth + 1, (int)sid);
            radix_split(P, b + L, e, dstB, bit + 1, piv_ord, sg.pivot_v, sg.depth + 1, used ? -1 : (int)sid);
            return;
        }
        Bnd parent{};
        parent.has_lb = sg.info & I_HAS_LB;
        parent.lb = sg.lb;
        parent.lbv = sg.lb_v;
        parent.has_ub = sg.info & I_HAS_UB;
        parent.ub = sg.ub;
        parent.ubv = sg.ub_v;
        if (!(sg.info & I_LEFT)) {
            if (tid == 0) sh.s_part_right++;
            if (sh.fE == m) {
                // Every key is bitwise equal to the pivot: whichever buffer A holds (the untouched
                // source, or this pass's output) already is the final, constant run.
                if (tid == 0) finish_keys(P, (unsigned long long)m);
                csync();
                return;
            }
            const int64_t R = m - L;
            const int64_t thr = m >> P.bad_shift;  // driver.py:123
            const bool bad = L < thr || R < thr;
            if (tid == 0 && bad) sh.s_bad++;
            const int nb = sg.budget - (bad ? 1 : 0);
            const bool perturb = bad && P.use_break;
            Bnd lbd = parent, rbd = parent;  // left: [lb, pivot), right: [pivot, ub)
            lbd.has_ub = true;
            lbd.ub = piv_ord;
            lbd.ubv = sg.pivot_v;
            rbd.has_lb = true;
            rbd.lb = piv_ord;
            rbd.lbv = sg.pivot_v;
            if (!spawn_pair(P, b, b + L, e, dstB, lbd, rbd, nb, sg.depth + 1, perturb, (int)sid)) {
                bool used = spawn(P, b, b + L, dstB, lbd, nb, sg.depth + 1, perturb, (int)sid);
                spawn(P, b + L, e, dstB, rbd, nb, sg.depth + 1, perturb, used ? -1 : (int)sid);
            }
        } else {
            if (tid == 0) sh.s_part_left++;
            bool used = false;
            if (srcB) {
                // lefts were written straight into A during the pass
                if (tid == 0 && L) finish_keys(P, (unsigned long long)L);
                csync();
            } else {
                used = fill_final(P, b, b + L, piv_ord, sg.pivot_v, (int)sid);
            }
            Bnd rbd = parent;  // (pivot, ub): the pivot is a valid lower bound
            rbd.has_lb = true;
            rbd.lb = piv_ord;
            rbd.lbv = sg.pivot_v;
            spawn(P, b + L, e, dstB, rbd, sg.budget, sg.depth + 1, false, used ? -1 : (int)sid);
        }
    }


    // Every key of [b, e) (in buffer srcB) is bitwise identical: make A hold it.
    __device__ static void finish_constant(const Params &P, int64_t b, int64_t e, bool srcB) {
        if (srcB) {
            const U k0 = ldcg((const U *)P.b_keys + b);
            const uint32_t v0 = KV ? ldcg(P.b_vals + b) : 0u;
            fill_final(P, b, e, (uint64_t)O::to(k0), v0, -1);
        } else {
            if (threadIdx.x == 0) finish_keys(P, (unsigned long long)(e - b));
            csync();
        }
    }

    // ---- K5: 8-bit digit passes (the role of heapsort, driver.py:209-213; small_sorts.py:134-154) ------
    // A segment whose bad-partition budget is spent leaves quicksort for MSD radix passes over the bits of
    // its (ordered key, payload) composite below the prefix its bounds already fix.  One pass = a
    // histogram over the segment's tiles (T_RHIST: w bytes read per element, or w + 4 once the digit
    // reaches the payload) into the segment's slot of 256 counters, an exclusive scan into scatter cursors
    // (the finalizer), and a scatter over the same tiles (T_RSCAT: 2 (w + p) bytes per element): each
    // tile is reordered by digit in its own stage, reserves one run per digit with one atomic on that
    // digit's cursor, and writes its runs to the other buffer.  The 256 children then become leaves or
    // radix segments on the next 8 bits -- the work is bounded by the key width, never quadratic.  A pass
    // whose histogram finds a single digit skips the scatter.  (Bits are MSB-first composite positions.)
    // Digit width of a pass over m elements: 8 bits, or fewer when 256 runs would be much smaller than a
    // leaf (a uniform segment then splits into runs of about half the base-case size instead of many tiny
    // leaves); never past the composite's last bit.  Stored in the segment (Seg::pivot_v).
    __device__ __forceinline__ static int rwidth(const Params &P, int64_t m, int rbit) {
        const int64_t target = P.base_size / 2 > 64 ? P.base_size / 2 : 64;
        int nd = 1;
        while (nd < 8 && (m >> nd) > target) ++nd;
        return nd < NBITS - rbit ? nd : NBITS - rbit;
    }
    __device__ __forceinline__ static int rdigits(const Seg &sg) { return (int)sg.pivot_v; }
    __device__ __forceinline__ static bool hist_keys_only(uint64_t task, const Seg &sg) {
        return ((uint32_t)(task >> 45) & 7u) == T_RHIST && (int)sg.rbit + rdigits(sg) <= KBITS;
    }
    __device__ __forceinline__ static uint32_t digit_of(U k, uint32_t v, int rbit, int nd) {
        const uint32_t mask = (1u << nd) - 1u;
        if (rbit + nd <= KBITS) return (uint32_t)((uint64_t)k >> (KBITS - rbit - nd)) & mask;
        if (rbit >= KBITS) return (v >> (32 - (rbit - KBITS) - nd)) & mask;
        const int kb = KBITS - rbit, vb = nd - kb;
        return ((((uint32_t)(uint64_t)k) & ((1u << kb) - 1u)) << vb) | (v >> (32 - vb));
    }
    // per-tile digit extractor: MODE 0 = the digit lies in the key, 1 = in the payload, 2 = straddles
    struct Dig {
        int mode, ks, vs;
        uint32_t mask;
        __device__ __forceinline__ Dig(int rbit, int nd) {
            mask = (1u << nd) - 1u;
            mode = rbit + nd <= KBITS ? 0 : (rbit >= KBITS ? 1 : 2);
            ks = mode == 0 ? KBITS - rbit - nd : nd - (KBITS - rbit);  // mode 2: bits taken from the payload
            vs = mode == 1 ? 32 - (rbit - KBITS) - nd : 32 - ks;
        }
        template <int MODE>
        __device__ __forceinline__ uint32_t get(U k, uint32_t v) const {
            if (MODE == 0) return (uint32_t)((uint64_t)k >> ks) & mask;
            if (MODE == 1) return (v >> vs) & mask;
            return (((uint32_t)(uint64_t)k << ks) | (v >> vs)) & mask;
        }
    };
    // the prefix (pk, pv) with digit dv at composite bits [rbit, rbit + nd)
    __device__ __forceinline__ static void put_digit(uint64_t &pk, uint32_t &pv, int rbit, int nd, uint32_t dv) {
        if (rbit + nd <= KBITS) {
            pk |= (uint64_t)dv << (KBITS - rbit - nd);
        } else if (rbit >= KBITS) {
            pv |= dv << (32 - (rbit - KBITS) - nd);
        } else {
            const int kb = KBITS - rbit, vb = nd - kb;
            pk |= (uint64_t)(dv >> vb);
            pv |= (dv & ((1u << vb) - 1u)) << (32 - vb);
        }
    }
    // warp-aggregated shared-memory counter increment: one atomic when every valid lane has the same digit
    __device__ __forceinline__ static uint32_t count_digit(uint32_t *cnt, bool valid, uint32_t d) {
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        if (!vm) return 0;
        const int lead = __ffs(vm) - 1;
        const uint32_t d0 = __shfl_sync(0xffffffffu, d, lead);
        if (__all_sync(0xffffffffu, !valid || d == d0)) {
            uint32_t base = 0;
            if ((int)(threadIdx.x & 31) == lead) base = atomicAdd(&cnt[d0], (uint32_t)__popc(vm));
            base = __shfl_sync(0xffffffffu, base, lead);
            return base + (uint32_t)__popc(vm & lanemask_lt());
        }
        return valid ? atomicAdd(&cnt[d], 1u) : 0u;
    }

    // T_RHIST tile: digit histogram of the tile, added to the segment's slot (kc holds the counters)
    __device__ static void hist_tile(const Params &P, uint32_t tile, unsigned &ci) {
        Shared &sh = g_sh;
        const int tid = threadIdx.x;
        const Seg &sg = sh.seg;
        const int64_t b = sg.begin, e = sg.end;
        const int64_t tbase = tile_base(b, tile);
        const int lo_i = (int)((b > tbase ? b : tbase) - tbase), hi_i = (int)((e < tbase + TL ? e : tbase + TL) - tbase);
        const int st = (int)(ci % B::NSTAGE);
        const U *sk = B::stage(st);
        const uint32_t *sv = KV ? B::vstage(st) : nullptr;
        const int rbit = (int)sg.rbit, nd = rdigits(sg);
        uint32_t *cnt = reinterpret_cast<uint32_t *>(B::kc());
        cnt[tid] = 0;  // THREADS == RDIG
        mbar_wait(&sh.bar[st], (ci / B::NSTAGE) & 1u);
        ++ci;
        csync();
        const Dig dg(rbit, nd);
        auto hist = [&](auto mode_c) {
            constexpr int MODE = decltype(mode_c)::value;
            if (lo_i == 0 && hi_i == TL) {  // a whole tile: every lane holds an element in every round
#pragma unroll 4
                for (int i = tid; i < TL; i += THREADS) {
                    const uint32_t d = dg.template get<MODE>(O::to(sk[i]), (KV && MODE != 0) ? sv[i] : 0u);
                    const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
                    if (__all_sync(0xffffffffu, d == d0)) {
                        if ((tid & 31) == 0) atomicAdd(&cnt[d0], 32u);
                    } else {
                        atomicAdd(&cnt[d], 1u);
                    }
                }
            } else {
                for (int i0 = lo_i; i0 < hi_i; i0 += THREADS) {
                    const int i = i0 + tid;
                    const bool valid = i < hi_i;
                    uint32_t d = 0;
                    if (valid) d = dg.template get<MODE>(O::to(sk[i]), (KV && MODE != 0) ? sv[i] : 0u);
                    count_digit(cnt, valid, d);
                }
            }
        };
        if (dg.mode == 0)
            hist(std::integral_constant<int, 0>());
        else if (dg.mode == 1)
            hist(std::integral_constant<int, 1>());
        else
            hist(std::integral_constant<int, 2>());
        csync();  // histogram complete, stage consumed
        if (tid == 0) {
            sh.ci = ci;
            pump_loads(P);
            sh.s_tiles++;
            sh.s_bytes += (unsigned long long)(hi_i - lo_i) * (rbit + nd <= KBITS ? sizeof(U) : ELEM_BYTES);
        }
        const uint32_t c = cnt[tid];
        if (c) atomicAdd(&P.rslots[(size_t)sg.rslot * RDIG + tid], (unsigned long long)c);
        csync();  // kc is free again
    }

    // T_RSCAT tile: reorder the tile by digit in its own stage, reserve one run per digit, write the runs
    __device__ static void rscat_tile(const Params &P, uint32_t tile, unsigned &ci) {
        Shared &sh = g_sh;
        const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
        const Seg &sg = sh.seg;
        const int64_t b = sg.begin, e = sg.end;
        const int64_t tbase = tile_base(b, tile);
        const int lo_i = (int)((b > tbase ? b : tbase) - tbase), hi_i = (int)((e < tbase + TL ? e : tbase + TL) - tbase);
        const int st = (int)(ci % B::NSTAGE);
        U *sk = B::stage(st);
        uint32_t *sv = KV ? B::vstage(st) : nullptr;
        const int rbit = (int)sg.rbit, nd = rdigits(sg);
        const bool srcB = sg.info & I_SRC_B;
        U *dst = (U *)(srcB ? P.a_keys : P.b_keys);
        uint32_t *dstv = srcB ? P.a_vals : P.b_vals;
        uint32_t *cnt = reinterpret_cast<uint32_t *>(B::kc());
        uint32_t *lst = cnt + RDIG;
        long long *gd = reinterpret_cast<long long *>(cnt + 2 * RDIG);
        uint32_t *wsum = cnt + 4 * RDIG;
        cnt[tid] = 0;
        mbar_wait(&sh.bar[st], (ci / B::NSTAGE) & 1u);
        ++ci;
        csync();
        U kx[IT];
        uint32_t vx[IT], pk[IT];
        const Dig dg(rbit, nd);
        auto slots = [&](auto mode_c) {
            constexpr int MODE = decltype(mode_c)::value;
            if (lo_i == 0 && hi_i == TL) {  // a whole tile: one atomic per warp when its 32 digits agree
#pragma unroll
                for (int r = 0; r < IT; ++r) {
                    const int i = r * THREADS + tid;
                    kx[r] = sk[i];
                    vx[r] = KV ? sv[i] : 0u;
                    const uint32_t d = dg.template get<MODE>(O::to(kx[r]), vx[r]);
                    const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
                    uint32_t sl;
                    if (__all_sync(0xffffffffu, d == d0)) {
                        uint32_t base = 0;
                        if ((tid & 31) == 0) base = atomicAdd(&cnt[d0], 32u);
                        sl = __shfl_sync(0xffffffffu, base, 0) + (tid & 31);
                    } else {
                        sl = atomicAdd(&cnt[d], 1u);
                    }
                    pk[r] = d << 16 | sl;
                }
            } else {
#pragma unroll
                for (int r = 0; r < IT; ++r) {
                    const int i = r * THREADS + tid;
                    const bool valid = i >= lo_i && i < hi_i;
                    kx[r] = valid ? sk[i] : (U)0;
                    vx[r] = (KV && valid) ? sv[i] : 0u;
                    const uint32_t d = valid ? dg.template get<MODE>(O::to(kx[r]), vx[r]) : 0u;
                    const uint32_t sl = count_digit(cnt, valid, d);
                    pk[r] = valid ? (d << 16 | sl) : 0xFFFFFFFFu;
                }
            }
        };
        if (dg.mode == 0)
            slots(std::integral_constant<int, 0>());
        else if (dg.mode == 1)
            slots(std::integral_constant<int, 1>());
        else
            slots(std::integral_constant<int, 2>());
        csync();
        {  // digit t = thread t: exclusive scan of the tile's counts, then one cursor atomic per digit
            const uint32_t c = cnt[tid];
            uint32_t inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) wsum[warp] = inc;
            csync();
            uint32_t wpre = 0;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) wpre += (w < warp) ? wsum[w] : 0u;
            const uint32_t ex = wpre + inc - c;
            lst[tid] = ex;
            long long g = 0;
            if (c) g = (long long)atomicAdd(&P.rslots[(size_t)sg.rslot * RDIG + tid], (unsigned long long)c);
            gd[tid] = g - (long long)ex;
        }
        csync();  // every input element is in registers: the stage is rewritten in digit order
#pragma unroll
        for (int r = 0; r < IT; ++r) {
            if (pk[r] != 0xFFFFFFFFu) {
                const uint32_t pos = lst[pk[r] >> 16] + (pk[r] & 0xFFFFu);
                sk[pos] = kx[r];
                if (KV) sv[pos] = vx[r];
            }
        }
        csync();
        const int nv = hi_i - lo_i;
        auto out = [&](auto mode_c) {
            constexpr int MODE = decltype(mode_c)::value;
#pragma unroll 4
            for (int p = tid; p < nv; p += THREADS) {  // consecutive threads write consecutive slots of a run
                const U k = sk[p];
                const uint32_t v = KV ? sv[p] : 0u;
                const long long g = gd[dg.template get<MODE>(O::to(k), v)] + p;
                dst[g] = k;
                if (KV) dstv[g] = v;
            }
        };
        if (dg.mode == 0)
            out(std::integral_constant<int, 0>());
        else if (dg.mode == 1)
            out(std::integral_constant<int, 1>());
        else
            out(std::integral_constant<int, 2>());
        csync();  // stage consumed, kc free
        if (tid == 0) {
            sh.ci = ci;
            pump_loads(P);
            sh.s_tiles++;
            sh.s_bytes += 2ull * ELEM_BYTES * (unsigned long long)nv;
        }
    }

    // one warp sorts [b, b + m), m <= 64, from buffer srcB into A (tiny_sort for any warp)
    __device__ static void tiny_sort_warp(const Params &P, bool srcB, int64_t b, int m) {
        Shared &sh = g_sh;
        const int lane = threadIdx.x & 31;
        const U *src = (const U *)(srcB ? P.b_keys : P.a_keys);
        const uint32_t *srcv = srcB ? P.b_vals : P.a_vals;
        uint64_t x[2];
        uint32_t y[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int i = 2 * lane + q;
            x[q] = i < m ? (uint64_t)O::to(ldcg(src + b + i)) : ~0ull;
            y[q] = (KV && i < m) ? ldcg(srcv + b + i) : 0xFFFFFFFFu;
        }
        warp_bitonic<2>(x, y);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int i = 2 * lane + q;
            if (i < m) {
                ((U *)P.a_keys)[b + i] = O::from((U)x[q]);
                if (KV) P.a_vals[b + i] = y[q];
            }
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) {
            atomicAdd(&sh.s_base, 1ull);
            atomicAdd(&sh.s_bytes, 2ull * ELEM_BYTES * m);
            finish_keys(P, (unsigned long long)m);
        }
    }

    // Start a digit-pass segment [b, e) in buffer srcB on composite bit `bit` with known prefix (pk, pv).
    // Falls back to one-bit radix exchange when the radix slots are exhausted.  Returns true iff the
    // reusable descriptor was consumed.
    __device__ static bool radix8_start(const Params &P, int64_t b, int64_t e, bool srcB, int bit, uint64_t pk,
                                        uint32_t pv, int depth, int reuse_sid) {
        Shared &sh = g_sh;
        const int tid = threadIdx.x;
        const int64_t m = e - b;
        if (m <= 0) return false;
        if (bit >= NBITS || m == 1) {
            finish_constant(P, b, e, srcB);
            return false;
        }
        if (m <= P.base_size) {
            Bnd nb{};
            return spawn(P, b, e, srcB, nb, 1, depth, false, reuse_sid);  // leaf
        }
        if (tid == 0) sh.new_sid = atomicAdd(&P.st->rslot_alloc, 1u);
        csync();
        const uint32_t slot = sh.new_sid;
        csync();
        if (slot >= P.rslot_cap) return radix_split(P, b, e, srcB, bit, pk, pv, depth, reuse_sid);
        P.rslots[(size_t)slot * RDIG + tid] = 0ull;  // THREADS == RDIG
        __threadfence();
        csync();
        const uint32_t ntiles = tiles_of(b, e);
        if (tid == 0) {
            const uint32_t sid = reuse_sid >= 0 ? (uint32_t)reuse_sid : atomicAdd(&P.st->seg_alloc, 1u);
            sh.new_sid = sid;
            if (sid >= P.seg_cap) {
                fail(P, -6);
            } else {
                Seg *s = &P.segs[sid];
                s->begin = b;
                s->end = e;
                s->pivot = 0;
                s->pivot_v = (uint32_t)rwidth(P, m, bit);  // digit width of the pass
                s->lb = pk;
                s->lb_v = pv;
                s->ntiles = ntiles;
                s->info = (srcB ? I_SRC_B : 0) | I_RADIX8;
                s->rbit = (unsigned)bit;
                s->rslot = slot;
                s->budget = 0;
                s->depth = depth;
                s->cnt_left = 0;
                s->cnt_right = 0;
                s->cnt_eq = 0;
                s->tiles_done = 0;
                __threadfence();
                sh.push_pos = atomicAdd(&P.st->q_tail, (unsigned long long)seg_ntasks(ntiles, P.chunk));
            }
            if (depth > sh.s_max_depth) sh.s_max_depth = depth;
        }
        csync();
        if (sh.new_sid < P.seg_cap) push_tasks(P, T_RHIST, sh.new_sid, ntiles);
        csync();
        return reuse_sid >= 0;
    }

    // 64-bit exclusive scan of one value per thread (CTA-wide; contains barriers)
    __device__ __forceinline__ static unsigned long long block_excl_u64(unsigned long long v) {
        Shared &sh = g_sh;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        unsigned long long inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) sh.red_max[warp] = inc;
        csync();
        unsigned long long pre = 0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) pre += (w < warp) ? sh.red_max[w] : 0ull;
        csync();
        return pre + inc - v;
    }

    // the histogram of a digit pass is complete: turn it into scatter cursors (or skip a one-digit pass)
    __device__ __noinline__ static void radix_hist_done(const Params &P, const Seg &sg, uint32_t sid) {
        Shared &sh = g_sh;
        const int tid = threadIdx.x;
        unsigned long long *cs = P.rslots + (size_t)sg.rslot * RDIG;
        const int64_t b = sg.begin, e = sg.end, m = e - b;
        const bool srcB = sg.info & I_SRC_B;
        const int rbit = (int)sg.rbit, nd = rdigits(sg);
        const unsigned long long c = __ldcg(&cs[tid]);
        const unsigned long long ex = block_excl_u64(c);
        if (c == (unsigned long long)m) sh.aL = tid;  // the one digit every element has
        if (tid == 0) sh.s_part_right++;
        if (csync_or(c == (unsigned long long)m)) {
            uint64_t pk = sg.lb;
            uint32_t pv = sg.lb_v;
            put_digit(pk, pv, rbit, nd, (uint32_t)sh.aL);
            if (rbit + nd >= NBITS) {
                finish_constant(P, b, e, srcB);
                return;
            }
            cs[tid] = 0ull;  // the next digit's histogram, same segment, same buffer
            __threadfence();
            csync();
            if (tid == 0) {
                Seg *gs = &P.segs[sid];
                gs->rbit = (unsigned)(rbit + nd);
                gs->pivot_v = (uint32_t)rwidth(P, m, rbit + nd);
                gs->lb = pk;
                gs->lb_v = pv;
                gs->tiles_done = 0;
                __threadfence();
                sh.push_pos = atomicAdd(&P.st->q_tail, (unsigned long long)seg_ntasks(sg.ntiles, P.chunk));
            }
            csync();
            push_tasks(P, T_RHIST, sid, sg.ntiles);
            csync();
            return;
        }
        cs[tid] = (unsigned long long)b + ex;  // scatter cursor of digit tid
        __threadfence();
        csync();
        if (tid == 0) {
            P.segs[sid].tiles_done = 0;
            __threadfence();
            sh.push_pos = atomicAdd(&P.st->q_tail, (unsigned long long)seg_ntasks(sg.ntiles, P.chunk));
        }
        csync();
        push_tasks(P, T_RSCAT, sid, sg.ntiles);
        csync();
    }

    // the scatter of a digit pass is complete: the 256 digit runs are the children (thread t: digit t)
    __device__ __noinline__ static void radix_scat_done(const Params &P, const Seg &sg, uint32_t sid) {
        Shared &sh = g_sh;
        const int tid = threadIdx.x, warp = tid >> 5;
        unsigned long long *cs = P.rslots + (size_t)sg.rslot * RDIG;
        unsigned long long *E = reinterpret_cast<unsigned long long *>(B::kc());  // run ends
        uint8_t *tiny = reinterpret_cast<uint8_t *>(E + RDIG), *seq = tiny + RDIG;
        E[tid] = __ldcg(&cs[tid]);
        if (tid == 0) {
            sh.rl_tiny = 0;
            sh.rl_seq = 0;
        }
        csync();
        const int rbit = (int)sg.rbit, nd = rdigits(sg), nrbit = rbit + nd;
        const bool dstB = !(sg.info & I_SRC_B);
        const int64_t cb = tid ? (int64_t)E[tid - 1] : sg.begin, ce = (int64_t)E[tid], mc = ce - cb;
        uint64_t pk = sg.lb;
        uint32_t pv = sg.lb_v;
        put_digit(pk, pv, rbit, nd, (uint32_t)tid);
        if (mc == 1) {
            if (dstB) {
                ((U *)P.a_keys)[cb] = ldcg((const U *)P.b_keys + cb);
                if (KV) P.a_vals[cb] = ldcg(P.b_vals + cb);
                atomicAdd(&sh.s_bytes, 2ull * ELEM_BYTES);
                __threadfence();
            }
            finish_keys(P, 1ull);
        } else if (mc > 1 && nrbit >= NBITS && !dstB) {
            finish_keys(P, (unsigned long long)mc);  // every bit decided: a constant run, already in A
        } else if (mc > 1 && mc <= 64 && nrbit < NBITS) {
            tiny[atomicAdd(&sh.rl_tiny, 1)] = (uint8_t)tid;
        } else if (mc > 1 && mc <= P.base_size) {
            // a leaf for the base-case kernel (a constant run in B is copied by it as well)
            const unsigned long long pos = atomicAdd(&P.st->leaf_count, 1ull);
            if (pos < P.leaf_cap)
                P.leaves[pos] = (uint64_t)cb << 16 | (uint64_t)(mc - 1) << 1 | (dstB ? 1u : 0u);
            else
                fail(P, -6);
            finish_keys(P, (unsigned long long)mc);
        } else if (mc > 1 && nrbit < NBITS) {
            // a radix segment on the next digit
            const uint32_t slot = atomicAdd(&P.st->rslot_alloc, 1u);
            const uint32_t csid = slot < P.rslot_cap ? atomicAdd(&P.st->seg_alloc, 1u) : 0xFFFFFFFFu;
            if (slot >= P.rslot_cap) {
                seq[atomicAdd(&sh.rl_seq, 1)] = (uint8_t)tid;
            } else if (csid >= P.seg_cap) {
                fail(P, -6);
            } else {
                unsigned long long *ccs = P.rslots + (size_t)slot * RDIG;
                for (int q = 0; q < RDIG; ++q) ccs[q] = 0ull;
                const uint32_t ntiles = tiles_of(cb, ce);
                Seg *s = &P.segs[csid];
                s->begin = cb;
                s->end = ce;
                s->pivot = 0;
                s->pivot_v = (uint32_t)rwidth(P, mc, nrbit);
                s->lb = pk;
                s->lb_v = pv;
                s->ntiles = ntiles;
                s->info = (dstB ? I_SRC_B : 0) | I_RADIX8;
                s->rbit = (unsigned)nrbit;
                s->rslot = slot;
                s->budget = 0;
                s->depth = sg.depth + 1;
                s->cnt_left = 0;
                s->cnt_right = 0;
                s->cnt_eq = 0;
                s->tiles_done = 0;
                __threadfence();
                const uint32_t nt = seg_ntasks(ntiles, P.chunk);
                const unsigned long long pos = atomicAdd(&P.st->q_tail, (unsigned long long)nt);
                const uint64_t mask = (1ull << P.log_q) - 1;
                for (uint32_t t = 0; t < nt; ++t)
                    *(volatile uint64_t *)&P.ring[(pos + t) & mask] =
                        task_word(pos + t, P.log_q, T_RHIST, csid, t * P.chunk);
                atomicMax(&sh.s_max_depth, (long long)(sg.depth + 1));
            }
        } else if (mc > 1) {
            seq[atomicAdd(&sh.rl_seq, 1)] = (uint8_t)tid;  // a constant run in B longer than a leaf
        }
        csync();
        for (int i = warp; i < sh.rl_tiny; i += WARPS) {
            const int d = tiny[i];
            const int64_t tb = d ? (int64_t)E[d - 1] : sg.begin;
            tiny_sort_warp(P, dstB, tb, (int)((int64_t)E[d] - tb));
        }
        csync();
        const int nseq = sh.rl_seq;
        for (int i = 0; i < nseq; ++i) {
            // This loop can run for a millisecond (up to 256 children started one after another).  The CTA
            // holds a claimed ring position all that time; if the other CTAs push a whole ring's worth of
            // tasks meanwhile (many one-tile digit passes of tiny segments), the slot is overwritten before it
            // is read and its task is lost (found by tools/fuzz.py: the queue stalled).  Copying the task out
            // of the ring as soon as it appears bounds the exposure to one iteration.
            if (tid == 0 && sh.nstate == 1) poll_next(P);
            const int d = seq[i];
            const int64_t tb = d ? (int64_t)E[d - 1] : sg.begin, te = (int64_t)E[d];
            if (nrbit >= NBITS) {
                finish_constant(P, tb, te, dstB);
            } else {
                uint64_t qk = sg.lb;
                uint32_t qv = sg.lb_v;
                put_digit(qk, qv, rbit, nd, (uint32_t)d);
                radix_split(P, tb, te, dstB, nrbit, qk, qv, sg.depth + 1, -1);
            }
        }
        csync();
    }

    // ---- thread 0: issue the TMA bulk load of tile `tile` of segment `sg` into the next stage ----------
    __device__ static void issue_load(const Params &P, const Seg &sg, uint32_t tile, bool keys_only = false) {
        Shared &sh = g_sh;
        const int st = (int)(sh.li % B::NSTAGE);
        ++sh.li;
        const int64_t b = sg.begin, e = sg.end;
        const bool srcB = sg.info & I_SRC_B;
        const U *src = (const U *)(srcB ? P.b_keys : P.a_keys);
        const uint32_t *srcv = srcB ? P.b_vals : P.a_vals;
        const int64_t tbase = tile_base(b, tile);
        const int64_t lo = b > tbase ? b : tbase;
        const int64_t hi = e < tbase + TL ? e : tbase + TL;
        const int64_t nfl = P.n & ~(int64_t)(AL - 1);
        const int64_t lo_al = lo & ~(int64_t)(AL - 1);
        int64_t hi_al = (hi + AL - 1) & ~(int64_t)(AL - 1);
        if (hi_al > nfl) hi_al = nfl;
        U *sk = B::stage(st);
        uint32_t *sv = KV ? B::vstage(st) : nullptr;
        // the array's last < 16 bytes cannot be bulk-copied: scalar loads
        for (int64_t g = (hi_al > lo ? hi_al : lo); g < hi; ++g) {
            sk[g - tbase] = ldcg(src + g);
            if (KV && !keys_only) sv[g - tbase] = ldcg(srcv + g);
        }
        const unsigned kb = hi_al > lo_al ? (unsigned)((hi_al - lo_al) * sizeof(U)) : 0u;
        const unsigned vb = (KV && !keys_only && hi_al > lo_al) ? (unsigned)((hi_al - lo_al) * 4) : 0u;
        fence_proxy_async();
        mbar_expect_tx(&sh.bar[st], kb + vb);  // the stage barrier's single arrival (+ bytes, maybe 0)
        if (kb) {
            bulk_g2s(sk + (lo_al - tbase), src + lo_al, kb, &sh.bar[st]);
            if (vb) bulk_g2s(sv + (lo_al - tbase), srcv + lo_al, vb, &sh.bar[st]);
        }
    }

    // ---- K2/K3: one partition tile (compute warps) ------------------------------------------------
    __device__ __forceinline__ static void stvec(U *g, const U (&x)[VEC]) {
        if constexpr (sizeof(U) == 4)
            *reinterpret_cast<uint4 *>(g) = make_uint4(x[0], x[1], x[2], x[3]);
        else
            *reinterpret_cast<ulonglong2 *>(g) = make_ulonglong2(x[0], x[1]);
    }
    __device__ __forceinline__ static void ldvec(const U *s, int q, U (&x)[VEC]) {
        if constexpr (sizeof(U) == 4) {
            const uint4 y = reinterpret_cast<const uint4 *>(s)[q];
            x[0] = y.x;
            x[1] = y.y;
            x[2] = y.z;
            x[3] = y.w;
        } else {
            const ulonglong2 y = reinterpret_cast<const ulonglong2 *>(s)[q];
            x[0] = y.x;
            x[1] = y.y;
        }
    }

    // Per-thread classification of the IT keys of thread t (the VEC-key vectors
    // q = jj*THREADS + t); lmask/vmask record left/valid per item.
    template <bool FULL>
    __device__ __forceinline__ static void classify(const U *sk, const uint32_t *sv, int lo_i, int hi_i, U piv,
                                                    uint32_t pv, bool left_mode, bool count_eq, unsigned &lmask,
                                                    unsigned &vmask, int &eqc) {
        const int tid = threadIdx.x;
#pragma unroll
        for (int jj = 0; jj < IT / VEC; ++jj) {
            const int q = jj * THREADS + tid;
            U kk[VEC];
            ldvec(sk, q, kk);
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                const int r = jj * VEC + e;
                const int idx = q * VEC + e;
                const uint32_t v = KV ? sv[idx] : 0u;
                const bool valid = FULL || (idx >= lo_i && idx < hi_i);
                const bool isl = valid && (left_mode ? !lt_raw(piv, pv, kk[e], v) : lt_raw(kk[e], v, piv, pv));
                lmask |= (unsigned)isl << r;
                if (!FULL) vmask |= (unsigned)valid << r;
                if (count_eq) eqc += (valid && kk[e] == piv && (!KV || v == pv)) ? 1 : 0;
            }
        }
        if (FULL) vmask = (1u << IT) - 1;
    }

    // ballot of (m & bit) != 0 (bit a compile-time constant after unrolling): one LOP3 to a predicate
    // and one VOTE; the generic form costs a shift, a LOP3 and an ISETP more per item
    __device__ __forceinline__ static unsigned ballot_bit(unsigned m, unsigned bit) {
        unsigned b;
        asm("{\n .reg .pred p;\n .reg .b32 t;\n and.b32 t, %1, %2;\n setp.ne.b32 p, t, 0;\n"
            " vote.sync.ballot.b32 %0, p, 0xffffffff;\n}\n"
            : "=r"(b)
            : "r"(m), "r"(bit));
        return b;
    }

    // Branch-free compaction of this warp's keys into kc: its lefts fill [li, ...), its rights
    // [ri, ...).  Ranks come from one ballot per item slot, so the 32 lanes of every store land in
    // two contiguous runs of kc (at most a 2-way bank conflict; a per-thread prefix would put
    // lanes ~8 words apart, an 8-way conflict).  Order within a side is free (no stability,
    // PAPER.md:28-29).  The keys are re-read from the stage (registers are the occupancy limit).
    template <bool FULL>
    __device__ __forceinline__ static void scatter(const U *sk, const uint32_t *sv, U *kc, uint32_t *vc,
                                                   unsigned lmask, unsigned vmask, int li, int ri) {
        const int tid = threadIdx.x;
        const unsigned ltm = lanemask_lt();
        if constexpr (FULL) {
            // every lane holds a valid item in every round: a right's rank is (lane - lefts before it),
            // so one ballot and two popcounts per round place all 32 items
            int rw = ri + (tid & 31);
#pragma unroll
            for (int jj = 0; jj < IT / VEC; ++jj) {
                const int q = jj * THREADS + tid;
                U kk[VEC];
                ldvec(sk, q, kk);
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    const unsigned bl = ballot_bit(lmask, 1u << (jj * VEC + e));
                    const bool isl = (bl >> (tid & 31)) & 1u;
                    const int d = __popc(bl & ltm), c = __popc(bl);
                    const int pos = isl ? li + d : rw - d;
                    PDQ_CHECK(pos >= 0 && pos < B::SLOT, "partition compaction slot");
                    kc[pos] = kk[e];
                    if (KV) vc[pos] = sv[q * VEC + e];
                    li += c;
                    rw += 32 - c;
                }
            }
        } else {
#pragma unroll
            for (int jj = 0; jj < IT / VEC; ++jj) {
                const int q = jj * THREADS + tid;
                U kk[VEC];
                ldvec(sk, q, kk);
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    const unsigned bit = 1u << (jj * VEC + e);
                    const unsigned bl = ballot_bit(lmask, bit), br = ballot_bit(vmask, bit) & ~bl;
                    const unsigned me = 1u << (tid & 31);
                    const int pos = (bl & me) ? li + __popc(bl & ltm) : ri + __popc(br & ltm);
                    if ((bl | br) & me) {
                        PDQ_CHECK(pos >= 0 && pos < B::SLOT, "partition compaction slot (edge tile)");
                        kc[pos] = kk[e];
                        if (KV) vc[pos] = sv[q * VEC + e];
                    }
                    li += __popc(bl);
                    ri += __popc(br);
                }
            }
        }
    }

    // Store the run kc[a, a + len) (and vc) to dk[g, g + len) (and dv), a = g mod AL: the 16-byte
    // aligned body by one TMA bulk store per array (issued by thread 0, committed by the caller),
    // the < AL-element head and tail by threads t0 + i (warp 0).
    __device__ __forceinline__ static void emit_run(const U *kc, const uint32_t *vc, U *dk, uint32_t *dv,
                                                    long long g, int a, int len, int t0) {
        const int tid = threadIdx.x;
        int h = (int)((AL - (g & (AL - 1))) & (AL - 1));
        if (h > len) h = len;
        const int nb = ((len - h) / AL) * AL;
        const int i = tid - t0;
        if (i >= 0 && i < AL) {
            if (i < h) {
                dk[g + i] = kc[a + i];
                if (KV) dv[g + i] = vc[a + i];
            }
            const int j = h + nb + i;
            if (j < len) {
                dk[g + j] = kc[a + j];
                if (KV) dv[g + j] = vc[a + j];
            }
        }
        if (tid == 0 && nb) {
            bulk_s2g(dk + g + h, kc + a + h, (unsigned)(nb * sizeof(U)));
            if (KV) bulk_s2g(dv + g + h, vc + a + h, (unsigned)(nb * 4));
        }
    }

    // Contiguous coalesced store of `len` elements of shared memory run `s` to global `g`: lane
    // stride 1 on both sides (conflict-free shared reads; alignment of g is arbitrary).
    template <class T, class F>
    __device__ __forceinline__ static void store_lin(T *g, int len, F get) {
        for (int i = threadIdx.x; i < len; i += THREADS) g[i] = get(i);
    }

    // Partition the tile in stage `s`; returns after the stores are issued.  Releases the stage
    // (empty barrier) as soon as its buffer has been consumed.
    //   left = key <  pivot  (partition_right: equals go right, partition.py:76-77)
    //   left = key <= pivot  (partition_left: equals go left, partition.py:134-135)
    // Each warp sums its counts; the per-warp totals (packed left | right << 16) give every warp its
    // runs in the compaction buffer kc.  One 64-bit atomic per CTA reserves both output runs before
    // the scatter, so each run is placed in kc at the 16-byte phase of its destination and its body
    // leaves by one TMA bulk store (no per-key store instructions).
    // One partition tile of the current task (sh.seg), whose TMA load is in flight in the stage.
    // After the stage is consumed thread 0 starts the next load (next tile of this chunk, or the
    // first tile of the already-claimed next task), so the load overlaps this tile's stores.
    __device__ static void part_tile(const Params &P, uint32_t sid, uint32_t tile, unsigned &ci) {
        Shared &sh = g_sh;
        const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
        const Seg &sg = sh.seg;
        const int64_t b = sg.begin, e = sg.end;
        const bool srcB = sg.info & I_SRC_B;
        const bool left_mode = sg.info & I_LEFT;
        const bool count_eq = (sg.info & I_COUNT_EQ) && !left_mode;
        const bool packed = (e - b) < (1ll << 32);
        const int64_t tbase = tile_base(b, tile);
        const int64_t lo = b > tbase ? b : tbase;
        const int64_t hi = e < tbase + TL ? e : tbase + TL;
        const int st = (int)(ci % B::NSTAGE);
        const U *sk = B::stage(st);
        const uint32_t *sv = KV ? B::vstage(st) : nullptr;
        const U piv = (U)sg.pivot;
        const uint32_t pv = sg.pivot_v;
        const int lo_i = (int)(lo - tbase), hi_i = (int)(hi - tbase);
        const long long q0 = clock64();
        mbar_wait(&sh.bar[st], (ci / B::NSTAGE) & 1u);
        ++ci;
        const long long q1 = clock64();
#ifndef PDQ_BIG_PHASES
        if (tid == 0) sh.s_sch_claim += q1 - q0;  // (profiling) stage wait
#endif
        unsigned lmask = 0, vmask = 0;
        int eqc = 0;
        if (lo_i == 0 && hi_i == TL)
            classify<true>(sk, sv, lo_i, hi_i, piv, pv, left_mode, count_eq, lmask, vmask, eqc);
        else
            classify<false>(sk, sv, lo_i, hi_i, piv, pv, left_mode, count_eq, lmask, vmask, eqc);
        const int nl = __popc(lmask), nv = __popc(vmask);
        const uint32_t mine = (uint32_t)nl | ((uint32_t)(nv - nl) << 16);
        const uint32_t wsum = __reduce_add_sync(0xffffffffu, mine);  // warp totals, left | right << 16
        if (count_eq) eqc = __reduce_add_sync(0xffffffffu, eqc);
        if (lane == 0) {
            sh.scan[warp] = wsum;
            sh.weq[warp] = eqc;
        }
        csync();
        uint32_t wpre = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
            const uint32_t x = sh.scan[w];
            wpre += (w < warp) ? x : 0u;
            tot += x;
        }
        const int L = (int)(tot & 0xFFFF), R = (int)(tot >> 16);
        const bool write_left = !left_mode || srcB;  // K3 from A: the lefts are filled later
        if (tid == 0) {
            // one atomic per CTA reserves both runs (left grows up from `begin`, right grows down
            // from `end`); the runs are placed in kc at the 16-byte phase of their destinations
            Seg *gs = &P.segs[sid];
            long long lOff, rOff;
            if (packed) {
                const unsigned long long r =
                    atomicAdd(&gs->cnt_left, (unsigned long long)L | ((unsigned long long)R << 32));
                lOff = (long long)(r & 0xFFFFFFFFull);
                rOff = (long long)(r >> 32);
            } else {
                lOff = (long long)atomicAdd(&gs->cnt_left, (unsigned long long)L);
                rOff = (long long)atomicAdd(&gs->cnt_right, (unsigned long long)R);
            }
            if (count_eq) {
                int E = 0;
#pragma unroll
                for (int w = 0; w < WARPS; ++w) E += sh.weq[w];
                if (E) atomicAdd(&gs->cnt_eq, (unsigned long long)E);
            }
            const long long gl = b + lOff, gr = e - rOff - R;
            PDQ_CHECK(gl >= b && gl + L <= gr && gr + R <= e, "tile reservation inside its segment");
            const int aL = (int)(gl & (AL - 1));
            const int aR = aL + L + (int)((gr - (aL + L)) & (AL - 1));
            sh.lOff = gl;
            sh.rOff = gr;
            sh.aL = aL;
            sh.aR = aR;
            sh.s_tiles++;
            sh.s_bytes += (unsigned long long)ELEM_BYTES * (L + R) +
                          (unsigned long long)ELEM_BYTES * (R + (write_left ? L : 0));
            bulk_wait_read();  // the previous tile's bulk stores have left kc
        }
        csync();
        const int aL = sh.aL, aR = sh.aR;
        const int li0 = aL + (int)(wpre & 0xFFFF), ri0 = aR + (int)(wpre >> 16);  // this warp's runs in kc
        U *kc = B::kc();
        uint32_t *vc = KV ? B::vc() : nullptr;
        if (lo_i == 0 && hi_i == TL)  // CTA-uniform (the ballots need every lane)
            scatter<true>(sk, sv, kc, vc, lmask, vmask, li0, ri0);
        else
            scatter<false>(sk, sv, kc, vc, lmask, vmask, li0, ri0);
        fence_proxy_async();  // kc (generic writes) is read next by the TMA engine
        csync();              // stage consumed, kc complete
        const long long gl = sh.lOff, gr = sh.rOff;
        U *dst = (U *)(srcB ? P.a_keys : P.b_keys);
        uint32_t *dstv = srcB ? P.a_vals : P.b_vals;
        if (tid == 0) {
            sh.ci = ci;
            pump_loads(P);
        }
        if (L && write_left) emit_run(kc, vc, dst, dstv, gl, aL, L, 1);
        if (R) emit_run(kc, vc, dst, dstv, gr, aR, R, 8);
        if (tid == 0) bulk_commit();
#ifndef PDQ_BIG_PHASES
        if (tid == 0) sh.s_sch_idle += clock64() - q1;  // (profiling) whole tile after the stage wait
#endif
    }

    // thread 0: keep NST tile loads in flight ahead of the compute side, walking the current task's
    // chunk and then, once it is published, the next task's chunk.
    __device__ __forceinline__ static void pump_loads(const Params &P) {
        Shared &sh = g_sh;
        while (sh.li < sh.ci + B::NSTAGE) {
            if (sh.lslot == 0) {
                if (sh.task && tile_task((uint32_t)(sh.task >> 45) & 7u)) {
                    const uint32_t end = task_end_tile((uint32_t)(sh.task & 0x7FFFFF), sh.seg.ntiles, P.chunk);
                    if (sh.ltile < end) {
                        issue_load(P, sh.seg, sh.ltile++, hist_keys_only(sh.task, sh.seg));
                        continue;
                    }
                }
                // the current task has no more tiles: move to the next task
                if (sh.nstate == 1) poll_next(P);
                if (sh.nstate != 2) return;
                sh.lslot = 1;
                sh.ltile = tile_task((uint32_t)(sh.ntask >> 45) & 7u) ? ((uint32_t)sh.ntask & 0x7FFFFF) : 0u;
            }
            // load cursor in the next task
            if (!tile_task((uint32_t)(sh.ntask >> 45) & 7u)) return;
            const uint32_t end = task_end_tile((uint32_t)(sh.ntask & 0x7FFFFF), sh.nseg.ntiles, P.chunk);
            if (sh.ltile >= end) return;
            issue_load(P, sh.nseg, sh.ltile++, hist_keys_only(sh.ntask, sh.nseg));
        }
    }

    // thread 0: non-blocking poll of the claimed next ring position
    __device__ static void poll_next(const Params &P) {
        Shared &sh = g_sh;
        const uint64_t mask = (1ull << P.log_q) - 1;
        const unsigned long long pos = sh.npos;
        const uint64_t w = ld_acquire_u64(P.ring + (pos & mask));
        if ((w >> 48) == ((pos >> P.log_q) & 0xFFFFull)) {
            const uint32_t sid = (uint32_t)(w >> 23) & 0x3FFFFF;
            const ulonglong2 *gsrc = reinterpret_cast<const ulonglong2 *>(&P.segs[sid]);
            ulonglong2 *sdst = reinterpret_cast<ulonglong2 *>(&sh.nseg);
#pragma unroll
            for (int q = 0; q < 8; ++q) sdst[q] = __ldcg(gsrc + q);
            sh.ntask = w;
            sh.nstate = 2;
            fence_proxy_async_global();  // the task's data (acquired above) is read by TMA bulk loads
        }
    }

    // thread 0: make the claimed next task current (blocking until it is published or the sort is
    // done), start its first load if it was not prefetched, and claim the position after it.
    __device__ static void advance(const Params &P) {
        Shared &sh = g_sh;
        if (sh.nstate == 1) {
            const uint64_t t0 = globaltimer_ns();
            unsigned ns = 32;
            for (;;) {
                poll_next(P);
                if (sh.nstate == 2) break;
                if (ld_volatile_u32(&P.st->done)) {
                    sh.nstate = 3;
                    break;
                }
                if (globaltimer_ns() - t0 > WATCHDOG_NS) {  // no task for 10 s: report, never hang
                    fail(P, -8);
                    sh.nstate = 3;
                    break;
                }
                __nanosleep(ns);
                if (ns < PDQ_SLEEP_CAP) ns <<= 1;
            }
        }
        if (sh.nstate == 3) {
            sh.task = 0;
            return;
        }
        const bool cursor_ahead = sh.lslot == 1;
        sh.task = sh.ntask;
        sh.seg = sh.nseg;
        sh.lslot = 0;
        if (!cursor_ahead) sh.ltile = tile_task((uint32_t)(sh.task >> 45) & 7u) ? ((uint32_t)sh.task & 0x7FFFFF) : 0u;
        // claim the following position now: its atomic overlaps the whole current task
        sh.npos = atomicAdd(&P.st->q_head, 1ull);
        sh.nstate = 1;
        pump_loads(P);
    }

    __device__ static void fill_tile(const Params &P, const Seg &sg, uint32_t tile) {
        Shared &sh = g_sh;
        const int64_t tbase = tile_base(sg.begin, tile);
        const int64_t lo = sg.begin > tbase ? sg.begin : tbase;
        const int64_t hi = sg.end < tbase + TL ? sg.end : tbase + TL;
        const U raw = O::from((U)sg.pivot);
        const uint32_t pv = sg.pivot_v;
        store_run<U>((U *)P.a_keys + lo, (int)(hi - lo), [&](int) { return raw; });
        if (KV) store_run<uint32_t>(P.a_vals + lo, (int)(hi - lo), [&](int) { return pv; });
        __threadfence();
        csync();
        if (threadIdx.x == 0) {
            sh.s_bytes += (unsigned long long)ELEM_BYTES * (hi - lo);
            finish_keys(P, (unsigned long long)(hi - lo));
        }
    }

    __device__ static void zero_counters() {
        Shared &sh = g_sh;
        sh.s_part_right = sh.s_part_left = sh.s_bad = sh.s_fallback = sh.s_base = sh.s_tiles = sh.s_bytes = 0;
        sh.s_max_depth = 0;
        sh.s_cyc_wait = sh.s_cyc_work = sh.s_cyc_base = sh.s_cyc_spawn = 0;
        sh.s_sch_retire = sh.s_sch_claim = sh.s_sch_fetch = sh.s_sch_idle = 0;
    }
    __device__ static void flush_counters(const Params &P) {
        Shared &sh = g_sh;
        State *st = P.st;
        if (sh.s_part_right) atomicAdd(&st->c_part_right, sh.s_part_right);
        if (sh.s_part_left) atomicAdd(&st->c_part_left, sh.s_part_left);
        if (sh.s_bad) atomicAdd(&st->c_bad, sh.s_bad);
        if (sh.s_fallback) atomicAdd(&st->c_fallback, sh.s_fallback);
        if (sh.s_base) atomicAdd(&st->c_base, sh.s_base);
        if (sh.s_tiles) atomicAdd(&st->c_tiles, sh.s_tiles);
        if (sh.s_bytes) atomicAdd(&st->c_bytes, sh.s_bytes);
        if (sh.s_max_depth) atomicMax(&st->c_max_depth, (unsigned long long)sh.s_max_depth);
        atomicAdd(&st->c_cyc_wait, sh.s_cyc_wait);
        atomicAdd(&st->c_cyc_work, sh.s_cyc_work);
        atomicAdd(&st->c_cyc_base, sh.s_cyc_base);
        atomicAdd(&st->c_cyc_spawn, sh.s_cyc_spawn);
        atomicAdd(&st->c_sch_retire, sh.s_sch_retire);
        atomicAdd(&st->c_sch_claim, sh.s_sch_claim);
        atomicAdd(&st->c_sch_fetch, sh.s_sch_fetch);
        atomicAdd(&st->c_sch_idle, sh.s_sch_idle);
    }
};

// ---- K4: adjacent-compare reduction with early exit ---------------------------------------------
// One pass over adjacent pairs: bit 0 a descent was seen, bit 1 an ascent, bit 2 a descent in the first
// half of the array, bit 3 a descent in the second half (for arrays too short for the two-run path every
// descent sets both).  The pass is cut short once bits 1, 2 and 3 are all set: the input is then neither
// sorted, nor reversed, nor a sorted run of at least half the array next to a second run; uniform input
// stops after one or two chunks per CTA.  When the pass runs to the end, the first and last descent and the
// first and last ascent are exact (k_init reads them to recognise two runs: small_sorts.py:76-115's
// "nearly sorted" case on the GPU is a sorted run of at least half the array next to anything).
#ifndef PDQ_CHECK_MINB
#define PDQ_CHECK_MINB 1
#endif
template <class U, bool FLOAT, bool KV>
__global__ void __launch_bounds__(THREADS, PDQ_CHECK_MINB) k_check(const __grid_constant__ Params P) {
    using O = Ord<U, FLOAT>;
    __shared__ unsigned s_pub;
    __shared__ unsigned long long s_red[4][WARPS];
    const int tid = threadIdx.x, lane = tid & 31;
    pdl_trigger();  // k_init (one CTA) may be scheduled now; it waits for this grid before reading
    {  // the task ring starts empty (all-ones words match no round tag); k_init pushes after this grid
        uint4 *r4 = reinterpret_cast<uint4 *>(P.ring);
        const int64_t words = (1ll << P.log_q) / 2;
        for (int64_t i = (int64_t)blockIdx.x * THREADS + tid; i < words; i += (int64_t)gridDim.x * THREADS)
            r4[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
    }
    if (tid == 0) s_pub = 0;
    __syncthreads();
    const U *a = (const U *)P.a_keys;
    const int64_t n = P.n;
#ifndef PDQ_CHECK_STEPS
#define PDQ_CHECK_STEPS 4
#endif
    constexpr int E = 4, STEPS = PDQ_CHECK_STEPS;  // a thread reads 4 elements (16-byte vectors) per step
    const int64_t CH = (int64_t)THREADS * STEPS * E;
    // a descent at index i < early leaves a sorted prefix shorter than half the array, one at i >= late a
    // sorted suffix shorter than half
    const bool two_run = n >= P.runs_min;
    const int64_t early = two_run ? (n + 1) / 2 - 1 : n, late = two_run ? n / 2 : 0;
    constexpr unsigned long long NONE = ~0ull;
    // this thread's first descent, last descent + 1, first ascent, last ascent + 1
    unsigned long long d1 = NONE, dl = 0, fa = NONE, la = 0;
    unsigned long long bytes = 0;
    // Half of the CTAs stride over the chunks of the first half of the array, the others over the second
    // half: two contiguous windows move through the array (a CTA-contiguous split costs 30 % of the pass's
    // bandwidth), a thread's indices only grow, and the first wave already sees both halves.
    const int64_t nchunks = (n - 1 + CH - 1) / CH;
    // (Even CTAs take the first half, odd CTAs the second: whatever subset of the grid is resident sees both
    // halves -- with the halves split by CTA index, a grid of two waves ran the whole first half before any
    // CTA of the second half started.)
    const int64_t G = gridDim.x, G1 = G >= 2 ? (G + 1) / 2 : G, mid = G >= 2 ? nchunks / 2 : nchunks;
    const bool lower = G < 2 || (blockIdx.x & 1u) == 0;
    const int64_t ch0 = lower ? (int64_t)(blockIdx.x >> (G >= 2 ? 1 : 0)) : mid + (int64_t)(blockIdx.x >> 1);
    const int64_t c_end = lower ? mid : nchunks, c_step = lower ? G1 : G - G1;
    for (int64_t ch = ch0; ch < c_end; ch += c_step) {
        const int64_t c0 = ch * CH;
        // the verdict so far (its latency overlaps the chunk's loads; threads may leave one chunk apart)
        const unsigned flag = ld_volatile_u32(&P.st->check_bits);
        unsigned bits = 0;
        // all of the chunk's loads first (a whole chunk needs no bounds checks: one 16-byte vector per
        // step and thread in flight, the element after each vector from the next lane or, for lane 31,
        // by one scalar load); the array's last chunk loads element by element
        U kk[STEPS][E + 1];
        uint32_t vv[STEPS][E + 1];
        const bool whole = c0 + CH < n;
        if (whole) {
#pragma unroll
            for (int st = 0; st < STEPS; ++st) {
                const int64_t i = c0 + ((int64_t)st * THREADS + tid) * E;
                if constexpr (sizeof(U) == 4) {
                    const uint4 y = __ldg(reinterpret_cast<const uint4 *>(a + i));
                    kk[st][0] = (U)y.x; kk[st][1] = (U)y.y; kk[st][2] = (U)y.z; kk[st][3] = (U)y.w;
                } else {
                    const ulonglong2 y0 = __ldg(reinterpret_cast<const ulonglong2 *>(a + i));
                    const ulonglong2 y1 = __ldg(reinterpret_cast<const ulonglong2 *>(a + i + 2));
                    kk[st][0] = (U)y0.x; kk[st][1] = (U)y0.y; kk[st][2] = (U)y1.x; kk[st][3] = (U)y1.y;
                }
                if constexpr (KV) {
                    const uint4 z = __ldg(reinterpret_cast<const uint4 *>(P.a_vals + i));
                    vv[st][0] = z.x; vv[st][1] = z.y; vv[st][2] = z.z; vv[st][3] = z.w;
                } else {
                    vv[st][0] = vv[st][1] = vv[st][2] = vv[st][3] = 0;
                }
                kk[st][E] = 0;
                vv[st][E] = 0;
                if (lane == 31) {
                    kk[st][E] = __ldg(a + i + E);
                    if constexpr (KV) vv[st][E] = __ldg(P.a_vals + i + E);
                }
            }
        } else {
#pragma unroll
            for (int st = 0; st < STEPS; ++st) {
                const int64_t i = c0 + ((int64_t)st * THREADS + tid) * E;
#pragma unroll
                for (int q = 0; q <= E; ++q) {
                    kk[st][q] = 0;
                    vv[st][q] = 0;
                    if (i + q < n && (q < E || lane == 31)) {
                        kk[st][q] = a[i + q];
                        if constexpr (KV) vv[st][q] = P.a_vals[i + q];
                    }
                }
            }
        }
#pragma unroll
        for (int st = 0; st < STEPS; ++st) {
            const int64_t i = c0 + ((int64_t)st * THREADS + tid) * E;
            U(&k)[E + 1] = kk[st];
            uint32_t(&v)[E + 1] = vv[st];
            // the element after this thread's vector: the next lane's first (lane 31 loaded it)
            {
                U nk;
                if constexpr (sizeof(U) == 4) nk = (U)__shfl_down_sync(0xffffffffu, (uint32_t)k[0], 1);
                else nk = (U)__shfl_down_sync(0xffffffffu, (unsigned long long)k[0], 1);
                const uint32_t nv = KV ? __shfl_down_sync(0xffffffffu, v[0], 1) : 0u;
                if (lane != 31) {
                    k[E] = nk;
                    v[E] = nv;
                }
            }
            // ordered images once per element; the four pairs' verdicts as two 4-bit masks, so the 64-bit
            // index bookkeeping runs once per vector (and only when a mask is non-zero)
            uint64_t o[E + 1];
#pragma unroll
            for (int q = 0; q <= E; ++q) o[q] = (uint64_t)O::to(k[q]);
            unsigned dm = 0, am = 0;
#pragma unroll
            for (int q = 0; q < E; ++q) {
                dm |= (pless<KV>(o[q + 1], v[q + 1], o[q], v[q]) ? 1u : 0u) << q;
                am |= (pless<KV>(o[q], v[q], o[q + 1], v[q + 1]) ? 1u : 0u) << q;
            }
            if (i + E > n - 1) {  // the array's last vectors: pairs (j, j + 1) exist for j < n - 1
                const int64_t left = n - 1 - i;
                const unsigned keep = left <= 0 ? 0u : (1u << left) - 1u;
                dm &= keep;
                am &= keep;
            }
            if (dm) {  // (a thread's indices only grow)
                const int64_t lo = i + (__ffs(dm) - 1), hi = i + (31 - __clz(dm));
                bits |= 1u | (lo < early ? 4u : 0u) | (hi >= late ? 8u : 0u);
                if (d1 == NONE) d1 = (unsigned long long)lo;
                dl = (unsigned long long)hi + 1;
            }
            if (am) {
                bits |= 2u;
                if (fa == NONE) fa = (unsigned long long)(i + (__ffs(am) - 1));
                la = (unsigned long long)(i + (31 - __clz(am))) + 1;
            }
        }
        bits = __reduce_or_sync(0xffffffffu, bits);
        // publish only what neither this CTA nor anyone else has published yet: thousands of atomics on
        // one word serialise in its L2 slice (8 per CTA x 1184 CTAs cost ~25 us at the start of every sort)
        if (lane == 0 && bits) {
            const unsigned fresh = bits & ~atomicOr(&s_pub, bits);
            if (fresh && (fresh & ~ld_volatile_u32(&P.st->check_bits))) atomicOr(&P.st->check_bits, fresh);
        }
        if (tid == 0) {
            const int64_t hi = c0 + CH < n ? c0 + CH : n;
            bytes += (unsigned long long)(hi - c0) * (sizeof(U) + (KV ? 4 : 0));
        }
        if ((flag & 14u) == 14u) break;
    }
    // CTA reduction of the run marks, one atomic each
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a1 = __shfl_xor_sync(0xffffffffu, d1, o), a2 = __shfl_xor_sync(0xffffffffu, dl, o),
                                 a3 = __shfl_xor_sync(0xffffffffu, la, o), a4 = __shfl_xor_sync(0xffffffffu, fa, o);
        d1 = a1 < d1 ? a1 : d1;
        dl = a2 > dl ? a2 : dl;
        la = a3 > la ? a3 : la;
        fa = a4 < fa ? a4 : fa;
    }
    if (lane == 0) {
        s_red[0][tid >> 5] = d1;
        s_red[1][tid >> 5] = dl;
        s_red[2][tid >> 5] = la;
        s_red[3][tid >> 5] = fa;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < WARPS; ++w) {
            d1 = s_red[0][w] < d1 ? s_red[0][w] : d1;
            dl = s_red[1][w] > dl ? s_red[1][w] : dl;
            la = s_red[2][w] > la ? s_red[2][w] : la;
            fa = s_red[3][w] < fa ? s_red[3][w] : fa;
        }
        if (d1 != NONE) atomicMax(&P.st->run_d1_inv, ~d1);
        if (dl) atomicMax(&P.st->run_dl, dl);
        if (la) atomicMax(&P.st->run_la, la);
        if (fa != NONE) atomicMax(&P.st->run_fa_inv, ~fa);
        if (bytes) atomicAdd(&P.st->c_bytes_check, bytes);
    }
}

// ---- init: decide from K4, reverse flag, root segment --------------------------------------------
// K4 verdicts: no descent -> sorted; no ascent -> reversed in place; no descent in the first half (the
// pass then ran to the end) -> two runs: A[0, s) is sorted, s = first descent + 1 >= n / 2, and the rest
// is left as it is (ascending: a single descent), reversed (no ascent beyond s) or sorted by the tree as
// the root segment [s, n); mirrored, no descent in the second half -> A[s, n) is sorted, s = last descent
// + 1 <= n / 2, and A[0, s) is left, reversed or sorted by the tree.  The leaf kernel then merges the two
// runs (RunsMerge).  Anything else: the root segment is the whole array.
template <class U, bool FLOAT, bool KV>
__global__ void __launch_bounds__(THREADS) k_init(const __grid_constant__ Params P) {
    using S = Sorter<U, FLOAT, KV>;
    Shared &sh = g_sh;
    __shared__ int s_action;
    __shared__ long long s_rb, s_re;
    const int tid = threadIdx.x;
    pdl_wait();     // k_check's verdict
    pdl_trigger();  // the sorter's CTAs may be scheduled; they wait for this grid before reading
    if (tid == 0) {
        S::zero_counters();
        State *st = P.st;
        const unsigned bits = st->check_bits;
        int action = 0;  // 0 = sort [rb, re), 1 = done (sorted), 2 = reverse [rb, re)
        long long rb = 0, re = P.n;
        if (P.n <= 1) action = 1;
        else if (P.use_check && !(bits & 1u)) action = 1;
        else if (P.use_check && !(bits & 2u)) action = 2;
        else if (P.use_check && P.n >= P.runs_min && !(bits & 4u)) {
            const unsigned long long s = ~st->run_d1_inv + 1;  // the second run starts here
            st->run_split = s;
            rb = (long long)s;
            if (st->run_dl == s) {  // a single descent: the second run is ascending
                st->run_kind = 1;
                action = 1;
            } else if (st->run_la <= s) {  // no ascent beyond s: the second run is reversed in place
                st->run_kind = 2;
                action = 2;
            } else {  // the tree sorts [s, n)
                st->run_kind = 3;
            }
        } else if (P.use_check && P.n >= P.runs_min && !(bits & 8u)) {
            const unsigned long long s = st->run_dl;  // the sorted second run starts here (last descent + 1)
            st->run_split = s;
            re = (long long)s;
            if (~st->run_d1_inv + 1 == s) {  // a single descent: the first run is ascending (and shorter)
                st->run_kind = 5;
                action = 1;
            } else if (st->run_fa_inv == 0 || ~st->run_fa_inv + 1 >= s) {  // no ascent inside [0, s): reversed
                st->run_kind = 6;
                action = 2;
            } else {  // the tree sorts [0, s)
                st->run_kind = 7;
            }
        }
        s_action = action;
        s_rb = rb;
        s_re = re;
        if (action == 1) {
            st->keys_final = P.n;
            st->done = 1;
        } else if (action == 2) {
            st->reverse = 1;
            st->rev_begin = (unsigned long long)rb;
            st->rev_end = (unsigned long long)re;
            st->keys_final = P.n;
            st->done = 1;
            sh.s_bytes += 2ull * (sizeof(U) + (KV ? 4 : 0)) * (unsigned long long)(re - rb);
        } else {
            st->keys_final = (unsigned long long)(P.n - (re - rb));  // the sorted run is final for the tree
        }
    }
    __syncthreads();
    if (s_action == 0) {
        const int64_t m = s_re - s_rb;
        int budget = P.budget0;
        if (budget < 0) budget = 63 - __clzll((long long)m);  // driver.py:263: n.bit_length() - 1
        typename S::Bnd none{};
        S::spawn(P, s_rb, s_re, false, none, budget, 0, false, -1);
    }
    __syncthreads();
    if (tid == 0) S::flush_counters(P);
}

// ---- K7 for 4-byte keys-only sorts: leaves of up to BIG_BASE - 4 = 24572 keys ------------------------
// One CTA of 1024 threads per SM; a leaf lives in registers (BIG_BASE / 1024 = 24 keys per thread) while it is bucketed:
//   1. ordered image, block min/max; a constant leaf is already sorted (copied to A if it is in B);
//   2. bucket(x) = hi32(((x - min) << clz(range)) * F), a monotone map onto 8192 buckets; a shared-memory
//      atomic gives every key its slot, one block scan turns counts into (start, count) words;
//   3. keys go to kc[start + slot]; a key whose bucket holds other keys is ranked among them (number
//      of smaller keys, ties by slot), every other key keeps its slot; the result goes to kd at the
//      16-byte phase of the leaf's place in A and leaves by one TMA bulk store.
// A leaf with a bucket larger than CMAX takes the slow path: such a bucket is accepted if it is
// constant (repeated keys), otherwise the leaf is sorted by stable 8-bit LSD radix passes over
// (key - min).  On the fast path the next leaf's loads fly while the current one is ranked.
// Replaces insertion_sort / unguarded_insertion_sort (small_sorts.py:16-73) with a 24K-key leaf, which
// removes the two to three deepest partition levels of a 2^28-key sort (2^28 / 2^14 = 16384-key segments
// are leaves whatever the sampling noise of their pivots).
#ifndef PDQ_BIG_SKIP
#define PDQ_BIG_SKIP 0  // profiling builds only: 1 = no in-bucket ranking (output NOT sorted)
#endif
#ifdef PDQ_BIG_PHASES
// profiling builds (tools/leaf_phases.py): thread 0 of k_base_big charges the cycles of leaf phase i to
// one of the scheduler counters (k_sort's own uses of them are compiled out): 0 load + min/max,
// 1 slots + scan, 2 scatter, 3 ranking + store
#define PHASE_MARK(i)                                                                                  \
    do {                                                                                               \
        if (threadIdx.x == 0) {                                                                        \
            const long long t_ = clock64();                                                            \
            unsigned long long *c_[4] = {&sh.s_sch_retire, &sh.s_sch_claim, &sh.s_sch_fetch, &sh.s_sch_idle}; \
            *c_[i] += t_ - pm;                                                                         \
            pm = t_;                                                                                   \
        }                                                                                              \
    } while (0)
#else
#define PHASE_MARK(i) \
    do {              \
    } while (0)
#endif
template <bool FLOAT>
struct BigLeaf {
    using U = uint32_t;
    using O = Ord<U, FLOAT>;
    static constexpr int BT = 1024, BW = BT / 32, BI = BIG_BASE / BT;
    static_assert(BIG_BASE % (4 * BT) == 0, "a leaf is read as 16-byte vectors: BIG_BASE = 4096 k");
#ifndef PDQ_BIG_LOGBK
#define PDQ_BIG_LOGBK 13
#endif
    static constexpr int LOG_BK = PDQ_BIG_LOGBK, BBK = 1 << LOG_BK;  // buckets
    static constexpr int CMAX = 32;                       // largest bucket ranked by comparisons
    static constexpr int KD_OFF = BIG_BASE, CNT_OFF = KD_OFF + BIG_BASE + 16, RED_OFF = CNT_OFF + BBK,
                         WORDS = RED_OFF + 128;
    __host__ __device__ static constexpr int bytes() { return WORDS * 4; }
    __device__ __forceinline__ static uint32_t *wd() { return reinterpret_cast<uint32_t *>(g_dsm); }
    __device__ __forceinline__ static void bsync() { asm volatile("bar.sync 1, %0;" ::"n"(BT) : "memory"); }
    __device__ __forceinline__ static int bsync_or(int p) {
        int r;
        asm volatile(
            "{\n .reg .pred a, b;\n setp.ne.s32 a, %1, 0;\n bar.red.or.pred b, 1, %2, a;\n selp.s32 %0, 1, 0, b;\n}\n"
            : "=r"(r)
            : "r"(p), "n"(BT)
            : "memory");
        return r;
    }
    __device__ __forceinline__ static uint32_t warp_incl_scan(uint32_t v) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        return v;
    }
    // exclusive block scan of one value per thread, and the block max of `mx` (red[0, 64) scratch;
    // contains a barrier)
    __device__ __forceinline__ static uint32_t block_excl_scan(uint32_t v, uint32_t *red, uint32_t mx = 0,
                                                               uint32_t *bmax = nullptr) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const uint32_t inc = warp_incl_scan(v);
        if (bmax) mx = __reduce_max_sync(0xffffffffu, mx);
        if (lane == 31) red[warp] = inc;
        if (bmax && lane == 0) red[32 + warp] = mx;
        bsync();
        const uint32_t t = warp_incl_scan(red[lane]);
        if (bmax) *bmax = __reduce_max_sync(0xffffffffu, red[32 + lane]);
        const uint32_t wpre = __shfl_sync(0xffffffffu, t, (warp + 31) & 31);
        return (warp ? wpre : 0u) + inc - v;
    }

    // Register j of thread t holds leaf element eidx(j) = 4 ((j / 4) BT + t) + j % 4 - (b mod 4): the
    // leaf is read as 16-byte vectors from its 16-byte-aligned base (a quarter of the load
    // instructions of a scalar layout); slots outside [0, m) are padding.
    __device__ __forceinline__ static int eidx(int j, int off) {
        return 4 * ((j >> 2) * BT + (int)threadIdx.x) + (j & 3) - off;
    }
    __device__ __forceinline__ static void load(const Params &P, uint64_t lf, U (&xs)[BI]) {
        const int tid = threadIdx.x;
        const int m = lf == ~0ull ? 0 : (int)((lf >> 1) & 0x7FFF) + 1;
        PDQ_CHECK(m <= BIG_BASE - 3, "leaf fits the vector layout (m + b mod 4 <= BIG_BASE)");
        const int64_t b = (int64_t)(lf >> 16);
        const int off = (int)(b & 3);
        const U *src = (const U *)((lf & 1u) ? P.b_keys : P.a_keys) + (b - off);
        const int64_t room = P.n - (b - off);  // elements readable from the aligned base
#pragma unroll
        for (int jv = 0; jv < BI / 4; ++jv) {
            const int e0 = 4 * (jv * BT + tid);  // first slot of this vector (before the offset)
            uint4 v = make_uint4(0, 0, 0, 0);
            if (m > 0 && e0 < off + m && e0 + 4 > off) {  // the vector holds an element of the leaf
                PDQ_CHECK((b - off) + e0 >= 0 && (b - off) + e0 < P.n, "leaf vector load in the array");
                if (e0 + 4 <= room) {
                    v = __ldcg(reinterpret_cast<const uint4 *>(src + e0));
                } else {  // the array's last partial vector: scalar reads
                    v.x = ldcg(src + e0);
                    if (e0 + 1 < room) v.y = ldcg(src + e0 + 1);
                    if (e0 + 2 < room) v.z = ldcg(src + e0 + 2);
                }
            }
            xs[4 * jv] = v.x;
            xs[4 * jv + 1] = v.y;
            xs[4 * jv + 2] = v.z;
            xs[4 * jv + 3] = v.w;
        }
    }

    // the monotone bucket map of a leaf: hi32(((x - mn) << sh) * F)
    struct Map {
        U mn;
        int sh;
        uint32_t F;
        __device__ __forceinline__ uint32_t operator()(U x) const { return __umulhi((x - mn) << sh, F); }
    };
    __device__ __forceinline__ static Map make_map(U mn, U range) {
        Map mp;
        mp.mn = mn;
        mp.sh = __clz(range);                 // range > 0
        const uint32_t ymax = range << mp.sh;  // in [2^31, 2^32)
        // F <= 2^(32 + LOG_BK) / (ymax + 1) keeps every bucket below BBK (the float quotient is at most
        // one unit high; the subtraction makes it safe)
        mp.F = (uint32_t)__fdividef((float)(1ull << (32 + LOG_BK)), (float)ymax + 1.0f) - 2u;
        return mp;
    }

    // rank of key x (at slot position p of kc) inside its bucket (start | count << 16)
    __device__ __forceinline__ static uint32_t rank_in_bucket(const uint32_t *kc, U x, uint32_t p, uint32_t sc) {
        const uint32_t s0 = sc & 0xFFFFu, c = sc >> 16;
        if (PDQ_BIG_SKIP || c <= 1) return p;
        // four independent loads per step (the bucket's neighbours beyond s0 + c are read but not counted)
        uint32_t r = s0;
        const uint32_t e = s0 + c;
        for (uint32_t i = s0; i < e; i += 4) {
            U y[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) y[q] = kc[i + q];
#pragma unroll
            for (int q = 0; q < 4; ++q) r += (i + q < e) & ((y[q] < x) | ((y[q] == x) & (i + q < p)));
        }
        return r;
    }

    // One stable 8-bit counting pass src -> dst over ((x - mn) >> shift) & 255 (ordered images); the
    // final pass writes raw keys.  Warp w owns elements [32 BI w, 32 BI (w + 1)) in BI rounds of 32; ranks
    // within a warp from a ballot multisplit, per-warp 16-bit digit counters, one digit-major block scan.
    __device__ __forceinline__ static void radix_pass(const uint32_t *src, uint32_t *dst, int m, U mn, int shift,
                                                      bool fin) {
        const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
        uint16_t *wc16 = reinterpret_cast<uint16_t *>(wd() + CNT_OFF);
        uint16_t *wc = wc16 + warp * 256;
        uint32_t *red = wd() + RED_OFF;
        reinterpret_cast<uint4 *>(wc)[lane] = make_uint4(0u, 0u, 0u, 0u);  // 256 counters
        __syncwarp();
        const unsigned ltm = lanemask_lt();
        uint32_t rd[BI];
#pragma unroll
        for (int j = 0; j < BI; ++j) {
            const int idx = warp * (32 * BI) + j * 32 + lane;
            const bool valid = idx < m;
            const uint32_t d = valid ? ((src[idx] - mn) >> shift) & 255u : 0u;
            unsigned peers = __ballot_sync(0xffffffffu, valid);
            peers = valid ? peers : ~peers;
#pragma unroll
            for (int bit = 0; bit < 8; ++bit) {
                const bool on = (d >> bit) & 1u;
                const unsigned bb = __ballot_sync(0xffffffffu, on);
                peers &= on ? bb : ~bb;
            }
            const uint32_t before = valid ? (uint32_t)wc[d] : 0u;
            const uint32_t r = (uint32_t)__popc(peers & ltm);
            __syncwarp();
            if (valid && r == 0) wc[d] = (uint16_t)(before + __popc(peers));
            __syncwarp();
            rd[j] = ((before + r) << 8) | d;
        }
        bsync();
        // digit-major scan over (digit, warp): thread t owns digit t >> 2, warps 8 (t & 3) .. + 8
        {
            const int d = tid >> 2, w0 = 8 * (tid & 3);
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c[q] = wc16[(w0 + q) * 256 + d];
                tot += c[q];
            }
            uint32_t run = block_excl_scan(tot, red);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                wc16[(w0 + q) * 256 + d] = (uint16_t)run;
                run += c[q];
            }
        }
        bsync();
#pragma unroll
        for (int j = 0; j < BI; ++j) {
            const int idx = warp * (32 * BI) + j * 32 + lane;
            if (idx < m) {
                const uint32_t pos = (uint32_t)wc[rd[j] & 0xFFu] + (rd[j] >> 8);
                const U x = src[idx];
                dst[pos] = fin ? O::from(x) : x;
            }
        }
        bsync();
    }

    // Slow path (a bucket holds more than CMAX keys).  kc holds the bucketed leaf and cnt the
    // (start, count) words; writes kd[a0 + i] = raw keys in order.
    __device__ __noinline__ static void slow_leaf(int m, int a0, const Map mp, U range) {
        const int tid = threadIdx.x;
        uint32_t *kc = wd(), *kd = wd() + KD_OFF, *cnt = wd() + CNT_OFF;
        int fb = 0;
#pragma unroll
        for (int j = 0; j < BI; ++j) {
            if (j * BT + tid < m) {
                const uint32_t p = j * BT + tid;
                const U x = kc[p];
                const uint32_t sc = cnt[mp(x)];
                if ((sc >> 16) > (uint32_t)CMAX && kc[sc & 0xFFFFu] != x) fb = 1;  // a big mixed bucket
            }
        }
        if (!bsync_or(fb)) {
            // every big bucket is constant: its keys keep their slots, the others are ranked
#pragma unroll
            for (int j = 0; j < BI; ++j) {
                if (j * BT + tid < m) {
                    const uint32_t p = j * BT + tid;
                    const U x = kc[p];
                    const uint32_t sc = cnt[mp(x)];
                    const uint32_t r = (sc >> 16) > (uint32_t)CMAX ? p : rank_in_bucket(kc, x, p, sc);
                    kd[a0 + r] = O::from(x);
                }
            }
            return;
        }
        // clustered distinct keys: LSD radix passes over (key - mn); the final pass reads kc, writes kd
        const int np = (32 - __clz(range) + 7) / 8;
        const uint32_t *src = kc;
        uint32_t *dst = kd;
        if ((np & 1) == 0) {
            for (int i = tid; i < m; i += BT) kd[i] = kc[i];
            bsync();
            src = kd;
            dst = kc;
        }
        for (int q = 0; q < np; ++q) {
            const bool fin = q == np - 1;
            radix_pass(src, fin ? kd + a0 : dst, m, mp.mn, 8 * q, fin);
            const uint32_t *t = src;
            src = dst;
            dst = const_cast<uint32_t *>(t);
        }
    }

    // ---- fast path: window networks over a swizzled kc ----------------------------------------------
    // Positions are in q-space: q = a0 + leaf position, a0 = b mod 4, so q and the leaf's global index
    // have the same 16-byte phase.  Row t = [24t, 24t + 24) is thread t's window.  Linear 16-byte chunk c
    // (= q / 4) lives at chunk c ^ ((c >> 3) & 1): the 8 lanes of a quarter-warp then hit 8 distinct bank
    // groups whether they read chunk j of their own rows, chunk j of the next rows, or 8 consecutive
    // chunks (checked exhaustively for every access pattern here); a row-rotation needs a division by 24.
    static constexpr int WIN = 24, HALF = WIN / 2;
    static constexpr uint32_t FAST_CMAX = HALF + 1;  // every bucket fits an aligned or an offset window
    static_assert(BIG_BASE == WIN * BT, "one window per thread");
    __device__ __forceinline__ static uint32_t swz(uint32_t q) { return q ^ ((q >> 3) & 4u); }
    __device__ __forceinline__ static uint32_t swz_chunk(uint32_t t, uint32_t j) { return swz(WIN * t + 4u * j); }
    __device__ __forceinline__ static void ld_chunk(const uint32_t *s, U *w) {
        const uint4 v = *reinterpret_cast<const uint4 *>(s);
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    }
    __device__ __forceinline__ static void st_chunk(uint32_t *s, const U *w) {
        *reinterpret_cast<uint4 *>(s) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    // Sort the bucketed leaf kc[q], q in [a0, qend) (swizzled), and store it to dst[q - a0] (global):
    //   pass 1: thread t sorts window [24t, 24t + 24) with a 132-comparator network;
    //   pass 2: thread t merges the two sorted halves of the offset window [24t + 12, 24t + 36) (45
    //           comparators) and writes it back to the same (swizzled) chunks it read -- windows are
    //           disjoint, so no barrier separates its loads from its stores;
    //   copy-out: consecutive threads read consecutive 16-byte chunks in linear order and store them to
    //           global memory (raw keys), 512 contiguous bytes per warp instruction.
    // Each element only moves inside its bucket; a bucket of <= 13 keys lies in one aligned or one offset
    // window, so after the two passes every bucket -- and so the leaf -- is in order.  Slots q < a0 read
    // as 0 (below every key), q >= qend as ~0 (above every key); neither is ever stored.
    // `sorted`: the bucketed leaf is already in order (every bucket holds one distinct key): copy-out only
    __device__ __forceinline__ static void window_sort(uint32_t *kc, uint32_t a0, uint32_t qend, U *dst, bool sorted) {
        const uint32_t t = threadIdx.x;
        if (!sorted && WIN * t < qend) {
            U w[WIN];
#pragma unroll
            for (int j = 0; j < 6; ++j) ld_chunk(kc + swz_chunk(t, j), w + 4 * j);
            if (WIN * t < a0 || WIN * t + WIN > qend) {  // the leaf's first / last window only
#pragma unroll
                for (int i = 0; i < WIN; ++i) {
                    const uint32_t q = WIN * t + i;
                    w[i] = q < a0 ? 0u : (q >= qend ? ~0u : w[i]);
                }
            }
            net_sort24(w);
#pragma unroll
            for (int j = 0; j < 6; ++j) st_chunk(kc + swz_chunk(t, j), w + 4 * j);
        }
        if (!sorted) bsync();
        if (!sorted && WIN * t + HALF < qend) {
            U w[WIN];
            const bool second = WIN * (t + 1) < qend;
#pragma unroll
            for (int j = 0; j < 3; ++j) ld_chunk(kc + swz_chunk(t, j + 3), w + 4 * j);
            if (second) {
#pragma unroll
                for (int j = 0; j < 3; ++j) ld_chunk(kc + swz_chunk(t + 1, j), w + HALF + 4 * j);
            } else {
#pragma unroll
                for (int i = HALF; i < WIN; ++i) w[i] = ~0u;
            }
            if (WIN * t + HALF + WIN > qend) {
#pragma unroll
                for (int i = HALF; i < WIN; ++i) {
                    const uint32_t q = WIN * t + HALF + i;
                    w[i] = q >= qend ? ~0u : w[i];
                }
            }
            net_merge12(w);
#pragma unroll
            for (int j = 0; j < 3; ++j) st_chunk(kc + swz_chunk(t, j + 3), w + 4 * j);
            if (second) {
#pragma unroll
                for (int j = 0; j < 3; ++j) st_chunk(kc + swz_chunk(t + 1, j), w + HALF + 4 * j);
            }
        }
        bsync();
        // copy-out: linear chunk c = q / 4; dst + (4c - a0) is 16-byte aligned
        const uint32_t nch = (qend + 3) / 4;
        for (uint32_t c = t; c < nch; c += BT) {
            U v[4];
            ld_chunk(kc + swz(4u * c), v);
            const uint32_t q = 4 * c;
            if (q >= a0 && q + 4 <= qend) {
                *reinterpret_cast<uint4 *>(dst + (q - a0)) = make_uint4(O::from(v[0]), O::from(v[1]), O::from(v[2]),
                                                                        O::from(v[3]));
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (q + e >= a0 && q + e < qend) dst[q + e - a0] = O::from(v[e]);
            }
        }
    }

    // thread 0: TMA bulk load of leaf `lf` into kd (from its 16-byte aligned base; the array's last
    // partial vector by scalar loads), completing on `bar`
    __device__ __forceinline__ static void prefetch(const Params &P, uint64_t lf, uint32_t *kd, uint64_t *bar) {
        const int m = (int)((lf >> 1) & 0x7FFF) + 1;
        const int64_t b = (int64_t)(lf >> 16);
        const int off = (int)(b & 3);
        const int64_t base = b - off;
        const U *src = (const U *)((lf & 1u) ? P.b_keys : P.a_keys) + base;
        const int64_t vec = ((int64_t)(off + m) + 3) & ~(int64_t)3;
        const int64_t room = P.n - base;
        const int64_t bulk = vec < (room & ~(int64_t)3) ? vec : (room & ~(int64_t)3);
        for (int64_t e = bulk; e < vec && e < room; ++e) kd[e] = ldcg(src + e);
        fence_proxy_async();
        mbar_expect_tx(bar, (unsigned)(bulk * 4));
        if (bulk > 0) bulk_g2s(kd, src, (unsigned)(bulk * 4), bar);
    }
    // every thread: its registers of leaf `lf` from kd (the register layout of load())
    __device__ __forceinline__ static void read_kd(const uint32_t *kd, uint64_t lf, U (&xs)[BI]) {
        const int tid = threadIdx.x;
        const int m = (int)((lf >> 1) & 0x7FFF) + 1;
        const int off = (int)((lf >> 16) & 3);
#pragma unroll
        for (int jv = 0; jv < BI / 4; ++jv) {
            const int e0 = 4 * (jv * BT + tid);
            uint4 v = make_uint4(0, 0, 0, 0);
            if (e0 < off + m) v = *reinterpret_cast<const uint4 *>(kd + e0);
            xs[4 * jv] = v.x;
            xs[4 * jv + 1] = v.y;
            xs[4 * jv + 2] = v.z;
            xs[4 * jv + 3] = v.w;
        }
    }

    __device__ static void run(const Params &P) {
        // Per-leaf scalars that only thread 0 needs (descriptors ahead, counters) live in shared memory:
        // with 1024 threads every register is precious (24 keys + 12 packed slots per thread).
        Shared &sh = g_sh;
        const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
        uint32_t *kc = wd(), *kd = wd() + KD_OFF, *cnt = wd() + CNT_OFF, *red = wd() + RED_OFF;
        constexpr uint64_t NONE = ~0ull;
        uint64_t *bar = &sh.bar[0];
        auto claim = [&]() -> uint64_t {  // thread 0
            unsigned long long count = *(volatile unsigned long long *)&P.st->leaf_count;
            if (count > P.leaf_cap) count = P.leaf_cap;
            const unsigned long long idx = atomicAdd(&P.st->leaf_next, 1ull);
            return idx < count ? ldcg(P.leaves + idx) : NONE;
        };
        if (tid == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            sh.lq[0] = claim();  // one leaf per CTA first: a small sort spreads over every SM
            if (sh.lq[0] != NONE) prefetch(P, sh.lq[0], kd, bar);
        }
        bsync();
        U xs[BI];
        unsigned kphase = 0;
        long long pm = clock64();  // (PDQ_BIG_PHASES profiling builds)
        for (;;) {
            const uint64_t cur = sh.lq[0];
            if (cur == NONE) break;
            if (tid == 0) {
                sh.lc0 = clock64();
                sh.lq[1] = claim();  // the next leaf: prefetched once this one has left kd
            }
            pm = clock64();
            mbar_wait(bar, kphase);
            kphase ^= 1u;
            read_kd(kd, cur, xs);
            const int m = (int)((cur >> 1) & 0x7FFF) + 1;
            const int64_t b = (int64_t)(cur >> 16);
            const bool srcB = cur & 1u;
            {  // zero the bucket counters
                uint4 *c4 = reinterpret_cast<uint4 *>(cnt);
#pragma unroll
                for (int q = 0; q < BBK / 4 / BT; ++q) c4[q * BT + tid] = make_uint4(0, 0, 0, 0);
            }
            const int off = (int)(b & 3);
            // vector jv of a thread holds leaf elements e0 .. e0 + 3, e0 = 4 (jv BT + t) - off: a vector is
            // whole, partial (the leaf's ends) or empty; vectors jv with 4 jv BT >= off + m are empty in
            // every thread (a CTA-uniform loop bound)
            const int nvec = (off + m + 4 * BT - 1) / (4 * BT);
            U mn = ~0u, mx = 0u;
#pragma unroll
            for (int jv = 0; jv < BI / 4; ++jv) {
                if (jv < nvec) {
                    const int e0 = 4 * (jv * BT + tid) - off;
                    const bool whole = e0 >= 0 && e0 + 4 <= m;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (whole || (unsigned)(e0 + q) < (unsigned)m) {
                            const U x = O::to(xs[4 * jv + q]);
                            xs[4 * jv + q] = x;
                            mn = min(mn, x);
                            mx = max(mx, x);
                        }
                    }
                }
            }
            mn = __reduce_min_sync(0xffffffffu, mn);
            mx = __reduce_max_sync(0xffffffffu, mx);
            if (lane == 0) {
                red[64 + warp] = mn;
                red[96 + warp] = mx;
            }
            bsync();  // kd has been read by every thread: the next leaf's load may land in it
            if (tid == 0 && sh.lq[1] != NONE) prefetch(P, sh.lq[1], kd, bar);
            PHASE_MARK(0);
            mn = __reduce_min_sync(0xffffffffu, red[64 + lane]);
            mx = __reduce_max_sync(0xffffffffu, red[96 + lane]);
            const U range = mx - mn;
            if (range == 0) {
                // a constant leaf is sorted; one in B is copied to its place in A
                if (srcB) {
                    U *a = (U *)P.a_keys + b;
#pragma unroll
                    for (int j = 0; j < BI; ++j)
                        if ((unsigned)eidx(j, off) < (unsigned)m) a[eidx(j, off)] = O::from(xs[j]);
                }
                bsync();  // every thread has read lq[0] and lq[1]
                if (tid == 0) {
                    sh.lq[0] = sh.lq[1];
                    sh.s_base++;
                    sh.s_bytes += (srcB ? 2ull : 1ull) * 4 * m;
                    sh.s_cyc_base += clock64() - sh.lc0;
                }
                bsync();
                continue;
            }
            const Map mp = make_map(mn, range);
            uint32_t pp[BI / 2];  // 16-bit slots
#pragma unroll
            for (int jv = 0; jv < BI / 4; ++jv) {
                pp[2 * jv] = pp[2 * jv + 1] = 0;
                if (jv < nvec) {
                    const int e0 = 4 * (jv * BT + tid) - off;
                    const bool whole = e0 >= 0 && e0 + 4 <= m;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int j = 4 * jv + q;
                        if (whole || (unsigned)(e0 + q) < (unsigned)m) pp[j / 2] |= atomicAdd(&cnt[mp(xs[j])], 1u) << ((j & 1) << 4);
                    }
                }
            }
            bsync();
            uint32_t cmax;
            {  // (start, count) words: thread t owns buckets [PB t, PB t + PB), scanned in two halves
                constexpr int PB = BBK / BT;
                uint4 *c4 = reinterpret_cast<uint4 *>(cnt + PB * tid);
                uint32_t tot = 0, mc = 0;
#pragma unroll
                for (int q = 0; q < PB / 4; ++q) {
                    const uint4 y = c4[q];
                    tot += y.x + y.y + y.z + y.w;
                    mc = max(mc, max(max(y.x, y.y), max(y.z, y.w)));
                }
                uint32_t run = block_excl_scan(tot, red, mc, &cmax);
#pragma unroll
                for (int q = 0; q < PB / 4; ++q) {
                    const uint4 y = c4[q];
                    uint4 o;
                    o.x = run | (y.x << 16); run += y.x;
                    o.y = run | (y.y << 16); run += y.y;
                    o.z = run | (y.z << 16); run += y.z;
                    o.w = run | (y.w << 16); run += y.w;
                    c4[q] = o;
                }
            }
            if (tid == 0) bulk_wait_read();  // the previous leaf's bulk store has left kc
            bsync();
            PHASE_MARK(1);
            const uint32_t a0 = (uint32_t)(b & 3);
            // A leaf spanning fewer than BBK / 2 distinct key values has at most one value per bucket (the
            // map advances by more than one bucket per key step), so bucketing alone sorts it: float32 keys
            // at 2^26+ (2^23 values per binade), low-cardinality integers
            const bool exact = range < (U)(BBK / 2);
            const bool fast = PDQ_BIG_SKIP || exact || cmax <= FAST_CMAX;
#pragma unroll
            for (int jv = 0; jv < BI / 4; ++jv) {
                if (jv < nvec) {
                    const int e0 = 4 * (jv * BT + tid) - off;
                    const bool whole = e0 >= 0 && e0 + 4 <= m;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int j = 4 * jv + q;
                        if (whole || (unsigned)(e0 + q) < (unsigned)m) {
                            PDQ_CHECK(mp(xs[j]) < (uint32_t)BBK, "leaf bucket");
                            const uint32_t p = (cnt[mp(xs[j])] & 0xFFFFu) + ((pp[j / 2] >> ((j & 1) << 4)) & 0xFFFFu);
                            PDQ_CHECK(p < (uint32_t)m, "leaf scatter slot");
                            kc[fast ? swz(a0 + p) : p] = xs[j];
                        }
                    }
                }
            }
            bsync();
            PHASE_MARK(2);
            if (fast) {
                window_sort(kc, a0, a0 + (uint32_t)m, (U *)P.a_keys + b, exact);
                if (tid == 0) {
                    sh.s_base++;
                    sh.s_bytes += 8ull * m;
                    sh.s_cyc_base += clock64() - sh.lc0;
                    sh.lq[0] = sh.lq[1];
                }
                PHASE_MARK(3);
                bsync();
                continue;
            }
            {
                // slow path (a bucket of > 13 keys): it needs kd, so the next leaf's prefetch is dropped
                // (after it lands) and issued again once this leaf's bulk store has read kd
                if (sh.lq[1] != NONE) {
                    mbar_wait(bar, kphase);
                    kphase ^= 1u;
                }
                bsync();
                slow_leaf(m, (int)a0, mp, range);
            }
            uint32_t *out = kd;
            fence_proxy_async();
            bsync();
            {  // out[a0, a0 + m) -> A[b, b + m): 16-byte body by one bulk store, head/tail by threads
                U *a = (U *)P.a_keys + b;
                int h = (4 - (int)a0) & 3;
                if (h > m) h = m;
                const int nb = ((m - h) / 4) * 4;
                if (tid > 0 && tid < 4 && tid - 1 < h) a[tid - 1] = out[a0 + tid - 1];
                if (tid >= 4 && tid < 8 && h + nb + tid - 4 < m) a[h + nb + tid - 4] = out[a0 + h + nb + tid - 4];
                if (tid == 0) {
                    if (nb) bulk_s2g(a + h, out + a0 + h, (unsigned)nb * 4u);
                    bulk_commit();
                    if (sh.lq[1] != NONE) {  // re-issue the dropped prefetch once kd is read
                        bulk_wait_read();
                        prefetch(P, sh.lq[1], kd, bar);
                    }
                    sh.s_base++;
                    sh.s_bytes += 8ull * m;
                    sh.s_cyc_base += clock64() - sh.lc0;
                    sh.lq[0] = sh.lq[1];
                }
            }
            PHASE_MARK(3);
            bsync();
        }
        if (tid == 0) bulk_wait_all();
        bsync();
    }
};

// ---- K7 for 8-byte keys and key-value sorts: leaves of up to 8188 elements -------------------------
// The design of BigLeaf for wider elements (1024 threads, 8 elements per thread, 4096 buckets):
// elements compare as (ordered key, payload) pairs; the bucket map reads the key (or, for a leaf of
// equal keys, the payload).  A bucket of more than CMAX elements is ranked by the same comparison loop
// over the whole bucket (quadratic in the bucket, but only clustered leaves have such buckets).  Keys and
// payloads leave by one TMA bulk store each.
template <class U, bool FLOAT, bool KV>
struct WideLeaf {
    using O = Ord<U, FLOAT>;
    using H = BigLeaf<false>;  // the 1024-thread block helpers
    static constexpr int BT = 1024, BI = 8, CAP = BT * BI;
    static constexpr int BBK = 8192, LOG_BK = 13;  // ~1 element per bucket: short, rarely divergent rank loops
    static constexpr int CMAX = 32;  // largest bucket ranked by comparisons; beyond it the leaf takes radix passes
    static constexpr int KB = (CAP + 16) * (int)sizeof(U), VB = KV ? (CAP + 16) * 4 : 0;
    static constexpr int KCK = 0, KCV = KB, KDK = KB + VB, KDV = 2 * KB + VB, CNT = 2 * KB + 2 * VB,
                         RED = CNT + BBK * 4;
    __host__ __device__ static constexpr int bytes() { return RED + 1024; }
    __device__ __forceinline__ static U *kck() { return reinterpret_cast<U *>(g_dsm + KCK); }
    __device__ __forceinline__ static uint32_t *kcv() { return reinterpret_cast<uint32_t *>(g_dsm + KCV); }
    __device__ __forceinline__ static U *kdk() { return reinterpret_cast<U *>(g_dsm + KDK); }
    __device__ __forceinline__ static uint32_t *kdv() { return reinterpret_cast<uint32_t *>(g_dsm + KDV); }
    __device__ __forceinline__ static uint32_t *cnt() { return reinterpret_cast<uint32_t *>(g_dsm + CNT); }
    __device__ __forceinline__ static uint64_t *red() { return reinterpret_cast<uint64_t *>(g_dsm + RED); }

    // register j of thread t holds leaf element 4 ((j / 4) BT + t) + j % 4 - (b mod 4) (16-byte vectors)
    __device__ __forceinline__ static int eidx(int j, int off) {
        return 4 * ((j >> 2) * BT + (int)threadIdx.x) + (j & 3) - off;
    }
    __device__ __forceinline__ static bool less(U a, uint32_t va, U b, uint32_t vb) {
        return a < b || (KV && a == b && va < vb);
    }
    __device__ __forceinline__ static U shfl_x(U x, int o) {
        if constexpr (sizeof(U) == 4) return (U)__shfl_xor_sync(0xffffffffu, (uint32_t)x, o);
        return (U)__shfl_xor_sync(0xffffffffu, (unsigned long long)x, o);
    }

    // One stable 8-bit counting pass over digit ((payload or key) - base) >> shift: warp w owns elements
    // [256w, 256w + 256) in 8 rounds of 32, ranks from a ballot multisplit, per-warp 16-bit counters,
    // one digit-major block scan.  The final pass writes raw keys to kd/vd at a0.
    __device__ __forceinline__ static void radix_pass(const U *sk, const uint32_t *sv, U *dk, uint32_t *dv, int m,
                                                      bool on_vals, uint64_t base, int shift, bool fin) {
        const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
        uint16_t *wc16 = reinterpret_cast<uint16_t *>(cnt());
        uint16_t *wc = wc16 + warp * 256;
        uint32_t *scr = reinterpret_cast<uint32_t *>(red()) + 128;
        reinterpret_cast<uint4 *>(wc)[lane] = make_uint4(0u, 0u, 0u, 0u);  // 256 counters
        __syncwarp();
        const unsigned ltm = lanemask_lt();
        uint32_t rdg[BI];
#pragma unroll
        for (int j = 0; j < BI; ++j) {
            const int idx = warp * (32 * BI) + j * 32 + lane;
            const bool valid = idx < m;
            const uint64_t src = valid ? (on_vals ? (uint64_t)sv[idx] : (uint64_t)sk[idx]) : 0ull;
            const uint32_t d = valid ? (uint32_t)((src - base) >> shift) & 255u : 0u;
            unsigned peers = __ballot_sync(0xffffffffu, valid);
            peers = valid ? peers : ~peers;
#pragma unroll
            for (int bit = 0; bit < 8; ++bit) {
                const bool on = (d >> bit) & 1u;
                const unsigned bb = __ballot_sync(0xffffffffu, on);
                peers &= on ? bb : ~bb;
            }
            const uint32_t before = valid ? (uint32_t)wc[d] : 0u;
            const uint32_t r = (uint32_t)__popc(peers & ltm);
            __syncwarp();
            if (valid && r == 0) wc[d] = (uint16_t)(before + __popc(peers));
            __syncwarp();
            rdg[j] = ((before + r) << 8) | d;
        }
        H::bsync();
        {  // digit-major scan over (digit, warp): thread t owns digit t >> 2, warps 8 (t & 3) .. + 8
            const int d = tid >> 2, w0 = 8 * (tid & 3);
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c[q] = wc16[(w0 + q) * 256 + d];
                tot += c[q];
            }
            uint32_t run = H::block_excl_scan(tot, scr);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                wc16[(w0 + q) * 256 + d] = (uint16_t)run;
                run += c[q];
            }
        }
        H::bsync();
#pragma unroll
        for (int j = 0; j < BI; ++j) {
            const int idx = warp * (32 * BI) + j * 32 + lane;
            if (idx < m) {
                const uint32_t pos = (uint32_t)wc[rdg[j] & 0xFFu] + (rdg[j] >> 8);
                const U x = sk[idx];
                dk[pos] = fin ? O::from(x) : x;
                if constexpr (KV) dv[pos] = sv[idx];
            }
        }
        H::bsync();
    }
    // kc/vc[0, m) -> kd/vd[a0 + i] in (key, payload) order: LSD passes over the payload digits, then
    // the key digits (both range-reduced); the final pass reads kc and writes kd
    __device__ __noinline__ static void radix_leaf(int m, int a0, U kmn, U krange, uint32_t vmn, uint32_t vrange) {
        U *kc = kck(), *kd = kdk();
        uint32_t *vc = kcv(), *vd = kdv();
        const int vb = (KV && vrange) ? 32 - __clz(vrange) : 0;
        const int kb = krange ? 8 * (int)sizeof(U) - (sizeof(U) == 4 ? __clz((uint32_t)krange) : __clzll((long long)krange)) : 0;
        const int npv = (vb + 7) / 8, npk = (kb + 7) / 8, np = npv + npk;
        const U *sk = kc;
        const uint32_t *sv = vc;
        U *dk = kd;
        uint32_t *dv = vd;
        if ((np & 1) == 0) {  // the final pass must read kc and write kd
            for (int i = threadIdx.x; i < m; i += BT) {
                kd[i] = kc[i];
                if constexpr (KV) vd[i] = vc[i];
            }
            H::bsync();
            sk = kd; sv = vd; dk = kc; dv = vc;
        }
        for (int q = 0; q < np; ++q) {
            const bool fin = q == np - 1, on_vals = q < npv;
            radix_pass(sk, sv, fin ? kd + a0 : dk, fin ? vd + a0 : dv, m, on_vals, on_vals ? (uint64_t)vmn : (uint64_t)kmn,
                       8 * (on_vals ? q : q - npv), fin);
            const U *tk = sk;
            const uint32_t *tv = sv;
            sk = dk; sv = dv;
            dk = const_cast<U *>(tk); dv = const_cast<uint32_t *>(tv);
        }
    }

    // thread 0: TMA bulk loads of leaf `lf` (keys, and payloads) into kd / vd from its 16-byte aligned base
    // (4-element granularity keeps both arrays' copies multiples of 16 bytes; the array's last partial
    // vector by scalar loads), completing on `bar`
    __device__ __forceinline__ static void prefetch(const Params &P, uint64_t lf, uint64_t *bar) {
        const int m = (int)((lf >> 1) & 0x7FFF) + 1;
        const int64_t b = (int64_t)(lf >> 16);
        const int off = (int)(b & 3);
        const int64_t base = b - off;
        const U *src = (const U *)((lf & 1u) ? P.b_keys : P.a_keys) + base;
        const uint32_t *srcv = KV ? ((lf & 1u) ? P.b_vals : P.a_vals) + base : nullptr;
        U *kd = kdk();
        uint32_t *vd = kdv();
        const int64_t vec = ((int64_t)(off + m) + 3) & ~(int64_t)3;
        const int64_t room = P.n - base;
        const int64_t bulk = vec < (room & ~(int64_t)3) ? vec : (room & ~(int64_t)3);
        for (int64_t e = bulk; e < vec && e < room; ++e) {
            kd[e] = ldcg(src + e);
            if constexpr (KV) vd[e] = ldcg(srcv + e);
        }
        fence_proxy_async();
        mbar_expect_tx(bar, (unsigned)(bulk * (int64_t)(sizeof(U) + (KV ? 4 : 0))));
        if (bulk > 0) {
            bulk_g2s(kd, src, (unsigned)(bulk * sizeof(U)), bar);
            if constexpr (KV) bulk_g2s(vd, srcv, (unsigned)(bulk * 4), bar);
        }
    }
    // every thread: its registers of leaf `lf` from kd / vd (the 16-byte vector layout of eidx)
    __device__ __forceinline__ static void read_kd(uint64_t lf, U (&xs)[BI], uint32_t (&vs)[BI]) {
        const int tid = threadIdx.x;
        const int m = (int)((lf >> 1) & 0x7FFF) + 1;
        const int off = (int)((lf >> 16) & 3);
        const U *kd = kdk();
        const uint32_t *vd = kdv();
#pragma unroll
        for (int jv = 0; jv < BI / 4; ++jv) {
            const int e0 = 4 * (jv * BT + tid);
            U k4[4] = {0, 0, 0, 0};
            uint32_t v4[4] = {0, 0, 0, 0};
            if (e0 < off + m) {
                if constexpr (sizeof(U) == 4) {
                    const uint4 y = *reinterpret_cast<const uint4 *>(kd + e0);
                    k4[0] = (U)y.x; k4[1] = (U)y.y; k4[2] = (U)y.z; k4[3] = (U)y.w;
                } else {
                    const ulonglong2 y0 = *reinterpret_cast<const ulonglong2 *>(kd + e0);
                    const ulonglong2 y1 = *reinterpret_cast<const ulonglong2 *>(kd + e0 + 2);
                    k4[0] = (U)y0.x; k4[1] = (U)y0.y; k4[2] = (U)y1.x; k4[3] = (U)y1.y;
                }
                if constexpr (KV) {
                    const uint4 z = *reinterpret_cast<const uint4 *>(vd + e0);
                    v4[0] = z.x; v4[1] = z.y; v4[2] = z.z; v4[3] = z.w;
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                xs[4 * jv + q] = k4[q];
                vs[4 * jv + q] = v4[q];
            }
        }
    }

    // Leaves of <= CAP - 4 elements, one per CTA at a time: the next leaf is prefetched into kd / vd by
    // TMA while the current one is bucketed into kc / vc (at q = a0 + position, a0 = b mod 4, the 16-byte
    // phase of the leaf in A), ranked in place inside its bucket (keys + payloads held in registers
    // across one barrier) and copied out to A by consecutive threads in 16-byte chunks.  A leaf with a
    // bucket of more than CMAX elements (e.g. argsort of low-cardinality keys) takes stable LSD radix
    // passes (they use kd, so the prefetch is waited for and issued again afterwards).
    __device__ static void run(const Params &P) {
        Shared &sh = g_sh;
        const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
        U *kc = kck();
        uint32_t *vc = kcv(), *cn = cnt();
        uint64_t *rd = red();
        constexpr uint64_t NONE = ~0ull;
        uint64_t *bar = &sh.bar[0];
        auto claim = [&]() -> uint64_t {  // thread 0
            unsigned long long count = *(volatile unsigned long long *)&P.st->leaf_count;
            if (count > P.leaf_cap) count = P.leaf_cap;
            const unsigned long long idx = atomicAdd(&P.st->leaf_next, 1ull);
            return idx < count ? ldcg(P.leaves + idx) : NONE;
        };
        if (tid == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            sh.lq[0] = claim();
            if (sh.lq[0] != NONE) prefetch(P, sh.lq[0], bar);
        }
        H::bsync();
        unsigned kphase = 0;
        U xs[BI];
        uint32_t vs[BI];
        for (;;) {
            const uint64_t cur = sh.lq[0];
            if (cur == NONE) break;
            if (tid == 0) {
                sh.lc0 = clock64();
                sh.lq[1] = claim();
            }
            mbar_wait(bar, kphase);
            kphase ^= 1u;
            read_kd(cur, xs, vs);
            const int m = (int)((cur >> 1) & 0x7FFF) + 1;
            const int64_t b = (int64_t)(cur >> 16);
            const bool srcB = cur & 1u;
            const int off = (int)(b & 3);
            {
                uint4 *c4 = reinterpret_cast<uint4 *>(cn);
#pragma unroll
                for (int q = 0; q < BBK / 4 / BT; ++q) c4[q * BT + tid] = make_uint4(0, 0, 0, 0);
            }
            const int nvec = (off + m + 4 * BT - 1) / (4 * BT);  // vectors holding leaf elements (CTA-uniform)
            U kmn = ~(U)0, kmx = 0;
            uint32_t vmn = 0xFFFFFFFFu, vmx = 0;
#pragma unroll
            for (int jv = 0; jv < BI / 4; ++jv) {
                if (jv < nvec) {
                    const int e0 = 4 * (jv * BT + tid) - off;
                    const bool whole = e0 >= 0 && e0 + 4 <= m;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int j = 4 * jv + q;
                        if (whole || (unsigned)(e0 + q) < (unsigned)m) {
                            const U x = O::to(xs[j]);
                            xs[j] = x;
                            kmn = x < kmn ? x : kmn;
                            kmx = x > kmx ? x : kmx;
                            vmn = min(vmn, vs[j]);
                            vmx = max(vmx, vs[j]);
                        }
                    }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const U a = shfl_x(kmn, o), c = shfl_x(kmx, o);
                kmn = a < kmn ? a : kmn;
                kmx = c > kmx ? c : kmx;
            }
            vmn = __reduce_min_sync(0xffffffffu, vmn);
            vmx = __reduce_max_sync(0xffffffffu, vmx);
            if (lane == 0) {
                rd[warp] = (uint64_t)kmn;
                rd[32 + warp] = (uint64_t)kmx;
                rd[64 + warp] = vmn;
                rd[96 + warp] = vmx;
            }
            H::bsync();  // kd / vd have been read by every thread: the next leaf may land in them
            if (tid == 0 && sh.lq[1] != NONE) prefetch(P, sh.lq[1], bar);
            {  // lane q reads warp q's extremes; one warp reduction (every warp computes the same)
                kmn = (U)rd[lane];
                kmx = (U)rd[32 + lane];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const U a = shfl_x(kmn, o), c = shfl_x(kmx, o);
                    kmn = a < kmn ? a : kmn;
                    kmx = c > kmx ? c : kmx;
                }
                vmn = __reduce_min_sync(0xffffffffu, (uint32_t)rd[64 + lane]);
                vmx = __reduce_max_sync(0xffffffffu, (uint32_t)rd[96 + lane]);
            }
            const U krange = kmx - kmn;
            if (krange == 0 && (!KV || vmn == vmx)) {
                // a constant leaf is sorted; one in B is copied to its place in A
                if (srcB) {
                    U *a = (U *)P.a_keys + b;
#pragma unroll
                    for (int j = 0; j < BI; ++j)
                        if ((unsigned)eidx(j, off) < (unsigned)m) {
                            a[eidx(j, off)] = O::from(xs[j]);
                            if constexpr (KV) P.a_vals[b + eidx(j, off)] = vs[j];
                        }
                }
                H::bsync();  // every thread has read lq[0] and lq[1]
                if (tid == 0) {
                    sh.lq[0] = sh.lq[1];
                    sh.s_base++;
                    sh.s_bytes += (srcB ? 2ull : 1ull) * (sizeof(U) + (KV ? 4 : 0)) * m;
                    sh.s_cyc_base += clock64() - sh.lc0;
                }
                H::bsync();
                continue;
            }
            // bucket source: the key, or the payload when every key is equal
            const bool by_key = krange != 0;
            const uint64_t smn = by_key ? (uint64_t)kmn : (uint64_t)vmn;
            const uint64_t srange = by_key ? (uint64_t)krange : (uint64_t)(vmx - vmn);
            const int sh64 = __clzll((long long)srange);
            const uint32_t ymax = (uint32_t)((srange << sh64) >> 32);
            const uint32_t F = (uint32_t)__fdividef((float)(1ull << (32 + LOG_BK)), (float)ymax + 1.0f) - 2u;
            auto bucket = [&](U x, uint32_t v) -> uint32_t {
                const uint64_t d = (by_key ? (uint64_t)x : (uint64_t)v) - smn;
                return __umulhi((uint32_t)((d << sh64) >> 32), F);
            };
            uint32_t pp[BI / 2];
#pragma unroll
            for (int jv = 0; jv < BI / 4; ++jv) {
                pp[2 * jv] = pp[2 * jv + 1] = 0;
                if (jv < nvec) {
                    const int e0 = 4 * (jv * BT + tid) - off;
                    const bool whole = e0 >= 0 && e0 + 4 <= m;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int j = 4 * jv + q;
                        if (whole || (unsigned)(e0 + q) < (unsigned)m)
                            pp[j / 2] |= atomicAdd(&cn[bucket(xs[j], vs[j])], 1u) << ((j & 1) << 4);
                    }
                }
            }
            H::bsync();
            uint32_t cmax;
            {  // (start, count) words: thread t owns buckets [PB t, PB t + PB)
                constexpr int PB = BBK / BT;
                uint4 *c4 = reinterpret_cast<uint4 *>(cn + PB * tid);
                uint32_t tot = 0, mc = 0;
#pragma unroll
                for (int q = 0; q < PB / 4; ++q) {
                    const uint4 y = c4[q];
                    tot += y.x + y.y + y.z + y.w;
                    mc = max(mc, max(max(y.x, y.y), max(y.z, y.w)));
                }
                uint32_t run = H::block_excl_scan(tot, reinterpret_cast<uint32_t *>(rd) + 128, mc, &cmax);
#pragma unroll
                for (int q = 0; q < PB / 4; ++q) {
                    const uint4 y = c4[q];
                    uint4 o;
                    o.x = run | (y.x << 16); run += y.x;
                    o.y = run | (y.y << 16); run += y.y;
                    o.z = run | (y.z << 16); run += y.z;
                    o.w = run | (y.w << 16); run += y.w;
                    c4[q] = o;
                }
            }
            if (tid == 0) bulk_wait_read();  // a slow leaf's bulk store has left kd (its prefetch follows it)
            H::bsync();
            const bool fast = cmax <= (uint32_t)CMAX;
            const int a0 = fast ? off : 0;  // fast path: q-space (the 16-byte phase of A); slow: linear
#pragma unroll
            for (int jv = 0; jv < BI / 4; ++jv) {
                if (jv < nvec) {
                    const int e0 = 4 * (jv * BT + tid) - off;
                    const bool whole = e0 >= 0 && e0 + 4 <= m;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int j = 4 * jv + q;
                        if (whole || (unsigned)(e0 + q) < (unsigned)m) {
                            const uint32_t pos = (cn[bucket(xs[j], vs[j])] & 0xFFFFu) + ((pp[j / 2] >> ((j & 1) << 4)) & 0xFFFFu);
                            PDQ_CHECK(pos < (uint32_t)m, "wide leaf scatter slot");
                            kc[a0 + pos] = xs[j];
                            if constexpr (KV) vc[a0 + pos] = vs[j];
                        }
                    }
                }
            }
            H::bsync();
            if (fast) {
                // rank every element inside its bucket ((key, payload) order, ties by position), then
                // write it to its rank in place (all reads precede the barrier)
                uint32_t rk[BI];
#pragma unroll
                for (int j = 0; j < BI; ++j) {
                    const int p = j * BT + tid;
                    rk[j] = 0xFFFFFFFFu;
                    if (p < m) {
                        const U x = kc[a0 + p];
                        const uint32_t v = KV ? vc[a0 + p] : 0u;
                        const uint32_t sc = cn[bucket(x, v)];
                        const uint32_t s0 = sc & 0xFFFFu, c = sc >> 16;
                        uint32_t r = s0;
                        if (c > 1) {
                            for (uint32_t i = s0; i < s0 + c; ++i) {
                                const U y = kc[a0 + i];
                                const uint32_t w = KV ? vc[a0 + i] : 0u;
                                r += less(y, w, x, v) | ((y == x) & (w == v) & (i < (uint32_t)p));
                            }
                        }
                        PDQ_CHECK(r < (uint32_t)m, "wide leaf rank");
                        rk[j] = r;
                        xs[j] = x;
                        vs[j] = v;
                    }
                }
                H::bsync();
#pragma unroll
                for (int j = 0; j < BI; ++j) {
                    if (rk[j] != 0xFFFFFFFFu) {
                        kc[a0 + rk[j]] = xs[j];
                        if constexpr (KV) vc[a0 + rk[j]] = vs[j];
                    }
                }
                H::bsync();
                // copy-out: 16-byte chunks of q-space (a0 + m slots) to A + b - a0, raw keys
                U *dstk = (U *)P.a_keys + (b - a0);
                const uint32_t qend = (uint32_t)(a0 + m);
                constexpr int KPC = 16 / (int)sizeof(U);  // keys per 16-byte chunk
                for (uint32_t c = tid; c < (qend + KPC - 1) / KPC; c += BT) {
                    const uint32_t q = c * KPC;
                    if (q >= (uint32_t)a0 && q + KPC <= qend) {
                        if constexpr (sizeof(U) == 4) {
                            const uint4 y = *reinterpret_cast<const uint4 *>(kc + q);
                            *reinterpret_cast<uint4 *>(dstk + q) =
                                make_uint4(O::from(y.x), O::from(y.y), O::from(y.z), O::from(y.w));
                        } else {
                            const ulonglong2 y = *reinterpret_cast<const ulonglong2 *>(kc + q);
                            *reinterpret_cast<ulonglong2 *>(dstk + q) = make_ulonglong2(O::from(y.x), O::from(y.y));
                        }
                    } else {
                        for (int e = 0; e < KPC; ++e)
                            if (q + e >= (uint32_t)a0 && q + e < qend) dstk[q + e] = O::from(kc[q + e]);
                    }
                }
                if constexpr (KV) {
                    uint32_t *dstv = P.a_vals + (b - a0);
                    for (uint32_t c = tid; c < (qend + 3) / 4; c += BT) {
                        const uint32_t q = c * 4;
                        if (q >= (uint32_t)a0 && q + 4 <= qend) {
                            *reinterpret_cast<uint4 *>(dstv + q) = *reinterpret_cast<const uint4 *>(vc + q);
                        } else {
                            for (int e = 0; e < 4; ++e)
                                if (q + e >= (uint32_t)a0 && q + e < qend) dstv[q + e] = vc[q + e];
                        }
                    }
                }
                if (tid == 0) {
                    sh.s_base++;
                    sh.s_bytes += 2ull * (sizeof(U) + (KV ? 4 : 0)) * m;
                    sh.s_cyc_base += clock64() - sh.lc0;
                    sh.lq[0] = sh.lq[1];
                }
                H::bsync();
                continue;
            }
            // slow path: the radix passes use kd / vd, so the next leaf's prefetch is dropped (after it
            // lands) and issued again once this leaf's bulk stores have read kd / vd
            if (sh.lq[1] != NONE) {
                mbar_wait(bar, kphase);
                kphase ^= 1u;
            }
            H::bsync();
            radix_leaf(m, off, kmn, krange, vmn, vmx - vmn);
            fence_proxy_async();
            H::bsync();
            {  // kd/vd[off, off + m) -> A[b, b + m): 16-byte bodies by bulk stores, head/tail by threads
                U *kd = kdk();
                uint32_t *vd = kdv();
                U *a = (U *)P.a_keys + b;
                uint32_t *av = KV ? P.a_vals + b : nullptr;
                int h = (4 - off) & 3;
                if (h > m) h = m;
                const int nb = ((m - h) / 4) * 4;
                if (tid > 0 && tid < 4 && tid - 1 < h) {
                    a[tid - 1] = kd[off + tid - 1];
                    if constexpr (KV) av[tid - 1] = vd[off + tid - 1];
                }
                if (tid >= 4 && tid < 8 && h + nb + tid - 4 < m) {
                    a[h + nb + tid - 4] = kd[off + h + nb + tid - 4];
                    if constexpr (KV) av[h + nb + tid - 4] = vd[off + h + nb + tid - 4];
                }
                if (tid == 0) {
                    if (nb) {
                        bulk_s2g(a + h, kd + off + h, (unsigned)(nb * sizeof(U)));
                        if constexpr (KV) bulk_s2g(av + h, vd + off + h, (unsigned)nb * 4u);
                    }
                    bulk_commit();
                    if (sh.lq[1] != NONE) {
                        bulk_wait_read();
                        prefetch(P, sh.lq[1], bar);
                    }
                    sh.s_base++;
                    sh.s_bytes += 2ull * (sizeof(U) + (KV ? 4 : 0)) * m;
                    sh.s_cyc_base += clock64() - sh.lc0;
                    sh.lq[0] = sh.lq[1];
                }
            }
            H::bsync();
        }
        if (tid == 0) bulk_wait_all();
        H::bsync();
    }
};

// ---- K4 two-run epilogue: merge A[0, s) and A[s, n) (both ascending) -----------------------------------
// Runs in the leaf kernel's persistent CTAs (one 1024-thread CTA per SM) after the leaves: wait until every
// leaf is in A, merge-path tiles A -> B, wait until every tile is written, copy B -> A.  The waits are
// progress counters, not grid barriers: leaves and tiles are claimed dynamically, so a CTA only waits for
// work that a running CTA holds, and concurrent sorts that cannot be co-resident do not deadlock.  A tile
// is T = 8192 outputs: its two input ranges come from a merge-path search over global memory (one warp per
// tile boundary, 32 probes per round), land in shared memory by cp.async (double-buffered), and every
// thread merges V = 8 consecutive outputs from its own diagonal and stores them as 16-byte vectors.  Ties
// take the first run's element (for keys-only sorts equal keys are identical bits; with a payload the
// order is the (key, payload) order, so there are no ties between distinct elements).
template <class U, bool FLOAT, bool KV>
struct RunsMerge {
    using O = Ord<U, FLOAT>;
    static constexpr int BT = 1024, V = 8, T = BT * V, BATCH = 32;
    // two stages of raw keys (+ payloads): tile k + 1 arrives by cp.async while tile k is merged
    static constexpr int VIN = T * (int)sizeof(U), STAGE = VIN + (KV ? T * 4 : 0), BND = 2 * STAGE;
    __host__ __device__ static constexpr int bytes() { return BND + (BATCH + 2) * 8; }
    __device__ __forceinline__ static U *kin(int st) { return reinterpret_cast<U *>(g_dsm + st * STAGE); }
    __device__ __forceinline__ static uint32_t *vin(int st) {
        return reinterpret_cast<uint32_t *>(g_dsm + st * STAGE + VIN);
    }
    __device__ __forceinline__ static int64_t *bnd() { return reinterpret_cast<int64_t *>(g_dsm + BND); }
    template <class E>
    __device__ __forceinline__ static void cp_async(E *sdst, const E *gsrc) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_addr(sdst)), "l"(gsrc), "n"((int)sizeof(E))
                     : "memory");
    }
    __device__ __forceinline__ static void bsync() { asm volatile("bar.sync 1, %0;" ::"n"(BT) : "memory"); }

    // thread 0 waits until *counter >= target (bracketed by CTA barriers and gpu-scope fences); like the
    // sorter's ring poll it gives up after 10 s and reports through the status word, never hangs
    __device__ static void wait_for(const Params &P, const unsigned long long *counter, unsigned long long target) {
        bsync();
        if (threadIdx.x == 0) {
            const uint64_t t0 = globaltimer_ns();
            while (*(const volatile unsigned long long *)counter < target) {
                if (globaltimer_ns() - t0 > WATCHDOG_NS) {
                    atomicCAS(&P.st->status, 0, -8);
                    break;
                }
                __nanosleep(128);
            }
            __threadfence();
        }
        bsync();
    }

    // Warp-cooperative 32-ary search: the first x in [lo, hi] with pred(x) false (pred is true below it,
    // false from it on; evaluated on [lo, hi) only).  Five rounds of 32 probes cover 2^25 positions, each
    // round one memory latency.
    template <class F>
    __device__ __forceinline__ static int64_t warp_first_false(int64_t lo, int64_t hi, F pred) {
        const int lane = threadIdx.x & 31;
        while (lo < hi) {
            const int64_t step = (hi - lo + 31) / 32;
            const int64_t p = lo + lane * step;
            const bool t = p < hi && pred(p);
            const int c = __popc(__ballot_sync(0xffffffffu, t));  // probes 0 .. c-1 are true
            if (c == 0) return lo;
            const int64_t nhi = lo + (int64_t)c * step;
            lo += (int64_t)(c - 1) * step + 1;
            hi = nhi < hi ? nhi : hi;
        }
        return lo;
    }
    __device__ __forceinline__ static uint64_t keyat(const Params &P, int64_t i) {
        return (uint64_t)O::to(ldcg((const U *)P.a_keys + i));
    }
    __device__ __forceinline__ static uint32_t valat(const Params &P, int64_t i) {
        return KV ? ldcg(P.a_vals + i) : 0u;
    }

    __device__ static void run(const Params &P) {
        Shared &sh = g_sh;
        const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
        const int64_t n = P.n, s = (int64_t)P.st->run_split;
        const U *a = (const U *)P.a_keys;
        U *b = (U *)P.b_keys;
        int64_t *bd = bnd();
        {  // every leaf is in A: this CTA's leaves are counted, then all of them awaited
            unsigned long long total = *(volatile unsigned long long *)&P.st->leaf_count;
            if (total > P.leaf_cap) total = P.leaf_cap;
            __threadfence();
            bsync();
            if (tid == 0 && sh.s_base) atomicAdd(&P.st->leaves_done, sh.s_base);
            wait_for(P, &P.st->leaves_done, total);
        }
        // The window that changes: first-run elements <= the second run's smallest stay where they are, and
        // so do second-run elements >= the first run's largest (appending slightly newer keys to a sorted
        // array merges only the overlap).  The window starts at a multiple of 8 elements (16-byte stores).
        if (warp == 0) {
            const uint64_t y = keyat(P, s);
            const uint32_t yv = valat(P, s);
            const int64_t p0 = warp_first_false(0, s, [&](int64_t i) { return !pless<KV>(y, yv, keyat(P, i), valat(P, i)); });
            if (lane == 0) bd[0] = p0 & ~(int64_t)7;
        } else if (warp == 1) {
            const uint64_t x = keyat(P, s - 1);
            const uint32_t xv = valat(P, s - 1);
            const int64_t q = warp_first_false(0, n - s, [&](int64_t j) { return pless<KV>(keyat(P, s + j), valat(P, s + j), x, xv); });
            if (lane == 0) bd[1] = s + q;
        }
        bsync();
        const int64_t o0 = bd[0], r2e = bd[1];
        PDQ_CHECK(o0 >= 0 && o0 <= s && r2e >= s && r2e <= n && (o0 & 7) == 0, "merge window");
        const int64_t len1 = s - o0, len2 = r2e - s, m = len1 + len2;
        bsync();
        const int64_t ntiles = (m + T - 1) / T;
        // tiles are claimed in batches of consecutive tiles: one batch per CTA when every CTA is running (each
        // batch pays one round of boundary searches), at most 32 tiles (one warp per boundary)
        int64_t batch = (ntiles + gridDim.x - 1) / gridDim.x;
        batch = batch < 1 ? 1 : (batch > BATCH ? BATCH : batch);
        unsigned long long moved = 0;
        for (;;) {
            bsync();
            if (tid == 0) bd[BATCH + 1] = (int64_t)atomicAdd(&P.st->merge_next, (unsigned long long)batch);
            bsync();
            const int64_t tb = bd[BATCH + 1];
            if (tb >= ntiles) break;
            const int64_t nb = ntiles - tb < batch ? ntiles - tb : batch;
            // merge path: first-run elements among the first d outputs, one boundary per warp at a time
            for (int64_t k = warp; k <= nb; k += BT / 32) {
                const int64_t d = (tb + k) * T < m ? (tb + k) * T : m;
                const int64_t lo = d > len2 ? d - len2 : 0, hi = d < len1 ? d : len1;
                const int64_t r = warp_first_false(lo, hi, [&](int64_t mid) {
                    return !pless<KV>(keyat(P, s + (d - 1 - mid)), valat(P, s + (d - 1 - mid)), keyat(P, o0 + mid),
                                      valat(P, o0 + mid));
                });
                if (lane == 0) bd[k] = r;
            }
            bsync();
            // tile k's two input ranges -> stage k & 1 (raw bits; the ordered image is taken on read)
            auto issue = [&](int64_t k) {
                const int64_t d0 = (tb + k) * T, d1 = d0 + T < m ? d0 + T : m;
                const int64_t i0 = bd[k], j0 = d0 - i0;
                const int L1 = (int)(bd[k + 1] - i0), L = (int)(d1 - d0);
                U *kd = kin((int)(k & 1));
                uint32_t *vd = vin((int)(k & 1));
                PDQ_CHECK(L1 >= 0 && L1 <= L && L <= T && j0 >= 0, "merge tile boundaries are monotone");
                for (int x = tid; x < L; x += BT) {
                    const int64_t src = x < L1 ? o0 + i0 + x : s + j0 + (x - L1);
                    PDQ_CHECK(src >= 0 && src < P.n && (x < L1 ? src < s : src >= s), "merge tile source inside its run");
                    cp_async(kd + x, a + src);
                    if constexpr (KV) cp_async(vd + x, P.a_vals + src);
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            issue(0);
            for (int64_t k = 0; k < nb; ++k) {
                const int64_t d0 = (tb + k) * T, d1 = d0 + T < m ? d0 + T : m;
                const int64_t i0 = bd[k], i1 = bd[k + 1];
                const int L1 = (int)(i1 - i0), L = (int)(d1 - d0), L2 = L - L1;
                if (k + 1 < nb) {
                    issue(k + 1);
                    asm volatile("cp.async.wait_group 1;" ::: "memory");
                } else {
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
                }
                bsync();
                const U *kr = kin((int)(k & 1));
                const uint32_t *vi = vin((int)(k & 1));
                auto ki = [&](int idx) -> U { return O::to(kr[idx]); };
                const int dl = tid * V < L ? tid * V : L;
                int lo = dl > L2 ? dl - L2 : 0, hi = dl < L1 ? dl : L1;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    const uint64_t x = (uint64_t)ki(mid), y = (uint64_t)ki(L1 + dl - 1 - mid);
                    const uint32_t xv = KV ? vi[mid] : 0u, yv = KV ? vi[L1 + dl - 1 - mid] : 0u;
                    if (!pless<KV>(y, yv, x, xv)) lo = mid + 1;
                    else hi = mid;
                }
                int ia = lo, ib = dl - lo;
                U ok[V];
                uint32_t ov[V];
                U xa = ia < L1 ? ki(ia) : (U)0, xb = ib < L2 ? ki(L1 + ib) : (U)0;
                uint32_t va = (KV && ia < L1) ? vi[ia] : 0u, vb = (KV && ib < L2) ? vi[L1 + ib] : 0u;
#pragma unroll
                for (int q = 0; q < V; ++q) {
                    const bool takeA = ib >= L2 || (ia < L1 && !pless<KV>((uint64_t)xb, vb, (uint64_t)xa, va));
                    ok[q] = O::from(takeA ? xa : xb);
                    ov[q] = takeA ? va : vb;
                    if (takeA) {
                        ++ia;
                        xa = ia < L1 ? ki(ia) : (U)0;
                        if constexpr (KV) va = ia < L1 ? vi[ia] : 0u;
                    } else {
                        ++ib;
                        xb = ib < L2 ? ki(L1 + ib) : (U)0;
                        if constexpr (KV) vb = ib < L2 ? vi[L1 + ib] : 0u;
                    }
                }
                U *dst = b + o0 + d0 + dl;
                PDQ_CHECK(o0 + d0 + L <= P.n, "merge tile output inside the array");
                if (dl + V <= L) {  // o0 + d0 + dl is a multiple of 8 elements: 16-byte aligned vectors
                    constexpr int KPV = 16 / (int)sizeof(U);
#pragma unroll
                    for (int q = 0; q < V / KPV; ++q) {
                        union {
                            U t[KPV];
                            uint4 u;
                        } pk;
#pragma unroll
                        for (int e = 0; e < KPV; ++e) pk.t[e] = ok[q * KPV + e];
                        reinterpret_cast<uint4 *>(dst)[q] = pk.u;
                    }
                    if constexpr (KV) {
                        uint4 *dv = reinterpret_cast<uint4 *>(P.b_vals + o0 + d0 + dl);
                        dv[0] = make_uint4(ov[0], ov[1], ov[2], ov[3]);
                        dv[1] = make_uint4(ov[4], ov[5], ov[6], ov[7]);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < V; ++q)
                        if (dl + q < L) {
                            dst[q] = ok[q];
                            if constexpr (KV) P.b_vals[o0 + d0 + dl + q] = ov[q];
                        }
                }
                moved += (tid == 0) ? (unsigned long long)L : 0ull;
                bsync();
            }
            __threadfence();  // this batch's tiles are in B
            bsync();
            if (tid == 0) atomicAdd(&P.st->merge_done, (unsigned long long)nb);
        }
        wait_for(P, &P.st->merge_done, (unsigned long long)ntiles);  // B holds the merged window
        {  // copy the window back, 16-byte vectors (o0 is a multiple of 8 elements)
            constexpr int KPV = 16 / (int)sizeof(U);
            const int64_t gt = (int64_t)blockIdx.x * BT + tid, gs = (int64_t)gridDim.x * BT;
            const int64_t nv = m / KPV;
            const uint4 *src = reinterpret_cast<const uint4 *>(b + o0);
            uint4 *dst = reinterpret_cast<uint4 *>((U *)P.a_keys + o0);
            for (int64_t c = gt; c < nv; c += gs) dst[c] = __ldcg(src + c);
            for (int64_t i = o0 + nv * KPV + gt; i < r2e; i += gs) ((U *)P.a_keys)[i] = b[i];
            if constexpr (KV) {
                const int64_t nw = m / 4;
                const uint4 *sv = reinterpret_cast<const uint4 *>(P.b_vals + o0);
                uint4 *dv = reinterpret_cast<uint4 *>(P.a_vals + o0);
                for (int64_t c = gt; c < nw; c += gs) dv[c] = __ldcg(sv + c);
                for (int64_t i = o0 + nw * 4 + gt; i < r2e; i += gs) P.a_vals[i] = P.b_vals[i];
            }
        }
        // merge + copy: 4 (w + p) bytes per element (SURVEY.md §8(d) counts a pass as read + write)
        if (tid == 0) sh.s_bytes += 4ull * (sizeof(U) + (KV ? 4 : 0)) * moved;
    }
};

template <class U, bool FLOAT, bool KV>
__global__ void __launch_bounds__(1024, 1) k_base_wide(const __grid_constant__ Params P) {
    using S = Sorter<U, FLOAT, KV>;
    Shared &sh = g_sh;
    const int tid = threadIdx.x;
    pdl_wait();  // the sorter's leaf queue
    const bool runs = P.st->run_split != 0;
    const bool rev = ld_volatile_u32(&P.st->reverse) != 0;
    if (rev && !runs) return;
    if (tid == 0) {
        S::zero_counters();
        atomicMax(&P.st->t_base_b_inv, ~globaltimer_ns());
    }
    if (!rev) WideLeaf<U, FLOAT, KV>::run(P);
    if (runs) {
        static_assert(RunsMerge<U, FLOAT, KV>::bytes() <= WideLeaf<U, FLOAT, KV>::bytes(), "merge tiles fit the leaf buffers");
        RunsMerge<U, FLOAT, KV>::run(P);
    }
    if (tid == 0) {
        atomicMax(&P.st->t_base_e, globaltimer_ns());
        atomicAdd(&P.st->c_bytes_base, sh.s_bytes);
        sh.s_bytes = 0;
        S::flush_counters(P);
    }
}

template <bool FLOAT>
__global__ void __launch_bounds__(BigLeaf<FLOAT>::BT, 1) k_base_big(const __grid_constant__ Params P) {
    using S = Sorter<uint32_t, FLOAT, false>;
    Shared &sh = g_sh;
    const int tid = threadIdx.x;
    pdl_wait();  // the sorter's leaf queue
    const bool runs = P.st->run_split != 0;
    const bool rev = ld_volatile_u32(&P.st->reverse) != 0;
    if (rev && !runs) return;
    if (tid == 0) {
        S::zero_counters();
        atomicMax(&P.st->t_base_b_inv, ~globaltimer_ns());
    }
    if (!rev) BigLeaf<FLOAT>::run(P);
    if (runs) {
        static_assert(RunsMerge<uint32_t, FLOAT, false>::bytes() <= BigLeaf<FLOAT>::bytes(), "merge tiles fit the leaf buffers");
        RunsMerge<uint32_t, FLOAT, false>::run(P);
    }
    if (tid == 0) {
        atomicMax(&P.st->t_base_e, globaltimer_ns());
        atomicAdd(&P.st->c_bytes_base, sh.s_bytes);
        sh.s_bytes = 0;
        S::flush_counters(P);
    }
}

// ---- K6: the persistent segment-queue sorter --------------------------------------------------------
#ifndef PDQ_MINB
#define PDQ_MINB 6
#endif
template <class U, bool KV>
constexpr int sort_min_blocks() {
    // CTAs that fit in shared memory (+ static shared memory and the per-CTA reserve), capped
    constexpr int fit = (228 * 1024) / (Bufs<U, KV>::bytes() + 2304);
    return fit > PDQ_MINB ? PDQ_MINB : (fit < 1 ? 1 : fit);
}

template <class U, bool FLOAT, bool KV>
__global__ void __launch_bounds__(THREADS, sort_min_blocks<U, KV>()) k_sort(const __grid_constant__ Params P) {
    using S = Sorter<U, FLOAT, KV>;
    Shared &sh = g_sh;
    const int tid = threadIdx.x;
    pdl_wait();  // k_init's root segment and verdict
    if (tid == 0) atomicMax(&P.st->t_sort_b_inv, ~globaltimer_ns());

    // K4 reverse: a non-increasing input (or the non-increasing one of two runs), [rev_begin, rev_end), is
    // reversed in place (one read + one write pass)
    if (ld_volatile_u32(&P.st->reverse)) {
        const int64_t r0 = (int64_t)P.st->rev_begin;
        U *a = (U *)P.a_keys + r0;
        uint32_t *av = KV ? P.a_vals + r0 : nullptr;
        const int64_t n = (int64_t)P.st->rev_end - r0, half = n / 2;
        const int64_t gt = (int64_t)blockIdx.x * THREADS + tid, gs = (int64_t)gridDim.x * THREADS;
        int64_t done = 0;
        if (n % S::AL == 0 && r0 % S::AL == 0) {
            // 16-byte vectors from both ends (the range and its end are then 16-byte aligned): vector c of
            // the front swaps with vector c of the back, each reversed in registers
            constexpr int V = S::VEC;
            const int64_t nv = half / S::AL * S::AL / V;  // key vectors per side (whole payload vectors too)
            for (int64_t c = gt; c < nv; c += gs) {
                U *f = a + c * V, *bk = a + n - (c + 1) * V;
                U x[V], y[V];
                S::ldvec(f, 0, x);
                S::ldvec(bk, 0, y);
                U rx[V], ry[V];
#pragma unroll
                for (int q = 0; q < V; ++q) {
                    rx[q] = x[V - 1 - q];
                    ry[q] = y[V - 1 - q];
                }
                S::stvec(f, ry);
                S::stvec(bk, rx);
            }
            if (KV) {
                const int64_t nw = half / S::AL * S::AL / 4;
                for (int64_t c = gt; c < nw; c += gs) {
                    uint4 *f = reinterpret_cast<uint4 *>(av + c * 4);
                    uint4 *bk = reinterpret_cast<uint4 *>(av + n - (c + 1) * 4);
                    const uint4 x = *f, y = *bk;
                    *f = make_uint4(y.w, y.z, y.y, y.x);
                    *bk = make_uint4(x.w, x.z, x.y, x.x);
                }
            }
            done = half / S::AL * S::AL;
        }
        // the rest (or all of an unaligned range: the second of two runs starts anywhere): element swaps,
        // four independent pairs in flight per thread
        for (int64_t i0 = done + gt; i0 < half; i0 += 4 * gs) {
            U x[4], y[4];
            uint32_t xv[4], yv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t i = i0 + q * gs;
                if (i < half) {
                    x[q] = a[i];
                    y[q] = a[n - 1 - i];
                    if (KV) {
                        xv[q] = av[i];
                        yv[q] = av[n - 1 - i];
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t i = i0 + q * gs;
                if (i < half) {
                    a[i] = y[q];
                    a[n - 1 - i] = x[q];
                    if (KV) {
                        av[i] = yv[q];
                        av[n - 1 - i] = xv[q];
                    }
                }
            }
        }
        __syncthreads();
        if (tid == 0) atomicMax(&P.st->t_sort_e, globaltimer_ns());
        return;
    }
    if (tid == 0) {
        S::zero_counters();
        for (int i = 0; i < S::B::NSTAGE; ++i) mbar_init(&sh.bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        sh.li = sh.ci = 0;
        sh.lslot = 0;
        sh.ltile = 0;
        sh.task = 0;
        sh.npos = atomicAdd(&P.st->q_head, 1ull);
        sh.nstate = 1;
        S::advance(P);
    }
    __syncthreads();
    unsigned ci = 0;  // tiles consumed (all threads keep the same count)
    long long c_prev = clock64();
    for (;;) {
        const uint64_t w = sh.task;
        if (!w) break;
        const uint32_t type = (uint32_t)(w >> 45) & 7u;
        const uint32_t sid = (uint32_t)(w >> 23) & 0x3FFFFF;
        if (S::tile_task(type)) {
            const uint32_t t0 = (uint32_t)w & 0x7FFFFF;
            const uint32_t t1 = task_end_tile(t0, sh.seg.ntiles, P.chunk);
            if (type == T_PART) {
                for (uint32_t t = t0; t < t1; ++t) S::part_tile(P, sid, t, ci);
            } else if (type == T_RHIST) {
                for (uint32_t t = t0; t < t1; ++t) S::hist_tile(P, t, ci);
            } else {
                for (uint32_t t = t0; t < t1; ++t) S::rscat_tile(P, t, ci);
            }
            // retire the chunk: the bulk stores complete, one gpu-scope fence per thread, one
            // counter update per CTA
            if (tid == 0) {
                bulk_wait_all();
                fence_proxy_async_global();
            }
            __threadfence();
            csync();
            if (tid == 0) {
                const long long c = clock64();
                const unsigned old = atomicAdd(&P.segs[sid].tiles_done, t1 - t0);
                sh.last = (old + (t1 - t0) == sh.seg.ntiles);
#ifndef PDQ_BIG_PHASES
                sh.s_sch_retire += clock64() - c;
#endif
            }
            csync();
            if (sh.last) {
                __threadfence();
                if (type == T_PART)
                    S::finalize_part(P, sh.seg, sid);
                else if (type == T_RHIST)
                    S::radix_hist_done(P, sh.seg, sid);
                else
                    S::radix_scat_done(P, sh.seg, sid);
            }
        } else {  // T_FILL
            S::fill_tile(P, sh.seg, (uint32_t)w & 0x7FFFFF);
        }
        csync();
        if (tid == 0) {
            const long long c = clock64();
            sh.s_cyc_work += c - c_prev;
            S::advance(P);
            const long long c2 = clock64();
            sh.s_cyc_wait += c2 - c;
            c_prev = c2;
        }
        csync();
    }
    if (tid == 0) {
        S::flush_counters(P);
        atomicMax(&P.st->t_sort_e, globaltimer_ns());
    }
}

}  // namespace pdq
