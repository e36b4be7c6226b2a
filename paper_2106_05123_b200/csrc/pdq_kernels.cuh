// pdq_kernels.cuh — the seven kernels of the B200 pdqsort path.
//
//   K1 sample pivot          spawn(): SAMPLES evenly spaced keys, CTA bitonic, median
//                            (generalises choose_pivot, driver.py:81-113)
//   K2 partition_right       part_tile(): TMA bulk tile -> classify -> ballot/popc ranks ->
//                            block scan -> one atomic per side per CTA -> 16 B stores
//                            (block_partition_right, partition.py:184-301)
//   K3 partition_left        part_tile() in I_LEFT mode (partition.py:128-181, driver.py:222-225)
//   K4 sortedness check      k_check(): adjacent-compare reduction; k_sort prologue reverses
//                            non-increasing input (partial_insertion_sort path, driver.py:244-250)
//   K5 bad-partition budget  finalize_part(): is_bad_partition (driver.py:116-124), budget,
//                            sample perturbation (break_patterns, driver.py:127-156)
//   K6 segment queue         k_sort(): persistent CTAs popping tasks from a device ring;
//                            the last tile of a segment spawns its children (driver.py:198-260)
//   K7 base case             base_case(): segment <= base_case_size sorted in shared memory
//                            (insertion_sort / unguarded_insertion_sort, small_sorts.py:16-73)
#pragma once

#include "pdq_device.cuh"

namespace pdq {

struct Shared {
    uint64_t bar;
    uint64_t task;
    Seg seg;
    int wl[WARPS], wv[WARPS], weq[WARPS], wloff[WARPS], wroff[WARPS];
    long long L, R, lOff, rOff, fL, fE;
    unsigned long long push_pos;
    int last, loaded;
    uint32_t new_sid;
    int reused;
    uint64_t samp_k[SAMPLES];
    uint32_t samp_v[SAMPLES];
    // per-CTA counters, flushed once at exit
    unsigned long long s_part_right, s_part_left, s_bad, s_fallback, s_base, s_tiles, s_bytes;
    long long s_max_depth;
};

__device__ __forceinline__ uint32_t mix32(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return (uint32_t)x;
}

template <class U, bool FLOAT, bool KV>
struct Sorter {
    using O = Ord<U, FLOAT>;
    static constexpr int VEC = 16 / sizeof(U);
    static constexpr int AL = KV ? 4 : VEC;  // element alignment making both key and payload 16 B aligned
    static constexpr int ELEM_BYTES = sizeof(U) + (KV ? 4 : 0);

    // ---- vectorised contiguous store of `len` elements produced by get(i) -----------
    template <class T, class F>
    __device__ __forceinline__ static void store_run(T *g, int64_t len, F get) {
        constexpr int V = 16 / sizeof(T);
        const int tid = threadIdx.x;
        int64_t mis = ((uintptr_t)g / sizeof(T)) & (V - 1);
        int64_t h = mis ? V - mis : 0;
        if (h > len) h = len;
        for (int64_t i = tid; i < h; i += THREADS) g[i] = get(i);
        int64_t nb = (len - h) / V;
        uint4 *gv = reinterpret_cast<uint4 *>(g + h);
        for (int64_t b = tid; b < nb; b += THREADS) {
            union {
                T t[V];
                uint4 u;
            } pk;
#pragma unroll
            for (int q = 0; q < V; ++q) pk.t[q] = get(h + b * V + q);
            gv[b] = pk.u;
        }
        for (int64_t i = h + nb * V + tid; i < len; i += THREADS) g[i] = get(i);
    }

    // ---- CTA bitonic sort in shared memory (mirror variant: every compare-exchange puts
    // the smaller element at the lower index, so virtual +inf padding never moves and pairs
    // whose upper index is >= m are skipped). ---------------------------------------------
    template <class K>
    __device__ static void bitonic(K *k, uint32_t *v, int m) {
        int P = 1;
        while (P < m) P <<= 1;
        const int tid = threadIdx.x;
        for (int kk = 2; kk <= P; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
                const int lj = __ffs(j) - 1;
                const bool mirror = (j == (kk >> 1));
                for (int p = tid; p < (P >> 1); p += THREADS) {
                    int i = ((p >> lj) << (lj + 1)) | (p & (j - 1));
                    int q = mirror ? (i ^ (kk - 1)) : (i + j);
                    if (q < m) {
                        K a = k[i], b = k[q];
                        uint32_t va = KV ? v[i] : 0, vb = KV ? v[q] : 0;
                        if (pless<KV>(b, vb, a, va)) {
                            k[i] = b;
                            k[q] = a;
                            if (KV) {
                                v[i] = vb;
                                v[q] = va;
                            }
                        }
                    }
                }
                __syncthreads();
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

    // ---- K7: base case ------------------------------------------------------------------
    __device__ static void base_case(const Params &P, Shared &sh, U *sk, uint32_t *sv, bool srcB,
                                     int64_t b, int m) {
        const int tid = threadIdx.x;
        const U *src = (const U *)(srcB ? P.b_keys : P.a_keys);
        const uint32_t *srcv = srcB ? P.b_vals : P.a_vals;
        for (int i = tid; i < m; i += THREADS) {
            sk[i] = O::to(ldcg(src + b + i));
            if (KV) sv[i] = ldcg(srcv + b + i);
        }
        __syncthreads();
        bitonic<U>(sk, sv, m);
        U *dk = (U *)P.a_keys + b;
        store_run<U>(dk, m, [&](int64_t i) { return O::from(sk[i]); });
        if (KV) store_run<uint32_t>(P.a_vals + b, m, [&](int64_t i) { return sv[i]; });
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            sh.s_base++;
            sh.s_bytes += 2ull * ELEM_BYTES * m;
            finish_keys(P, m);
        }
        __syncthreads();
    }

    // ---- write [b, e) of A with the pivot (equal-key runs are bitwise identical under the
    // total order, so a fill is exact).  Returns true if it took the reusable descriptor. ---
    __device__ static bool fill_final(const Params &P, Shared &sh, int64_t b, int64_t e, uint64_t piv,
                                      uint32_t pv, int reuse_sid) {
        const int tid = threadIdx.x;
        const int64_t m = e - b;
        if (m <= 0) return false;
        if (m <= INLINE_FILL) {
            const U raw = O::from((U)piv);
            store_run<U>((U *)P.a_keys + b, m, [&](int64_t) { return raw; });
            if (KV) store_run<uint32_t>(P.a_vals + b, m, [&](int64_t) { return pv; });
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                sh.s_bytes += (unsigned long long)ELEM_BYTES * m;
                finish_keys(P, m);
            }
            __syncthreads();
            return false;
        }
        const uint32_t ntiles = (uint32_t)((e - 1) / TILE - b / TILE + 1);
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
        __syncthreads();
        if (sh.new_sid < P.seg_cap) {
            const unsigned long long pos = sh.push_pos;
            const uint64_t mask = (1ull << P.log_q) - 1;
            for (uint32_t t = tid; t < ntiles; t += THREADS)
                *(volatile uint64_t *)&P.ring[(pos + t) & mask] = task_word(pos + t, P.log_q, T_FILL, sh.new_sid, t);
        }
        __syncthreads();
        return reuse_sid >= 0;
    }

    // ---- K1 + segment creation ------------------------------------------------------------
    // Creates the child segment [b, e) whose data lives in buffer srcB.  Small children are
    // finished right here (K7); big ones get a sampled pivot and their tiles are pushed.
    // Returns true iff the reusable descriptor `reuse_sid` was consumed.
    __device__ static bool spawn(const Params &P, Shared &sh, U *sk, uint32_t *sv, int64_t b, int64_t e,
                                 bool srcB, bool has_lb, uint64_t lb, uint32_t lbv, int budget, int depth,
                                 bool perturb, int reuse_sid) {
        const int tid = threadIdx.x;
        const int64_t m = e - b;
        if (m <= 0) return false;
        if (tid == 0 && depth > sh.s_max_depth) sh.s_max_depth = depth;
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
            __syncthreads();
            return false;
        }
        if (m <= P.base_size) {
            base_case(P, sh, sk, sv, srcB, b, (int)m);
            return false;
        }
        // K1: SAMPLES keys at stratified positions; perturbed strata after a bad partition.
        const U *src = (const U *)(srcB ? P.b_keys : P.a_keys);
        const uint32_t *srcv = srcB ? P.b_vals : P.a_vals;
        for (int i = tid; i < SAMPLES; i += THREADS) {
            int64_t off;
            if (perturb)
                off = ((int64_t)i * m + (int64_t)(mix32((uint64_t)b * 0x9E3779B97F4A7C15ull ^ (uint64_t)(depth * 977 + i)) %
                                                 (uint64_t)m)) / SAMPLES;
            else
                off = ((int64_t)(2 * i + 1) * m) / (2 * SAMPLES);
            sh.samp_k[i] = (uint64_t)O::to(ldcg(src + b + off));
            sh.samp_v[i] = KV ? ldcg(srcv + b + off) : 0;
        }
        __syncthreads();
        bitonic<uint64_t>(sh.samp_k, sh.samp_v, SAMPLES);
        const uint64_t piv = sh.samp_k[SAMPLES / 2];
        const uint32_t pv = sh.samp_v[SAMPLES / 2];
        // driver.py:222: a predecessor not less than the pivot equals it -> partition_left
        const bool left = P.use_left && has_lb && !pless<KV>(lb, lbv, piv, pv);
        const uint32_t ntiles = (uint32_t)((e - 1) / TILE - b / TILE + 1);
        if (tid == 0) {
            uint32_t sid = reuse_sid >= 0 ? (uint32_t)reuse_sid : atomicAdd(&P.st->seg_alloc, 1u);
            sh.new_sid = sid;
            sh.s_bytes += (unsigned long long)SAMPLES * ELEM_BYTES;
            if (!left && budget <= 0) sh.s_fallback++;
            if (sid >= P.seg_cap) {
                fail(P, -6);
            } else {
                Seg *s = &P.segs[sid];
                s->begin = b;
                s->end = e;
                s->pivot = piv;
                s->pivot_v = pv;
                s->lb = lb;
                s->lb_v = lbv;
                s->ntiles = ntiles;
                s->info = (srcB ? I_SRC_B : 0) | (left ? I_LEFT : 0) | (has_lb ? I_HAS_LB : 0) |
                          (perturb ? I_PERTURB : 0);
                s->budget = budget > 0 ? budget : 0;
                s->depth = depth;
                s->cnt_left = 0;
                s->cnt_right = 0;
                s->cnt_eq = 0;
                s->tiles_done = 0;
                __threadfence();
                sh.push_pos = atomicAdd(&P.st->q_tail, (unsigned long long)ntiles);
            }
        }
        __syncthreads();
        if (sh.new_sid < P.seg_cap) {
            const unsigned long long pos = sh.push_pos;
            const uint64_t mask = (1ull << P.log_q) - 1;
            const uint32_t sid = sh.new_sid;
            for (uint32_t t = tid; t < ntiles; t += THREADS)
                *(volatile uint64_t *)&P.ring[(pos + t) & mask] = task_word(pos + t, P.log_q, T_PART, sid, t);
        }
        __syncthreads();
        return reuse_sid >= 0;
    }

    // ---- K5 + K6: the last tile of a segment decides its children ----------------------------
    __device__ __noinline__ static void finalize_part(const Params &P, Shared &sh, U *sk, uint32_t *sv, uint32_t sid) {
        const int tid = threadIdx.x;
        if (tid == 0) {
            Seg *gs = &P.segs[sid];
            sh.fL = (long long)atomicAdd(&gs->cnt_left, 0ull);
            sh.fE = (long long)atomicAdd(&gs->cnt_eq, 0ull);
        }
        __syncthreads();
        const Seg sg = sh.seg;  // parent fields (immutable while it lived)
        const int64_t b = sg.begin, e = sg.end, m = e - b, L = sh.fL;
        const bool srcB = sg.info & I_SRC_B, dstB = !srcB;
        if (!(sg.info & I_LEFT)) {
            if (tid == 0) sh.s_part_right++;
            if (sh.fE == m) {
                // Every key is bitwise equal to the pivot: whichever buffer A holds (the untouched
                // source, or this pass's output) already is the final, constant run.
                if (tid == 0) finish_keys(P, (unsigned long long)m);
                __syncthreads();
                return;
            }
            const int64_t R = m - L;
            const int64_t thr = m >> P.bad_shift;  // driver.py:123
            const bool bad = L < thr || R < thr;
            if (tid == 0 && bad) sh.s_bad++;
            const int nb = sg.budget - (bad ? 1 : 0);
            const bool perturb = bad && P.use_break;
            bool used = spawn(P, sh, sk, sv, b, b + L, dstB, sg.info & I_HAS_LB, sg.lb, sg.lb_v, nb, sg.depth + 1,
                              perturb, (int)sid);
            spawn(P, sh, sk, sv, b + L, e, dstB, true, sg.pivot, sg.pivot_v, nb, sg.depth + 1, perturb,
                  used ? -1 : (int)sid);
        } else {
            if (tid == 0) sh.s_part_left++;
            bool used = false;
            if (srcB) {
                // lefts were written straight into A during the pass
                if (tid == 0 && L) finish_keys(P, (unsigned long long)L);
                __syncthreads();
            } else {
                used = fill_final(P, sh, b, b + L, sg.pivot, sg.pivot_v, (int)sid);
            }
            spawn(P, sh, sk, sv, b + L, e, dstB, true, sg.pivot, sg.pivot_v, sg.budget, sg.depth + 1, false,
                  used ? -1 : (int)sid);
        }
    }

    // ---- K2/K3: one partition tile ------------------------------------------------------------
    __device__ static void part_tile(const Params &P, Shared &sh, U *sk, uint32_t *sv, U *ck, uint32_t *cv,
                                     uint32_t sid, uint32_t tile, unsigned &phase) {
        const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
        const Seg &sg = sh.seg;
        const int64_t b = sg.begin, e = sg.end;
        const bool srcB = sg.info & I_SRC_B;
        const bool left_mode = sg.info & I_LEFT;
        const U *src = (const U *)(srcB ? P.b_keys : P.a_keys);
        U *dst = (U *)(srcB ? P.a_keys : P.b_keys);
        const uint32_t *srcv = srcB ? P.b_vals : P.a_vals;
        uint32_t *dstv = srcB ? P.a_vals : P.b_vals;
        const int64_t tbase = (b / TILE + tile) * (int64_t)TILE;
        const int64_t lo = b > tbase ? b : tbase;
        const int64_t hi = e < tbase + TILE ? e : tbase + TILE;
        const int64_t nfl = P.n & ~(int64_t)(AL - 1);
        const int64_t lo_al = lo & ~(int64_t)(AL - 1);
        int64_t hi_al = (hi + AL - 1) & ~(int64_t)(AL - 1);
        if (hi_al > nfl) hi_al = nfl;
        const bool bulk = hi_al > lo_al;
        if (tid == 0 && bulk) {
            const unsigned kb = (unsigned)((hi_al - lo_al) * sizeof(U));
            const unsigned vb = KV ? (unsigned)((hi_al - lo_al) * 4) : 0u;
            fence_proxy_async();
            mbar_expect_tx(&sh.bar, kb + vb);
            bulk_g2s(sk + (lo_al - tbase), src + lo_al, kb, &sh.bar);
            if (KV) bulk_g2s(sv + (lo_al - tbase), srcv + lo_al, vb, &sh.bar);
        }
        // the array's last < 16 bytes cannot be bulk-copied: scalar loads
        for (int64_t g = (hi_al > lo ? hi_al : lo) + tid; g < hi; g += THREADS) {
            sk[g - tbase] = ldcg(src + g);
            if (KV) sv[g - tbase] = ldcg(srcv + g);
        }
        if (bulk) {
            mbar_wait(&sh.bar, phase);
            phase ^= 1;
        }
        __syncthreads();

        // classify: left = key < pivot (partition_right, equals go right, partition.py:76-77)
        //           left = key <= pivot (partition_left, equals go left, partition.py:134-135)
        // Pass 1 counts per warp with ballot/popc; pass 2 recomputes the same ballots and
        // scatters into the compaction buffer, so no per-key state lives in registers.
        const uint64_t piv = sg.pivot;
        const uint32_t pv = sg.pivot_v;
        const unsigned ltm = lanemask_lt();
        const int lo_i = (int)(lo - tbase), hi_i = (int)(hi - tbase);
        int wl = 0, wv = 0, eqc = 0;
#pragma unroll 4
        for (int j = 0; j < ITEMS; ++j) {
            const int idx = j * THREADS + tid;
            const bool valid = idx >= lo_i && idx < hi_i;
            const uint64_t ok = (uint64_t)O::to(sk[idx]);
            const uint32_t v = KV ? sv[idx] : 0u;
            const bool isl = valid && (left_mode ? !pless<KV>(piv, pv, ok, v) : pless<KV>(ok, v, piv, pv));
            eqc += (valid && ok == piv && (!KV || v == pv)) ? 1 : 0;
            wl += __popc(__ballot_sync(0xffffffffu, isl));
            wv += __popc(__ballot_sync(0xffffffffu, valid));
        }
        eqc = __reduce_add_sync(0xffffffffu, eqc);
        if (lane == 0) {
            sh.wl[warp] = wl;
            sh.wv[warp] = wv;
            sh.weq[warp] = eqc;
        }
        __syncthreads();
        if (tid == 0) {
            int offL = 0, offR = 0, E = 0;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) {
                sh.wloff[w] = offL;
                sh.wroff[w] = offR;
                offL += sh.wl[w];
                offR += sh.wv[w] - sh.wl[w];
                E += sh.weq[w];
            }
            Seg *gs = &P.segs[sid];
            sh.L = offL;
            sh.R = offR;
            // one atomic per side per CTA: the left run grows up from `begin`, the right
            // run grows down from `end`
            sh.lOff = offL ? (long long)atomicAdd(&gs->cnt_left, (unsigned long long)offL) : 0;
            sh.rOff = offR ? (long long)atomicAdd(&gs->cnt_right, (unsigned long long)offR) : 0;
            if (!left_mode && E) atomicAdd(&gs->cnt_eq, (unsigned long long)E);
            sh.s_tiles++;
            const bool write_left = !left_mode || srcB;
            sh.s_bytes += (unsigned long long)ELEM_BYTES * (offL + offR) +
                          (unsigned long long)ELEM_BYTES * (offR + (write_left ? offL : 0));
        }
        __syncthreads();
        const int L = (int)sh.L;
        {
            int lrun = sh.wloff[warp], rrun = L + sh.wroff[warp];
#pragma unroll 4
            for (int j = 0; j < ITEMS; ++j) {
                const int idx = j * THREADS + tid;
                const bool valid = idx >= lo_i && idx < hi_i;
                const U k = sk[idx];
                const uint64_t ok = (uint64_t)O::to(k);
                const uint32_t v = KV ? sv[idx] : 0u;
                const bool isl = valid && (left_mode ? !pless<KV>(piv, pv, ok, v) : pless<KV>(ok, v, piv, pv));
                const unsigned bl = __ballot_sync(0xffffffffu, isl);
                const unsigned br = __ballot_sync(0xffffffffu, valid && !isl);
                if (valid) {
                    const int pos = isl ? lrun + __popc(bl & ltm) : rrun + __popc(br & ltm);
                    ck[pos] = k;
                    if (KV) cv[pos] = v;
                }
                lrun += __popc(bl);
                rrun += __popc(br);
            }
        }
        __syncthreads();
        const int R = (int)sh.R;
        const long long lOff = sh.lOff, rOff = sh.rOff;
        if (L && (!left_mode || srcB)) {
            store_run<U>(dst + b + lOff, L, [&](int64_t i) { return ck[i]; });
            if (KV) store_run<uint32_t>(dstv + b + lOff, L, [&](int64_t i) { return cv[i]; });
        }
        if (R) {
            store_run<U>(dst + e - rOff - R, R, [&](int64_t i) { return ck[L + i]; });
            if (KV) store_run<uint32_t>(dstv + e - rOff - R, R, [&](int64_t i) { return cv[L + i]; });
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            unsigned old = atomicAdd(&P.segs[sid].tiles_done, 1u);
            sh.last = (old == sg.ntiles - 1);
        }
        __syncthreads();
        if (sh.last) {
            __threadfence();
            finalize_part(P, sh, sk, sv, sid);
        }
    }

    __device__ static void fill_tile(const Params &P, Shared &sh, uint32_t tile) {
        const Seg &sg = sh.seg;
        const int64_t tbase = (sg.begin / TILE + tile) * (int64_t)TILE;
        const int64_t lo = sg.begin > tbase ? sg.begin : tbase;
        const int64_t hi = sg.end < tbase + TILE ? sg.end : tbase + TILE;
        const U raw = O::from((U)sg.pivot);
        const uint32_t pv = sg.pivot_v;
        store_run<U>((U *)P.a_keys + lo, hi - lo, [&](int64_t) { return raw; });
        if (KV) store_run<uint32_t>(P.a_vals + lo, hi - lo, [&](int64_t) { return pv; });
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            sh.s_bytes += (unsigned long long)ELEM_BYTES * (hi - lo);
            finish_keys(P, (unsigned long long)(hi - lo));
        }
    }

    __device__ static void zero_counters(Shared &sh) {
        sh.s_part_right = sh.s_part_left = sh.s_bad = sh.s_fallback = sh.s_base = sh.s_tiles = sh.s_bytes = 0;
        sh.s_max_depth = 0;
    }
    __device__ static void flush_counters(const Params &P, Shared &sh) {
        State *st = P.st;
        if (sh.s_part_right) atomicAdd(&st->c_part_right, sh.s_part_right);
        if (sh.s_part_left) atomicAdd(&st->c_part_left, sh.s_part_left);
        if (sh.s_bad) atomicAdd(&st->c_bad, sh.s_bad);
        if (sh.s_fallback) atomicAdd(&st->c_fallback, sh.s_fallback);
        if (sh.s_base) atomicAdd(&st->c_base, sh.s_base);
        if (sh.s_tiles) atomicAdd(&st->c_tiles, sh.s_tiles);
        if (sh.s_bytes) atomicAdd(&st->c_bytes, sh.s_bytes);
        if (sh.s_max_depth) atomicMax(&st->c_max_depth, (unsigned long long)sh.s_max_depth);
    }
};

// ---- K4: adjacent-compare reduction with early exit ---------------------------------------------
template <class U, bool FLOAT, bool KV>
__global__ void __launch_bounds__(THREADS) k_check(Params P) {
    using O = Ord<U, FLOAT>;
    __shared__ unsigned s_stop;
    const int tid = threadIdx.x;
    const U *a = (const U *)P.a_keys;
    const int64_t n = P.n;
    const int64_t CH = (int64_t)THREADS * ITEMS;
    unsigned long long bytes = 0;
    for (int64_t c0 = (int64_t)blockIdx.x * CH; c0 < n - 1; c0 += (int64_t)gridDim.x * CH) {
        if (tid == 0) s_stop = (ld_volatile_u32(&P.st->check_bits) == 3u);
        __syncthreads();
        if (s_stop) break;
        unsigned bits = 0;
        const int64_t i0 = c0 + (int64_t)tid * ITEMS;
        if (i0 < n - 1) {
            uint64_t prev = (uint64_t)O::to(a[i0]);
            uint32_t pvv = KV ? P.a_vals[i0] : 0u;
            const int64_t lim = (i0 + ITEMS < n - 1) ? i0 + ITEMS : n - 1;
            for (int64_t i = i0 + 1; i <= lim; ++i) {
                const uint64_t cur = (uint64_t)O::to(a[i]);
                const uint32_t cv = KV ? P.a_vals[i] : 0u;
                bits |= pless<KV>(cur, cv, prev, pvv) ? 1u : 0u;
                bits |= pless<KV>(prev, pvv, cur, cv) ? 2u : 0u;
                prev = cur;
                pvv = cv;
            }
        }
        bits = __reduce_or_sync(0xffffffffu, bits);
        if ((tid & 31) == 0 && bits) atomicOr(&P.st->check_bits, bits);
        const int64_t hi = c0 + CH < n ? c0 + CH : n;
        bytes += (unsigned long long)(hi - c0) * (sizeof(U) + (KV ? 4 : 0));
        __syncthreads();
    }
    if (tid == 0 && bytes) atomicAdd(&P.st->c_bytes_check, bytes);
}

// ---- init: decide from K4, reverse flag, root segment --------------------------------------------
template <class U, bool FLOAT, bool KV>
__global__ void __launch_bounds__(THREADS) k_init(Params P) {
    using S = Sorter<U, FLOAT, KV>;
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ Shared sh;
    __shared__ int s_action;
    U *sk = reinterpret_cast<U *>(dsm);
    uint32_t *sv = reinterpret_cast<uint32_t *>(dsm + 2 * sizeof(U) * TILE);
    const int tid = threadIdx.x;
    if (tid == 0) {
        S::zero_counters(sh);
        const unsigned bits = P.st->check_bits;
        int action = 0;  // 0 = sort, 1 = done (sorted), 2 = reverse
        if (P.n <= 1) action = 1;
        else if (P.use_check && !(bits & 1u)) action = 1;
        else if (P.use_check && !(bits & 2u)) action = 2;
        s_action = action;
        if (action == 1) {
            P.st->keys_final = P.n;
            P.st->done = 1;
        } else if (action == 2) {
            P.st->reverse = 1;
            P.st->keys_final = P.n;
            P.st->done = 1;
            sh.s_bytes += 2ull * (sizeof(U) + (KV ? 4 : 0)) * (unsigned long long)P.n;
        }
    }
    __syncthreads();
    if (s_action == 0) {
        int budget = P.budget0;
        if (budget < 0) {  // driver.py:263: n.bit_length() - 1
            budget = 63 - __clzll((long long)P.n);
        }
        S::spawn(P, sh, sk, sv, 0, P.n, false, false, 0, 0, budget, 0, false, -1);
    }
    __syncthreads();
    if (tid == 0) S::flush_counters(P, sh);
}

// ---- K6: the persistent segment-queue sorter -----------------------------------------------------
template <class U, bool FLOAT, bool KV>
__global__ void __launch_bounds__(THREADS) k_sort(Params P) {
    using S = Sorter<U, FLOAT, KV>;
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ Shared sh;
    U *sk = reinterpret_cast<U *>(dsm);
    U *ck = sk + TILE;
    uint32_t *sv = reinterpret_cast<uint32_t *>(dsm + 2 * sizeof(U) * TILE);
    uint32_t *cv = sv + TILE;
    const int tid = threadIdx.x;

    // K4 reverse: a non-increasing input is reversed in place (one read + one write pass)
    if (ld_volatile_u32(&P.st->reverse)) {
        U *a = (U *)P.a_keys;
        const int64_t half = P.n / 2;
        for (int64_t i = (int64_t)blockIdx.x * THREADS + tid; i < half; i += (int64_t)gridDim.x * THREADS) {
            const int64_t j = P.n - 1 - i;
            U x = a[i];
            a[i] = a[j];
            a[j] = x;
            if (KV) {
                uint32_t y = P.a_vals[i];
                P.a_vals[i] = P.a_vals[j];
                P.a_vals[j] = y;
            }
        }
        return;
    }
    if (tid == 0) {
        S::zero_counters(sh);
        mbar_init(&sh.bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned phase = 0;
    const uint64_t mask = (1ull << P.log_q) - 1;
    for (;;) {
        if (tid == 0) {
            const unsigned long long pos = atomicAdd(&P.st->q_head, 1ull);
            const uint64_t want = (pos >> P.log_q) & 0xFFFFull;
            const uint64_t *slot = P.ring + (pos & mask);
            uint64_t w;
            unsigned ns = 32;
            const uint64_t t0 = globaltimer_ns();
            for (;;) {
                w = ld_acquire_u64(slot);
                if ((w >> 48) == want) break;
                if (ld_volatile_u32(&P.st->done)) {
                    w = 0;
                    break;
                }
                __nanosleep(ns);
                if (ns < 1024) ns <<= 1;
                if (globaltimer_ns() - t0 > WATCHDOG_NS) {  // no task for 10 s: report, never hang
                    S::fail(P, -8);
                    w = 0;
                    break;
                }
            }
            sh.task = w;
            if (w) {
                const uint32_t sid = (uint32_t)(w >> 23) & 0x3FFFFF;
                const ulonglong2 *gsrc = reinterpret_cast<const ulonglong2 *>(&P.segs[sid]);
                ulonglong2 *sdst = reinterpret_cast<ulonglong2 *>(&sh.seg);
#pragma unroll
                for (int q = 0; q < 8; ++q) sdst[q] = __ldcg(gsrc + q);
            }
        }
        __syncthreads();
        const uint64_t w = sh.task;
        if (!w) break;
        const uint32_t type = (uint32_t)(w >> 45) & 7u;
        const uint32_t sid = (uint32_t)(w >> 23) & 0x3FFFFF;
        const uint32_t tile = (uint32_t)w & 0x7FFFFF;
        if (type == T_PART)
            S::part_tile(P, sh, sk, sv, ck, cv, sid, tile, phase);
        else
            S::fill_tile(P, sh, tile);
        __syncthreads();
    }
    if (tid == 0) S::flush_counters(P, sh);
}

}  // namespace pdq
