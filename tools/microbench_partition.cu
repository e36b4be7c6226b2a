// Microbenchmark (profiling aid, not product code): raw throughput of one 2-way partition pass of
// n uint32 keys with a fixed pivot, each CTA owning a static set of 4096-key tiles, with
// (a) direct 128-bit global loads into registers and (b) one packed 64-bit reservation atomic per
// tile, then shared-memory compaction and 16-byte stores.  Compares against a plain copy.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_partition.cu && /tmp/mb 28
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int THREADS = 256, ITEMS = 16, TILE = THREADS * ITEMS;

__global__ void __launch_bounds__(THREADS) copy_kernel(const uint4 *a, uint4 *b, int64_t n4) {
    for (int64_t i = blockIdx.x * (int64_t)THREADS + threadIdx.x; i < n4; i += (int64_t)gridDim.x * THREADS) b[i] = a[i];
}

template <int MINB>
__global__ void __launch_bounds__(THREADS, MINB) part_kernel(const uint32_t *src, uint32_t *dst, int64_t n,
                                                           uint32_t piv, unsigned long long *cnt) {
    __shared__ uint32_t kc[TILE];
    __shared__ uint32_t wsum[THREADS / 32];
    __shared__ unsigned long long off;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = n / TILE;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src + t * TILE);
        uint32_t k[ITEMS];
#pragma unroll
        for (int j = 0; j < ITEMS / 4; ++j) {
            uint4 v = s4[j * THREADS + tid];
            k[4 * j] = v.x; k[4 * j + 1] = v.y; k[4 * j + 2] = v.z; k[4 * j + 3] = v.w;
        }
        unsigned lm = 0;
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) lm |= (unsigned)((int)k[r] < (int)piv) << r;
        const int nl = __popc(lm);
        const uint32_t mine = nl | ((ITEMS - nl) << 16);
        uint32_t inc = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(~0u, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        uint32_t wpre = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < THREADS / 32; ++w) { uint32_t x = wsum[w]; wpre += w < warp ? x : 0; tot += x; }
        const int L = tot & 0xFFFF, R = tot >> 16;
        if (tid == 0) off = atomicAdd(cnt, (unsigned long long)L | ((unsigned long long)R << 32));
        const uint32_t pre = wpre + inc - mine;
        int li = pre & 0xFFFF, ri = L + (pre >> 16);
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
            const bool isl = (lm >> r) & 1;
            kc[isl ? li : ri] = k[r];
            li += isl; ri += !isl;
        }
        __syncthreads();
        const long long lo = (long long)(off & 0xffffffffull), ro = (long long)(off >> 32);
        // left run at [lo, lo+L), right run at n - ro - R (scalar-coalesced stores; alignment arbitrary)
        for (int i = tid; i < L; i += THREADS) dst[lo + i] = kc[i];
        for (int i = tid; i < R; i += THREADS) dst[n - ro - R + i] = kc[L + i];
        __syncthreads();
    }
}

int main(int argc, char **argv) {
    int lg = argc > 1 ? atoi(argv[1]) : 28;
    int64_t n = 1ll << lg;
    uint32_t *a, *b;
    unsigned long long *cnt;
    cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&cnt, 8);
    uint32_t *h = (uint32_t *)malloc(n * 4);
    uint64_t x = 88172645463325252ull;
    for (int64_t i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (uint32_t)x; }
    cudaMemcpy(a, h, n * 4, cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        copy_kernel<<<sms * 8, THREADS>>>((const uint4 *)a, (uint4 *)b, n / 4);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("copy: %.3f ms  %.0f GB/s\n", ms, 2.0 * n * 4 / ms / 1e6);
    auto run = [&](auto kern, int minb, const char *name) {
        int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, 0);
        for (int g : {1, 2}) {
            int grid = sms * occ * g;
            for (int rep = 0; rep < 3; ++rep) {
                cudaMemset(cnt, 0, 8);
                cudaEventRecord(e0);
                kern<<<grid, THREADS>>>(a, b, n, 0u, cnt);
                cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
            }
            printf("%s occ %d grid %d: %.3f ms  %.0f GB/s  err=%s\n", name, occ, grid, ms, 2.0 * n * 4 / ms / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
        }
    };
    run(part_kernel<2>, 2, "part minb2");
    run(part_kernel<4>, 4, "part minb4");
    run(part_kernel<6>, 6, "part minb6");
    return 0;
}
