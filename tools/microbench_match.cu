// Microbenchmark (profiling aid): throughput of __match_any_sync vs __shfl_sync on sm_100a.
#include <cstdio>
#include <cstdint>
__global__ void k_match(const uint32_t *in, uint32_t *out, int iters) {
    uint32_t x = in[threadIdx.x + blockIdx.x * blockDim.x], acc = 0;
    for (int i = 0; i < iters; ++i) {
        uint32_t m = __match_any_sync(0xffffffffu, (x + i) & 255u);
        acc += m;
        x ^= m;
    }
    out[threadIdx.x + blockIdx.x * blockDim.x] = acc;
}
__global__ void k_shfl(const uint32_t *in, uint32_t *out, int iters) {
    uint32_t x = in[threadIdx.x + blockIdx.x * blockDim.x], acc = 0;
    for (int i = 0; i < iters; ++i) {
        uint32_t m = __shfl_xor_sync(0xffffffffu, (x + i) & 255u, 1);
        acc += m;
        x ^= m;
    }
    out[threadIdx.x + blockIdx.x * blockDim.x] = acc;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int blocks = sms * 8, threads = 256, iters = 4096;
    uint32_t *in, *out; cudaMalloc(&in, blocks * threads * 4); cudaMalloc(&out, blocks * threads * 4);
    cudaMemset(in, 7, blocks * threads * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
    for (int r = 0; r < 2; ++r) {
        cudaEventRecord(a); k_match<<<blocks, threads>>>(in, out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double warp_ops = (double)blocks * threads / 32 * iters;
        printf("match_any: %.3f ms  %.2f warp-ops/clk/SM (at 1.9 GHz)\n", ms, warp_ops / (ms * 1e-3) / sms / 1.9e9);
        cudaEventRecord(a); k_shfl<<<blocks, threads>>>(in, out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("shfl:      %.3f ms  %.2f warp-ops/clk/SM\n", ms, warp_ops / (ms * 1e-3) / sms / 1.9e9);
    }
    return 0;
}
