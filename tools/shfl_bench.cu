// Microbenchmark (development aid): per-SM throughput of warp shuffles vs shared-memory LDS.32 / LDS.128 on the
// B200, to decide whether neighbouring lanes should share patch texels by shuffle.  Prints warp-instructions
// per SM-clock for each.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/shfl_bench tools/shfl_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_shfl(unsigned* out, int salt)
{
    unsigned a = threadIdx.x ^ salt, b = a * 3u, c = a * 5u, d = a * 7u;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        a += __shfl_down_sync(0xffffffffu, b, 1);
        b += __shfl_down_sync(0xffffffffu, c, 2);
        c += __shfl_down_sync(0xffffffffu, d, 3);
        d += __shfl_down_sync(0xffffffffu, a, 4);
    }
    if ((a ^ b ^ c ^ d) == 0x12345678u) out[0] = a;
}

__global__ void k_lds128(unsigned* out, int salt)
{
    __shared__ uint4 buf[8][40];
    for (int k = threadIdx.x; k < 8 * 40; k += blockDim.x) buf[k / 40][k % 40] = make_uint4(k, k + 1, k + 2, k + 3);
    __syncthreads();
    const int lane = threadIdx.x & 31, wy = (threadIdx.x >> 5) & 3;
    unsigned acc = salt;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        const uint4 v = buf[wy + (i & 3)][lane + (i & 7)];
        acc += v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void k_lds32(unsigned* out, int salt)
{
    __shared__ unsigned buf[8][160];
    for (int k = threadIdx.x; k < 8 * 160; k += blockDim.x) buf[k / 160][k % 160] = k;
    __syncthreads();
    const int lane = threadIdx.x & 31, wy = (threadIdx.x >> 5) & 3;
    unsigned acc = salt;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) acc += buf[wy + (i & 3)][lane + (i & 7)];
    if (acc == 0x12345678u) out[0] = acc;
}

template <class K>
float run(K kern, int per_iter, const char* name, unsigned* d)
{
    const int blocks = 148 * 8, threads = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    kern<<<blocks, threads>>>(d, 1);
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        kern<<<blocks, threads>>>(d, r);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warp_instr = (double)blocks * threads / 32 * ITERS * per_iter;
    const double per_sm_clk = warp_instr / 148 / (best * 1e-3 * clk * 1e3);
    printf("{\"op\": \"%s\", \"ms\": %.3f, \"warp_instr_per_sm_clk\": %.3f}\n", name, best, per_sm_clk);
    return (float)per_sm_clk;
}

int main()
{
    unsigned* d;
    cudaMalloc(&d, 16);
    run(k_shfl, 4, "SHFL.DOWN (32-bit)", d);
    run(k_lds128, 1, "LDS.128 (512 B per warp)", d);
    run(k_lds32, 1, "LDS.32 (128 B per warp)", d);
    return 0;
}
