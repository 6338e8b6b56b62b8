// l1_peak_bench.cu — measured L1 / shared data-path peak of the B200 for the PatchMatch roofline
// (bench.py `roofline`).  Prints one JSON object (committed as profiles/l1_peak.json).
//
//   (a) ldg128_l1hit: every warp streams LDG.128 over a 16 KiB per-CTA window that stays L1-resident
//       (32 lanes x 16 B = 512 B = 4 wavefronts per instruction, all hits): the L1 data-path ceiling in B/s.
//   (b) lds128: the same through LDS.128 from shared memory (the shared half of the same data path).
//   (c) rows_l2: the PatchMatch random-search pattern -- each lane gathers 5-texel rows (3 x LDG.128 from the
//       16-byte-aligned copy of an 8-byte-texel 520x520 plane, the SF8 level-0 source) at random positions,
//       the whole plane (4.3 MB in two copies) L2-resident: rows/s and the L1 wavefront-equivalent rate.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l1_peak_bench tools/l1_peak_bench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

// (a) L1-resident LDG.128: CTA b reads window b % nwin (16 KiB), each warp walks it in 512 B steps.
__global__ void __launch_bounds__(256) k_ldg_l1(const uint4* __restrict__ buf, int iters, uint32_t* out)
{
    const uint4* w = buf + (size_t)(blockIdx.x % 64) * 1024;  // 1024 x 16 B = 16 KiB per window
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t acc = 0;
    int idx = warp * 32 + lane;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint4 v = __ldg(w + ((idx + k * 128) & 1023));
            acc += v.x ^ v.y ^ v.z ^ v.w;
        }
        idx += 256;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// (b) LDS.128 over a 16 KiB shared window.
__global__ void __launch_bounds__(256) k_lds(int iters, uint32_t* out)
{
    __shared__ uint4 s[1024];
    for (int i = threadIdx.x; i < 1024; i += 256) s[i] = make_uint4(i, i * 3, i * 5, i * 7);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t acc = 0;
    int idx = warp * 32 + lane;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint4 v = s[(idx + k * 128) & 1023];
            acc += v.x ^ v.y ^ v.z ^ v.w;
        }
        idx += 256 + (acc & 1);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// (c) random 5-texel rows (3 x LDG.128) from the SF8-like plane, copy chosen by column parity.
__global__ void __launch_bounds__(128) k_rows(const uint2* __restrict__ plane, int pitch, int rows, int W, int H,
                                              int iters, uint32_t* out)
{
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        const uint32_t h = hash(tid * 2654435761u + it * 97u);
        const int r = (int)(h % (uint32_t)H) + 2, c = (int)((h >> 12) % (uint32_t)W) + 2;
        const int idx = r * pitch + c;
        const uint4* p = reinterpret_cast<const uint4*>(plane + (size_t)(idx & 1) * rows * pitch + (idx & ~1));
#pragma unroll
        for (int k = 0; k < 3; ++k) { const uint4 v = __ldg(p + k); acc += v.x ^ v.y ^ v.z ^ v.w; }
    }
    out[tid] = acc;
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    const int blocks = sms * 8;
    uint4* buf;
    uint32_t* out;
    CK(cudaMalloc(&buf, 64 * 16384));
    CK(cudaMemset(buf, 1, 64 * 16384));
    CK(cudaMalloc(&out, sizeof(uint32_t) * blocks * 256));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    auto time_ms = [&](auto&& launch) {
        launch();
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            CK(cudaEventRecord(a));
            launch();
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            best = ms < best ? ms : best;
        }
        return best;
    };
    const int it_a = 4096;
    const float ms_a = time_ms([&] { k_ldg_l1<<<blocks, 256>>>(buf, it_a, out); });
    const double bytes_a = (double)blocks * 256 * it_a * 8 * 16;
    const float ms_b = time_ms([&] { k_lds<<<blocks, 256>>>(it_a, out); });
    const double bytes_b = bytes_a;
    // (c) 512x512 level-0 plane with a 4-texel zero border, pitch multiple of 4, two copies
    const int W = 512, H = 512, pitch = (W + 8 + 3) & ~3, rows = H + 8;
    uint2* plane;
    CK(cudaMalloc(&plane, sizeof(uint2) * 2 * rows * pitch + 64));
    CK(cudaMemset(plane, 3, sizeof(uint2) * 2 * rows * pitch + 64));
    const int it_c = 2048, blocks_c = sms * 16;
    const float ms_c = time_ms([&] { k_rows<<<blocks_c, 128>>>(plane, pitch, rows, W - 4, H - 4, it_c, out); });
    const double rowsps = (double)blocks_c * 128 * it_c / (ms_c * 1e-3);
    const double nominal = (double)sms * 128.0 * 1965e6;
    printf("{\"l1_peak_gbs\": %.1f, \"lds_peak_gbs\": %.1f, \"nominal_gbs\": %.1f, \"sms\": %d, \"clock_rate_khz\": %d, "
           "\"random_rows_per_s\": %.4e, \"random_row_lane_loads_per_s\": %.4e, "
           "\"how\": \"tools/l1_peak_bench.cu: (a) LDG.128 over L1-resident 16 KiB windows, best of 5, %d CTAs x 256 "
           "threads; (b) LDS.128; (c) random 5-texel SF8 rows, 3 x LDG.128, 520x520 plane in L2\"}\n",
           bytes_a / (ms_a * 1e-3) / 1e9, bytes_b / (ms_b * 1e-3) / 1e9, nominal / 1e9, sms, clk, rowsps, 3 * rowsps, blocks);
    return 0;
}
