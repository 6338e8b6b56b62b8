// tma_gather_bench.cu — microbenchmark: can the TMA unit serve PatchMatch's scattered patch gathers?
//
// Each thread repeatedly fetches a (2p+2) x (2p+1) box of 8-byte texels (the SF8 source patch of one
// random-search candidate, 48 B x 5 rows = 240 B at p=2) at a random position, either
//   mode 0: with plain per-thread global loads (3 x LDG.128 per row, the current kernel's pattern), or
//   mode 1: with one cp.async.bulk.tensor.2d per patch into the thread's own shared-memory slot,
// then reduces the bytes so the loads are not dead.  Reports patches/s for the whole GPU.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_gather_bench tma_gather_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr int BW = 6, BH = 5;  // box: 6 texels (48 B) x 5 rows

__device__ __forceinline__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

__global__ void k_ldg(const uint2* __restrict__ img, int W, int H, int iters, uint32_t* out, int radius)
{
    uint32_t acc = 0;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    int x = hash(tid) % (W - 8), y = hash(tid * 7 + 1) % (H - 8);
    for (int it = 0; it < iters; ++it) {
        const uint32_t h = hash(tid * 1315423911u + it);
        int nx = x + (int)(h % (2 * radius + 1)) - radius, ny = y + (int)((h >> 16) % (2 * radius + 1)) - radius;
        nx = min(max(nx, 0), W - 8); ny = min(max(ny, 0), H - 6);
        const int o = nx & 1;
#pragma unroll
        for (int r = 0; r < BH; ++r) {
            const uint4* p = reinterpret_cast<const uint4*>(img + (size_t)(ny + r) * W + nx - o);
#pragma unroll
            for (int k = 0; k < 3; ++k) { uint4 v = __ldg(p + k); acc += v.x ^ v.y ^ v.z ^ v.w; }
        }
        if (acc & 1) { x = nx; y = ny; }  // data-dependent next center, like the RS chain
    }
    out[tid] = acc;
}

__device__ __forceinline__ void ldg256(const void* p, uint32_t (&w)[8])
{
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
}

// variant: shape 1 = 5 x LDG.64 per row; shape 2 = 2 x LDG.256 per row (32-byte aligned window)
template <int SHAPE>
__global__ void k_ldg_shape(const uint2* __restrict__ img, int W, int H, int iters, uint32_t* out, int radius)
{
    uint32_t acc = 0;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    int x = hash(tid) % (W - 8), y = hash(tid * 7 + 1) % (H - 8);
    for (int it = 0; it < iters; ++it) {
        const uint32_t h = hash(tid * 1315423911u + it);
        int nx = x + (int)(h % (2 * radius + 1)) - radius, ny = y + (int)((h >> 16) % (2 * radius + 1)) - radius;
        nx = min(max(nx, 0), W - 8); ny = min(max(ny, 0), H - 6);
#pragma unroll
        for (int r = 0; r < BH; ++r) {
            if (SHAPE == 1) {
                const uint2* p = img + (size_t)(ny + r) * W + nx;
#pragma unroll
                for (int k = 0; k < 5; ++k) { uint2 v = __ldg(p + k); acc += v.x ^ v.y; }
            } else {
                const uint2* p = img + (size_t)(ny + r) * W + (nx & ~3);
                uint32_t q[8];
                ldg256(p, q); acc += q[0] ^ q[3] ^ q[5] ^ q[7];
                ldg256(p + 4, q); acc += q[0] ^ q[3] ^ q[5] ^ q[7];
            }
        }
        if (acc & 1) { x = nx; y = ny; }
    }
    out[tid] = acc;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase)
{
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
                 :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(phase));
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(map), "r"(x), "r"(y),
                    "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}

template <int TPB>
__global__ void __launch_bounds__(TPB) k_tma(const __grid_constant__ CUtensorMap map, int W, int H, int iters, uint32_t* out, int radius)
{
    __shared__ __align__(128) uint2 buf[TPB][32];  // 256 B slot per thread (240 used)
    __shared__ uint64_t bars[TPB];
    const int t = threadIdx.x;
    mbar_init(&bars[t], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t acc = 0, phase = 0;
    const int tid = blockIdx.x * blockDim.x + t;
    int x = hash(tid) % (W - 8), y = hash(tid * 7 + 1) % (H - 8);
    for (int it = 0; it < iters; ++it) {
        const uint32_t h = hash(tid * 1315423911u + it);
        int nx = x + (int)(h % (2 * radius + 1)) - radius, ny = y + (int)((h >> 16) % (2 * radius + 1)) - radius;
        nx &= ~1;  // TMA: the inner box start must be 16-byte aligned (measured: odd 8-byte starts trap)
        mbar_expect_tx(&bars[t], BW * BH * 8);
        __syncwarp();
        const int lane = t & 31, wb = t & ~31;
        for (int l = 0; l < 32; ++l) {  // one lane issues the warp's 32 box loads (TMA issue is warp-scalar)
            const int xl = __shfl_sync(~0u, nx, l), yl = __shfl_sync(~0u, ny, l);
            if (lane == 0) tma_load_2d(buf[wb + l], &map, &bars[wb + l], xl, yl);  // OOB -> zero fill
        }
        mbar_wait(&bars[t], phase);
        phase ^= 1;
#pragma unroll
        for (int k = 0; k < BW * BH; k += 2) {
            const uint4 v = *reinterpret_cast<const uint4*>(&buf[t][(k + 2 * t) % 30]);  // stagger banks
            acc += v.x ^ v.y ^ v.z ^ v.w;
        }
        if (acc & 1) { x = min(max(nx, 0), W - 8); y = min(max(ny, 0), H - 6); }
    }
    out[tid] = acc;
}

int main(int argc, char** argv)
{
    const int W = 520, H = 520, NIMG = 1;
    const int radius = argc > 1 ? atoi(argv[1]) : 256;
    std::vector<uint2> h((size_t)W * H * NIMG);
    for (size_t i = 0; i < h.size(); ++i) h[i] = make_uint2((uint32_t)i * 2654435761u, (uint32_t)i);
    uint2* d; CK(cudaMalloc(&d, h.size() * 8)); CK(cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    const int threads = 148 * 384, iters = 200;
    uint32_t* out; CK(cudaMalloc(&out, threads * 4));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        k_ldg<<<threads / 128, 128>>>(d, W, H, iters, out, radius);
        cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    }
    printf("LDG  radius %d: %.2f G patches/s (%.2f ms)\n", radius, (double)threads * iters / ms / 1e6, ms);
    for (int shape = 1; shape <= 2; ++shape) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (shape == 1) k_ldg_shape<1><<<threads / 128, 128>>>(d, W, H, iters, out, radius);
            else k_ldg_shape<2><<<threads / 128, 128>>>(d, W, H, iters, out, radius);
            cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
        }
        printf("LDG shape %s radius %d: %.2f G patches/s\n", shape == 1 ? "5xLDG.64" : "2xLDG.256", radius,
               (double)threads * iters / ms / 1e6);
    }
    CUtensorMap map;
    cuuint64_t gdim[2] = {(cuuint64_t)W, (cuuint64_t)H};
    cuuint64_t gstride[1] = {(cuuint64_t)W * 8};
    cuuint32_t box[2] = {BW, BH}, estride[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, d, gdim, gstride, box, estride,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    for (int tpb : {64, 128}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (tpb == 128) k_tma<128><<<threads / 128, 128>>>(map, W, H, iters, out, radius);
            else if (tpb == 64) k_tma<64><<<threads / 64, 64>>>(map, W, H, iters, out, radius);
            cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
        }
        printf("TMA tpb %d radius %d: %.2f G patches/s (%.2f ms)\n", tpb, radius, (double)threads * iters / ms / 1e6, ms);
    }
    return 0;
}
