// Micro-benchmark (development aid): throughput of u8 -> f32 conversion forms on sm_100a.
//   A: I2F.U8 with byte select (one instruction)       B: PRMT into 0x4B0000xx + FADD (two instructions)
// Each thread converts the 4 bytes of 8 independent words per iteration and folds them with FADD/FFMA the
// way the loss does (sub + fma), so the mix is comparable to the patch loss.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(const uint32_t* __restrict__ in, float* out, int iters, float t)
{
    uint32_t w[8];
    for (int j = 0; j < 8; ++j) w[j] = in[(threadIdx.x + j * 97) & 1023];
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                float v;
                if (MODE == 0) {
                    v = (float)(uint8_t)(w[j] >> (8 * ch));
                } else {
                    v = __fsub_rn(__uint_as_float(__byte_perm(w[j], 0x4B000000u, 0x7440u + ch)), 8388608.0f);
                }
                const float d = __fsub_rn(t, v);
                acc[j] = __fmaf_rn(d, d, acc[j]);
            }
            w[j] = w[j] * 1664525u + 1013904223u;
        }
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main()
{
    uint32_t* in; float* out;
    cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 148 * 8 * 256 * 4);
    cudaMemset(in, 0x5a, 4096 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 2000;
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<148 * 8, 256>>>(in, out, iters, 1.5f);
            else k<1><<<148 * 8, 256>>>(in, out, iters, 1.5f);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            const double conv = 148.0 * 8 * 256 * iters * 8 * 3;
            if (rep) printf("%s: %.3f ms, %.1f G conversions/s (+ sub + fma each), %.1f per SM per clk @1.965GHz\n",
                            mode == 0 ? "I2F.U8 byte-select" : "PRMT+FADD        ", ms, conv / ms / 1e6,
                            conv / (ms * 1e-3) / 148 / 1.965e9);
        }
    }
    return 0;
}
