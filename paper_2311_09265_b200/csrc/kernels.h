// kernels.h — device-side descriptors and launchers of the sm_100a kernels (internal).
//
// Arithmetic contract shared with nothing but DESIGN.md §3: FP32 round-to-nearest-even, explicit
// __fadd_rn/__fsub_rn/__fmaf_rn/__fdiv_rn in the orders written in DESIGN.md (D20), images in 8-bit
// units (D5), zero padding (D9).  Compiled with -fmad=false so nothing else is ever contracted.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fbk {

// One NNF task (pair): pyramid base pointers (level 0; level k starts at +Lvl::off texels) and RNG key.
struct DTask {
    const float4* sg;   // source guide pyramid  G_src
    const float4* tg;   // target guide pyramid  G_tgt
    const float4* ss;   // source style pyramid  S_src (nullptr for BASE)
    float4* aux;        // aux image of this task at the current level (S^ or T-bar), h_k*w_k texels
    uint32_t c2;        // Philox counter word 2: source frame id (D21)
    uint32_t c3;        // Philox counter word 3: tag << 28 | target frame id (D21)
    uint32_t pad0, pad1;
};

// Geometry of one pyramid level.
struct Lvl {
    int h, w;
    long long off;  // texel offset of this level inside a pyramid
};

// Combine: out = (fma-accumulate over the ordered members of w_m * Y_m) / div, where Y_m is an image
// (task < 0) or the Alg. 2 remap of `img` under the current NNF of task `task` (D19).
struct DMember {
    const float4* img;  // image at the combine's level (already offset to the level)
    int task;           // -1: plain image; >= 0: remap img with F of this task
    float w;            // weight (exact powers of two, 1, -1, or the Eq. 9 weights)
};
struct DOut {
    int m0, nm;   // member range
    float div;    // IEEE divisor applied last (1 = none)
    int fmt;      // 0: float4 [h*w] image; 1: float [h*w*3] (API layout)
    void* out;
};

struct Rng {
    uint32_t k0, k1;  // Philox key = seed
};

// Field launch parameters.
struct FieldArgs {
    const DTask* tasks;
    const int2* Fin;
    int2* Fout;
    float* E;
    long long fstride;  // elements per task in F/E buffers
    Lvl L;
    int tiles_x, tiles_per_task;
    float alpha;
    Rng rng;
    uint32_t level, iter;  // for the Philox counter (D21)
    int rs_r0, rs_k;       // random search radius r0 and step count at this level (D13, D33)
};

// ---- launchers (return cudaGetLastError()) ---------------------------------------------------
cudaError_t launch_u8_to_pyr0(const uint8_t* frames, float4* pyr, int B, int H, int W, long long pyr_stride,
                              cudaStream_t s);
cudaError_t launch_box(float4* pyr, int B, long long pyr_stride, Lvl prev, Lvl cur, cudaStream_t s);
cudaError_t launch_init(const DTask* tasks, int T, int2* F, long long fstride, Lvl L, int identity, Rng rng,
                        uint32_t level, cudaStream_t s);
cudaError_t launch_upsample(const int2* Fc, int2* Ff, int T, long long fstride, Lvl Lc, Lvl Lf, cudaStream_t s);
cudaError_t launch_aux_remap(const DTask* tasks, int T, const int2* F, long long fstride, Lvl L, int p,
                             cudaStream_t s);
cudaError_t launch_combine(const DOut* outs, int n_outs, const DMember* mem, const int2* F, long long fstride,
                           int h, int w, int p, cudaStream_t s);
// phase 0: E init + propagation (-1,0); 1: (+1,0); 2: (0,-1); 3: (0,+1) + all random-search steps.
cudaError_t launch_field(const FieldArgs& a, int T, int p, int loss, int phase, cudaStream_t s);
cudaError_t launch_remap_f3(const float* src, const int2* F, float* out, int B, int H, int W, int p,
                            cudaStream_t s);
cudaError_t launch_f4_to_f3(const float4* in, long long in_stride, float* out, int B, int npx, cudaStream_t s);

}  // namespace fbk
