// kernels.h — device-side descriptors and launchers of the sm_100a kernels (internal).
//
// Arithmetic contract shared with nothing but DESIGN.md §3: FP32 round-to-nearest-even, explicit
// __fadd_rn/__fsub_rn/__fmaf_rn/__fdiv_rn in the orders written in DESIGN.md (D20), images in 8-bit
// units (D5), zero padding (D9).  Compiled with -fmad=false so nothing else is ever contracted.
//
// Data layout:
//  * float4 pyramids [slot][level-major texels] (RGB + 0) for remap inputs and packing;
//  * packed PatchMatch operands with a zero border of kBorder texels on every side (so patch taps never
//    need bounds checks: out-of-image taps read the border's zeros, reading D9) and an even pitch:
//      source  SF8  (level 0, uint8 style): uint2 {G rgb u8, S rgb u8 | 1 << 24 inside the image}  8 B
//              SF10 (level 1, uint8 style): uint2 {G, S} of 10-bit fields n = 4 v (r | g << 10 | b << 20),
//                   exact because level-1 values are multiples of 1/4 (D6); two copies like SF8        8 B
//              SF16 (levels 2..4, uint8 style): uint4 of u16 n = v * 4^k {G.r,G.g | G.b,0 |
//                   S.r,S.g | S.b,0}; exact because level-k values are multiples of 4^-k (D6) 16 B
//              SF8F (level 0, float style, e.g. blending-table cells): uint4 {G rgb u8, S.r, S.g, S.b
//                   as f32}; the guide is still u8-exact at level 0                              16 B
//              SF32 (otherwise):           float4 {G.r,G.g,G.b,S.r}, float4 {S.g,S.b,0,0}     32 B
//      target  TF16 (with SF8):            uint4  {G rgb u8, aux.r, aux.g, aux.b (f32 bits)}  16 B
//              TF10 (with SF10, level 1):  uint4  {G as SF10 10-bit fields, aux.r, aux.g, aux.b}  16 B
//              TF32 (with SF32):           float4 {G.r,G.g,G.b,aux.r}, float4 {aux.g,aux.b,0,0} 32 B
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fbk {

constexpr int kBorder = 4;  // >= the largest compiled patch radius
#ifndef FB_SF8_COPIES
#define FB_SF8_COPIES 2      // SF8 planes stored twice, copy 1 shifted left by one texel: every patch row
#endif                       // starts 16-byte aligned in copy (col & 1), so no parity selects are needed
constexpr int kSF8Copies = FB_SF8_COPIES;

enum SrcFmt { SF8 = 0, SF32 = 1, SF16 = 2, SF8F = 3, SF10 = 4 };
enum TgtFmt { TF16 = 0, TF32 = 1, TF10 = 2 };

// One NNF task (pair).
struct DTask {
    const char* src;   // packed source pyramid of the task's source slot (level k at +FieldArgs::src_off)
    char* tgt;         // packed target operand of the current level (per task, or shared by a MEAN_ALIGN group)
    const float4* ss;  // source style float4 pyramid (remap input of the S^ refresh)
    const float4* tg;  // target guide float4 pyramid (guide half of the packed target)
    uint32_t c2;       // Philox counter word 2: source frame id (D21)
    uint32_t c3;       // Philox counter word 3: tag << 28 | target frame id (D21)
    const char* psrc;  // PAIRWISE (Eq. 10): the counterpart task's packed source slot (its keyframe style)
    const int2* pF;    // PAIRWISE: the counterpart's NNF at the start of the iteration (D39), [h_k*w_k]
    const int2* trk[2];  // tracking (D42): NNFs of the tasks for T_{i-1}, T_{i+1} at the iteration start
};

// Geometry of one pyramid level (unpadded float4 pyramids).
struct Lvl {
    int h, w;
    long long off;  // texel offset of this level inside a float4 pyramid
};

// Padded geometry of one level of the packed operands: texel (r,c) at (r+kBorder)*pitch + c+kBorder.
struct PLvl {
    int h, w, pitch, rows;  // rows = h + 2*kBorder
    int k;                  // pyramid level (selects the SF16 scale 4^k)
};

// Combine: out = (fma-accumulate over the ordered members of w_m * Y_m) / div, where Y_m is an image
// (task < 0) or the Alg. 2 remap of `img` under the current NNF of task `task` (D19).
struct DMember {
    const float4* img;  // image at the combine's level (already offset to the level)
    int task;           // -1: plain image; >= 0: remap img with F of this task
    float w;            // weight (exact powers of two, 1, -1, or the Eq. 9 weights)
    const char* slot;   // optional packed source slot level block holding the same image exactly
    int sfmt;           // slot format (SF8 / SF16) or -1: remap reads 4/8 bytes per tap instead of 16
};
struct DOut {
    int m0, nm;           // member range
    float div;            // IEEE divisor applied last (1 = none)
    int fmt;              // 0: float4 [h*w]; 1: float [h*w*3] (API layout); 2: packed TF16; 3: packed TF32
    void* out;
    const float4* guide;  // fmt 2/3: target guide at this level (the G half of the packed target)
};

struct Rng {
    uint32_t k0, k1;  // Philox key = seed
};

struct FieldArgs {
    const DTask* tasks;
    const int2* Fin;
    int2* Fout;
    float* E;
    long long fstride;  // elements per task in F/E buffers
    PLvl L;
    long long src_off;  // byte offset of this level inside each packed source pyramid
    int tiles_x, tiles_per_task;
    float alpha;
    Rng rng;
    uint32_t level, iter;  // for the Philox counter (D21)
    int rs_r0, rs_k;       // random-search radius r0 and step count at this level (D13, D33)
    int src_fmt;           // SF16 or SF32 for the general kernel; SF8 or SF8F for the fast kernels
    int step;              // propagation step (jump flood scale, D41; 1 = P:72)
    int einit;             // phase 0 recomputes E <- L(F) (first field of the iteration)
    int do_rs;             // phase 3 runs the random search (last field of the iteration)
    float* Eout;           // fused fields 1-3: final E (nullable); E itself is read-only there
    int tgt_reg_rows;      // fused fields 1-3 (p = 2): target patch rows held in registers (0 = all)
    int pair0;             // general kernel phase 0 with E init: score E and the field-0 candidate together
    long long sum_off;     // byte offset of this level's patch-sum plane inside each source slot, or -1 (none):
                           // the random search then rejects candidates by the patch-sum bound
    long long tail_off;    // byte offset of the tail-row sums plane (SumJob::tail), or -1: the fused level-0
                           // kernel's random search then adds the partial + remainder bound
};

// Patch sums of a packed source level block (SF8 at level 0, SF10 at level 1, SF16 above, SF8F): for every texel
// (r, c) of the level, the sums over its (2p+1)^2 patch (zero padding, D9) of the integer fields n of each guide
// and style channel, as uint4 {lo, hi} of 21-bit fields (lo = sG.r | sG.g << 21 | sG.b << 42, hi the same of sS)
// at [r * w + c]; every sum is below 2^21 (checked by the caller).  SF8F: two uint4 per texel (see k_patch_sums).
// `tail` (SF8 only, nullable): the sums over the patch's last rows [tail_r0, 2p+1) -- the rows the fused level-0
// kernel scores after its partial-distance check -- as uint4 {G.r | G.g << 16, G.b | S.r << 16, S.g | S.b << 16, 0}.
struct SumJob {
    const char* blk;  // packed level block (copy 0)
    uint4* sums;      // [h * w]
    uint4* tail;      // [h * w] or NULL
};

// Packing jobs: one per (slot, level) for sources, one per task/group for BASE targets.
struct PackSrc {
    const uint8_t* g8;   // SF8: guide frame uint8 [H,W,3]
    const uint8_t* s8;   // SF8: style frame uint8 [H,W,3]
    const float4* gp;    // SF32: guide pyramid level pointer
    const float4* sp;    // SF32: style pyramid level pointer
    char* out;           // packed level block
};

// ---- launchers (return cudaGetLastError()) ---------------------------------------------------
cudaError_t launch_u8_to_pyr0(const uint8_t* frames, float4* pyr, int B, int H, int W, long long pyr_stride,
                              cudaStream_t s);
cudaError_t launch_box(float4* pyr, int B, long long pyr_stride, Lvl prev, Lvl cur, cudaStream_t s);
cudaError_t launch_pack_src(const PackSrc* jobs, int n, int fmt, PLvl L, cudaStream_t s);
cudaError_t launch_patch_sums(const SumJob* jobs, int n, int fmt, PLvl L, int p, cudaStream_t s);
// first tail row of SumJob::tail for patch radius p (the fused level-0 kernel's partial-distance check row)
int tail_row0(int p);
cudaError_t launch_pack_tgt_guide(const DTask* tasks, int T, Lvl L, PLvl P, int tfmt, cudaStream_t s);
cudaError_t launch_init(const DTask* tasks, int T, int2* F, long long fstride, Lvl L, int identity, Rng rng,
                        uint32_t level, cudaStream_t s);
cudaError_t launch_upsample(const int2* Fc, int2* Ff, int T, long long fstride, Lvl Lc, Lvl Lf, cudaStream_t s);
// sfmt: SF8 / SF16 remaps the style held in the task's packed source slot (level block at src_off), any
// other value the float4 style pyramid.
cudaError_t launch_aux_remap(const DTask* tasks, int T, const int2* F, long long fstride, Lvl L, PLvl P, int p,
                             int tfmt, int sfmt, long long src_off, cudaStream_t s);
cudaError_t launch_combine(const DOut* outs, int n_outs, const DMember* mem, const int2* F, long long fstride,
                           int h, int w, int p, int fmt, PLvl P, cudaStream_t s);
// phase 0: E init + propagation (-1,0); 1: (+1,0); 2: (0,-1); 3: (0,+1) + all random-search steps.
// kind: 0 general (SF16/SF32 source, TF32 target tile in smem), 1 fast (SF8/SF8F, TF16 target patch in
// registers, p <= 2), 2 mid (16-byte target tile in smem: level 0 SF8/SF8F + TF16, or level 1 SF10 + TF10
// at p = 2).
// loss: fb_loss (0 BASE, 1 GUIDE_STYLE, 2 MEAN_ALIGN, 3 PAIRWISE).
cudaError_t launch_field(const FieldArgs& a, int T, int p, int loss, int phase, int kind, cudaStream_t s);
// The whole updating sequence of one iteration (E init, four propagation fields, random search) in one
// launch, fast operands only (SF8/TF16, p <= 2).  Fin -> Fout, E written.
cudaError_t launch_iter_fast(const FieldArgs& a, int T, int p, int loss, cudaStream_t s);
// Fields 1-3 and the random search of one iteration in one launch (fast operands: SF8/SF8F + TF16 at
// level 0, SF10 + TF10 at level 1 for p = 2); Fin holds the field-0 result and E its errors.  Fin -> Fout.
cudaError_t launch_iter13_fast(const FieldArgs& a, int T, int p, int loss, cudaStream_t s);
cudaError_t launch_remap_f3(const float* src, const int2* F, float* out, int B, int H, int W, int p,
                            cudaStream_t s);

}  // namespace fbk
