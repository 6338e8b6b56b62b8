// kernels.cu — sm_100a kernels of the FastBlend hot path (arXiv 2311.09265).
//
// No tensor cores: the method has no dense contraction (patch distances are gathers of data-dependent
// patches).  The bound resources are the L1/shared data path and the issue rate (ncu: 81-89 % of peak L1
// wavefronts and 65-85 % issue on the top kernels, profiles/r02_v6_*, r02_v5_*); the design minimises the work
// and the load instructions per candidate evaluation: exact elimination (a Cauchy-Schwarz
// patch-sum bound before any patch row is read, partial distances after three rows), 8-byte packed exact
// texels at levels 0-1 (u8, 10-bit), a zero border instead of per-tap bounds checks, target tiles staged by
// the TMA bulk-copy engine, an exact integer guide term (dp4a) where the contract proves it equal to the FP32
// sum, exact integer remap sums, and occupancy bounds tuned per kernel.
//
// Every floating-point operation that decides a result is written with an explicit IEEE intrinsic
// (__fadd_rn, __fsub_rn, __fmaf_rn, __fdiv_rn) in the order DESIGN.md §3 fixes (D20), so the kernels
// are bit-identical to the contract regardless of scheduling or thread mapping.
#include <algorithm>
#include <mutex>
#include <unordered_map>
#include "kernels.h"

#include <algorithm>

namespace fbk {

static constexpr int TILE_X = 32, TILE_Y = 8;  // 256-thread 2D tiles: a warp is one row segment
static constexpr int FAST_TY = 4;              // fast kernel: 128-thread tiles, 3 CTAs/SM at <= 168 regs
static constexpr int B = kBorder;

// Debug bounds checks (build with -DFB_DEBUG_BOUNDS: tools/build_variant.sh dbg -DFB_DEBUG_BOUNDS): every
// gather's texel range is checked against its padded level block and a violation traps the kernel (the
// launch then fails with an error instead of reading a neighbour's data).  No-ops in the product build.
#ifdef FB_DEBUG_BOUNDS
#define FB_ASSERT(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define FB_ASSERT(cond) do { } while (0)
#endif
// Event counters of the fused level-0 kernel (development build with -DFB_COUNTERS: tools/build_variant.sh and
// fb_debug_counters); no-ops in the product build.
#ifdef FB_COUNTERS
__device__ unsigned long long g_fb_cnt[32];
#define FB_CNT(k) atomicAdd(&g_fb_cnt[(k)], 1ull)
#else
#define FB_CNT(k) do { } while (0)
#endif
// a patch row of D texels starting at padded texel idx (rounded down to even, NCH texel pairs) lies in
// the level block and in the row band the zero border provides
#define FB_ROW_OK(idx, L, D) ((idx) >= 0 && ((idx) & ~1) + 2 * (((D) + 2) / 2) <= (L).rows * (L).pitch && \
                              (idx) / (L).pitch >= 0 && (idx) / (L).pitch < (L).rows)

// ------------------------------------------------------------------------------------ Philox4x32-10
// Salmon et al. (SC'11).  Counter layout of D21: c0 = pixel, c1 = purpose<<28 | level<<22 | iter<<12 |
// step, c2 = source frame id, c3 = tag<<28 | target frame id.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        if (i) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

// ---- bulk-copy (TMA engine) staging of target tiles: one thread issues one cp.async.bulk per tile row (a
// contiguous run of 16-byte texels in the padded target plane), completing on an mbarrier the CTA waits on.
#ifndef FB_TILE_TMA
#define FB_TILE_TMA 1
#endif
// Random search of the fused level-0 kernel with the next step's patch-sum texel loaded one step ahead (exact)
#ifndef FB_RS_PREFETCH
#define FB_RS_PREFETCH 0
#endif
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// Stage rows [pr0, pr0 + NY) x columns [pc0, pc0 + NX) of a padded uint4 plane (row pitch `pitch` texels, `rows`
// rows) into tile[NY][NX]: rows / columns beyond the plane are left unwritten -- no valid pixel's patch reaches them
// (the plane's zero border is wider than every patch radius).  Call from all threads; returns with the tile ready.
template <int NY, int NX>
__device__ __forceinline__ void stage_tile_tma(uint4 (&tile)[NY][NX], const uint4* plane, int pitch, int rows, int pr0,
                                               int pc0, uint64_t* bar)
{
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        const int ny = min(NY, rows - pr0), nx = min(NX, pitch - pc0);
        mbar_expect_tx(bar, (uint32_t)(ny * nx * 16));
        for (int y = 0; y < ny; ++y) bulk_g2s(&tile[y][0], plane + (size_t)(pr0 + y) * pitch + pc0, (uint32_t)nx * 16u, bar);
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    mbar_wait(bar, 0);
}

// u8 channel `ch` of a packed rgb word as an exact float: 0x4B0000xx is 2^23 + xx.
__device__ __forceinline__ float u8f(uint32_t word, int ch)
{
    return __fsub_rn(__uint_as_float(__byte_perm(word, 0x4B000000u, 0x7440u + (uint32_t)ch)), 8388608.0f);
}
// SF16 channel: u16 lane `sel` (0x7410 low, 0x7432 high) of a word as the exact float n / 4^k, using
// the magic 2^(23-2k) whose bit pattern is ex = (75-k) << 24: bits(ex | n) = 2^(23-2k) + n 4^-k.
__device__ __forceinline__ float u16f(uint32_t word, uint32_t sel, uint32_t ex)
{
    return __fsub_rn(__uint_as_float(__byte_perm(word, ex, sel)), __uint_as_float(ex));
}
// SF10 channel (level 1: v = n / 4, n < 2^10 in 10-bit fields at bits 0, 10, 20) as the exact float n / 4:
// a field placed in the mantissa of 2^e with unit 2^-2 (e = 21 for bits 0-9, e = 11 for bits 10-19), then
// 2^e subtracted.
__device__ __forceinline__ float f10_0(uint32_t w) { return __fsub_rn(__uint_as_float((w & 0x3FFu) | 0x4A000000u), 2097152.0f); }
__device__ __forceinline__ float f10_1(uint32_t w) { return __fsub_rn(__uint_as_float((w & 0xFFC00u) | 0x45000000u), 2048.0f); }
__device__ __forceinline__ float f10_2(uint32_t w) { return __fsub_rn(__uint_as_float((w >> 20) | 0x4A000000u), 2097152.0f); }
__device__ __forceinline__ uint32_t pack_rgb(float r, float g, float b)  // exact for integer 0..255
{
    return (uint32_t)r | ((uint32_t)g << 8) | ((uint32_t)b << 16);
}
__device__ __forceinline__ uint32_t pack10(float r, float g, float b)  // SF10 / TF10 fields n = 4v (level 1, exact)
{
    return (uint32_t)(r * 4.0f) | ((uint32_t)(g * 4.0f) << 10) | ((uint32_t)(b * 4.0f) << 20);
}
// SF10 / TF10 channel as the exact value v = n / 4 biased by 2^21 (channels 0 and 2) or 2^11 (channel 1): the
// field is placed in the mantissa of the bias (one LOP3 / funnel shift, no add).  Two biased values of one
// channel differ by exactly t - s (same binade: Sterbenz), so the guide delta of D20 costs one FSUB.
__device__ __forceinline__ float b10_0(uint32_t w) { return __uint_as_float((w & 0x3FFu) | 0x4A000000u); }
__device__ __forceinline__ float b10_1(uint32_t w) { return __uint_as_float((w & 0xFFC00u) | 0x45000000u); }
__device__ __forceinline__ float b10_2(uint32_t w) { return __uint_as_float(__funnelshift_r(w, 0x4A000u, 20)); }

// ------------------------------------------------------------------------------------ pyramid (D6)
__global__ void k_u8_to_pyr0(const uint8_t* __restrict__ frames, float4* __restrict__ pyr, int npx,
                             long long pyr_stride)
{
    const int b = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npx; i += gridDim.x * blockDim.x) {
        const uint8_t* px = frames + ((long long)b * npx + i) * 3;
        pyr[(long long)b * pyr_stride + i] = make_float4((float)px[0], (float)px[1], (float)px[2], 0.0f);
    }
}

__global__ void k_box(float4* __restrict__ pyr, long long pyr_stride, Lvl prev, Lvl cur)
{
    const int b = blockIdx.y;
    const int n = cur.h * cur.w;
    float4* base = pyr + (long long)b * pyr_stride;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = i / cur.w, c = i - r * cur.w;
        const float4* p0 = base + prev.off + (long long)(2 * r) * prev.w + 2 * c;
        const float4 a = p0[0], bb = p0[1], d = p0[prev.w], e = p0[prev.w + 1];
        float4 o;  // ((a+b)+(d+e))*0.25, exact in 8-bit units (dyadic)
        o.x = __fmul_rn(__fadd_rn(__fadd_rn(a.x, bb.x), __fadd_rn(d.x, e.x)), 0.25f);
        o.y = __fmul_rn(__fadd_rn(__fadd_rn(a.y, bb.y), __fadd_rn(d.y, e.y)), 0.25f);
        o.z = __fmul_rn(__fadd_rn(__fadd_rn(a.z, bb.z), __fadd_rn(d.z, e.z)), 0.25f);
        o.w = 0.0f;
        base[cur.off + i] = o;
    }
}

// ------------------------------------------------------------------------------------ operand packing
// Source operands: the whole padded block is written (zeros in the border).
__global__ void k_pack_src(const PackSrc* __restrict__ jobs, int fmt, PLvl L)
{
    const PackSrc J = jobs[blockIdx.y];
    const int n = L.rows * L.pitch;
    const int copies = fmt == SF8 ? kSF8Copies : (fmt == SF10 ? 2 : 1);
    for (int ii = blockIdx.x * blockDim.x + threadIdx.x; ii < n * copies; ii += gridDim.x * blockDim.x) {
        const int cpy = ii / n, i = ii - cpy * n;  // copy cpy holds texel (pr, pc + cpy) at (pr, pc)
        const int pr = i / L.pitch, pc = i - pr * L.pitch;
        const int r = pr - B, c = pc + cpy - B;
        const bool in = (unsigned)r < (unsigned)L.h && (unsigned)c < (unsigned)L.w && pc + cpy < L.pitch;
        if (fmt == SF8) {
            uint2 v = make_uint2(0u, 0u);
            if (in) {
                const uint8_t* g = J.g8 + 3LL * (r * L.w + c);
                v.x = g[0] | (g[1] << 8) | (g[2] << 16);
                v.y = 1u << 24;  // byte 3: the in-image count the slot remaps accumulate (0 in the border)
                if (J.s8) {
                    const uint8_t* s = J.s8 + 3LL * (r * L.w + c);
                    v.y |= s[0] | (s[1] << 8) | (s[2] << 16);
                }
            }
            reinterpret_cast<uint2*>(J.out)[(size_t)cpy * n + i] = v;
        } else if (fmt == SF8F) {
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (in) {
                const float4 g = J.gp[r * L.w + c];
                const float4 sv = J.sp ? J.sp[r * L.w + c] : make_float4(0.f, 0.f, 0.f, 0.f);
                v = make_uint4(pack_rgb(g.x, g.y, g.z), __float_as_uint(sv.x), __float_as_uint(sv.y),
                               __float_as_uint(sv.z));
            }
            reinterpret_cast<uint4*>(J.out)[i] = v;
        } else if (fmt == SF10) {
            // level 1 of a u8 pyramid: v = n / 4 with n <= 1020; 10-bit fields {r, g, b} of G and of S
            uint2 v = make_uint2(0u, 0u);
            if (in) {
                const float4 g = J.gp[r * L.w + c];
                const float4 sv = J.sp ? J.sp[r * L.w + c] : make_float4(0.f, 0.f, 0.f, 0.f);
                v.x = (uint32_t)(g.x * 4.0f) | ((uint32_t)(g.y * 4.0f) << 10) | ((uint32_t)(g.z * 4.0f) << 20);
                v.y = (uint32_t)(sv.x * 4.0f) | ((uint32_t)(sv.y * 4.0f) << 10) | ((uint32_t)(sv.z * 4.0f) << 20);
            }
            reinterpret_cast<uint2*>(J.out)[(size_t)cpy * n + i] = v;
        } else if (fmt == SF16) {
            // level k of a u8 pyramid: v = n / 4^k with n < 2^16 (k <= 4); store n
            const float sc = (float)(1 << (2 * L.k));
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (in) {
                const float4 g = J.gp[r * L.w + c];
                const float4 s = J.sp ? J.sp[r * L.w + c] : make_float4(0.f, 0.f, 0.f, 0.f);
                v.x = (uint32_t)(g.x * sc) | ((uint32_t)(g.y * sc) << 16);
                v.y = (uint32_t)(g.z * sc);
                v.z = (uint32_t)(s.x * sc) | ((uint32_t)(s.y * sc) << 16);
                v.w = (uint32_t)(s.z * sc);
            }
            reinterpret_cast<uint4*>(J.out)[i] = v;
        } else {
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
            if (in) {
                const float4 g = J.gp[r * L.w + c];
                const float4 s = J.sp ? J.sp[r * L.w + c] : make_float4(0.f, 0.f, 0.f, 0.f);
                a = make_float4(g.x, g.y, g.z, s.x);
                b = make_float4(s.y, s.z, 0.0f, 0.0f);
            }
            reinterpret_cast<float4*>(J.out)[2 * i] = a;
            reinterpret_cast<float4*>(J.out)[2 * i + 1] = b;
        }
    }
}

// Patch sums (SumJob, kernels.h) of SF8 (u8 fields), SF10 (10-bit fields n = 4v) or SF16 (16-bit n = v 4^k)
// source blocks: integer sums over the (2p+1)^2 patch (zero border = zero padding, D9), exact; the caller checks
// that every sum fits its 21-bit field.  The patch rows are re-read per output texel (L1 hits).
template <int P>
__global__ void k_patch_sums(const SumJob* __restrict__ jobs, int fmt, PLvl L, int tail_r0)
{
    constexpr int D = 2 * P + 1;
    const SumJob J = jobs[blockIdx.y];
    const int n = L.h * L.w;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = i / L.w, c = i - r * L.w;
        if (fmt == SF8F) {  // u8 guide (exact integer sums) + f32 style (FP32 sums with an absolute margin)
            uint32_t g0 = 0, g1 = 0, g2 = 0;
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, b0 = 0.f, b1 = 0.f, b2 = 0.f;
            for (int dr = 0; dr < D; ++dr) {
                const size_t row0 = (size_t)(r + dr - P + B) * L.pitch + (c - P + B);
#pragma unroll
                for (int dc = 0; dc < D; ++dc) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4*>(J.blk) + row0 + dc);
                    g0 += v.x & 0xFFu; g1 += (v.x >> 8) & 0xFFu; g2 += (v.x >> 16) & 0xFFu;
                    const float t0 = __uint_as_float(v.y), t1 = __uint_as_float(v.z), t2 = __uint_as_float(v.w);
                    s0 = __fadd_rn(s0, t0); s1 = __fadd_rn(s1, t1); s2 = __fadd_rn(s2, t2);
                    b0 = __fadd_ru(b0, fabsf(t0)); b1 = __fadd_ru(b1, fabsf(t1)); b2 = __fadd_ru(b2, fabsf(t2));
                }
            }
            const float m = __fmul_ru(fmaxf(b0, fmaxf(b1, b2)), (float)(2 * D * D) * 0x1p-24f);
            J.sums[2 * i] = make_uint4(g0, g1, g2, __float_as_uint(s0));
            J.sums[2 * i + 1] = make_uint4(__float_as_uint(s1), __float_as_uint(s2), __float_as_uint(m), 0u);
            continue;
        }
        uint32_t g0 = 0, g1 = 0, g2 = 0, s0 = 0, s1 = 0, s2 = 0;
        uint32_t tl[3] = {0u, 0u, 0u};  // SF8 tail rows: {G.r | G.g << 16, G.b | S.r << 16, S.g | S.b << 16}
        for (int dr = 0; dr < D; ++dr) {
            if (dr == tail_r0) { tl[0] = g0 | (g1 << 16); tl[1] = g2 | (s0 << 16); tl[2] = s1 | (s2 << 16); }
            const size_t row0 = (size_t)(r + dr - P + B) * L.pitch + (c - P + B);
#pragma unroll
            for (int dc = 0; dc < D; ++dc) {
                if (fmt == SF16) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4*>(J.blk) + row0 + dc);
                    g0 += v.x & 0xFFFFu; g1 += v.x >> 16; g2 += v.y & 0xFFFFu;
                    s0 += v.z & 0xFFFFu; s1 += v.z >> 16; s2 += v.w & 0xFFFFu;
                } else {
                    const uint2 v = __ldg(reinterpret_cast<const uint2*>(J.blk) + row0 + dc);
                    if (fmt == SF8) {
                        g0 += v.x & 0xFFu; g1 += (v.x >> 8) & 0xFFu; g2 += (v.x >> 16) & 0xFFu;
                        s0 += v.y & 0xFFu; s1 += (v.y >> 8) & 0xFFu; s2 += (v.y >> 16) & 0xFFu;
                    } else {
                        g0 += v.x & 0x3FFu; g1 += (v.x >> 10) & 0x3FFu; g2 += v.x >> 20;
                        s0 += v.y & 0x3FFu; s1 += (v.y >> 10) & 0x3FFu; s2 += v.y >> 20;
                    }
                }
            }
        }
        const unsigned long long lo = g0 | ((unsigned long long)g1 << 21) | ((unsigned long long)g2 << 42);
        const unsigned long long hi = s0 | ((unsigned long long)s1 << 21) | ((unsigned long long)s2 << 42);
        J.sums[i] = make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi, (uint32_t)(hi >> 32));
        if (J.tail)  // SF8 (sums < 2^16): the tail rows = the whole patch minus the rows before tail_r0
            J.tail[i] = make_uint4((g0 | (g1 << 16)) - tl[0], (g2 | (s0 << 16)) - tl[1], (s1 | (s2 << 16)) - tl[2], 0u);
    }
}

// ---- patch-sum bound ("exact work elimination") ------------------------------------------
// Per channel, Cauchy-Schwarz gives sum_taps (t - s)^2 >= (sum t - sum s)^2 / D^2, so
//   LB = alpha * sum_c (dG_c)^2 / D^2 + sum_c (dS_c)^2 / D^2  <=  L*,
// the exact loss of the candidate over the stored operand values.  The FP32 loss the kernels compute
// (non-negative terms, every chain <= 23 roundings) is >= L* (1 - 23 u), u = 2^-24.  Guide sums are exact (integer
// multiples of 4^-k below 2^21 units); the target aux sums carry an absolute error <= 8 u sum|t| (two-pass sums),
// removed, with the rounding of the delta, from |dS_c| before squaring (margin m = 2 D^2 u sum|t|, an upper
// bound); LB is evaluated with round-down operations.  So rd(LB (1 - 2^-16)) >= E implies the candidate's
// FP32 loss is >= E: it cannot win the strict select (D16) and rejecting it changes nothing.
struct TSums {
    float g0, g1, g2;  // target guide patch sums (exact, level units)
    float a0, a1, a2;  // target aux patch sums (FP32)
    float m;           // absolute margin of the aux sums
};
// Random-search draws (D13, D21): one Philox block per two steps -- counter step field s >> 1; step s takes words
// (x, y) when even, (z, w) when odd -- so a pixel's K steps cost ceil(K/2) blocks.  rs_block is called at every
// even step (and at s when it starts a loop), rs_offset turns step s's words into a uniform offset in [-R, R]^2,
// R = max(r0 >> s, 1).
__device__ __forceinline__ uint4 rs_block(const FieldArgs& a, const DTask& T, int i, int s)
{
    return philox4x32_10(
        make_uint4((uint32_t)i, (1u << 28) | (a.level << 22) | (a.iter << 12) | (uint32_t)(s >> 1), T.c2, T.c3),
        a.rng.k0, a.rng.k1);
}
__device__ __forceinline__ int2 rs_offset(const FieldArgs& a, uint4 u, int s)
{
    const int R = max(a.rs_r0 >> s, 1);
    const uint32_t span = 2u * (uint32_t)R + 1u;
    const uint32_t ux = (s & 1) ? u.z : u.x, uy = (s & 1) ? u.w : u.y;
    return make_int2((int)__umulhi(ux, span) - R, (int)__umulhi(uy, span) - R);
}

// margin of a two-pass FP32 sum of D^2 aux values whose absolute values sum to <= absum
template <int D>
__device__ __forceinline__ float csb_margin(float absum) { return __fmul_ru(absum, (float)(2 * D * D) * 0x1p-24f); }
// q: the candidate's source patch sums (k_patch_sums, 21-bit fields in units of `scale` = 4^-k)
template <int D, bool TWO>
__device__ __forceinline__ bool csb_reject(uint4 q, const TSums& t, float scale, float alpha, float e)
{
    constexpr unsigned long long M21 = (1ull << 21) - 1;
    const unsigned long long lo = ((unsigned long long)q.y << 32) | q.x;
    const float d0 = __fsub_rn(t.g0, (float)(uint32_t)(lo & M21) * scale);  // exact: multiples of scale < 2^22
    const float d1 = __fsub_rn(t.g1, (float)(uint32_t)((lo >> 21) & M21) * scale);
    const float d2 = __fsub_rn(t.g2, (float)(uint32_t)(lo >> 42) * scale);
    const float inv = __frcp_rd((float)(D * D));
    float lb = __fmul_rd(__fmaf_rd(d2, d2, __fmaf_rd(d1, d1, __fmul_rd(d0, d0))), inv);
    if (TWO) {
        const unsigned long long hi = ((unsigned long long)q.w << 32) | q.z;
        constexpr float kS = 1.0f - 0x1p-22f;
        const float l0 = fmaxf(__fsub_rd(__fmul_rd(fabsf(__fsub_rn(t.a0, (float)(uint32_t)(hi & M21) * scale)), kS), t.m), 0.0f);
        const float l1 = fmaxf(__fsub_rd(__fmul_rd(fabsf(__fsub_rn(t.a1, (float)(uint32_t)((hi >> 21) & M21) * scale)), kS), t.m), 0.0f);
        const float l2 = fmaxf(__fsub_rd(__fmul_rd(fabsf(__fsub_rn(t.a2, (float)(uint32_t)(hi >> 42) * scale)), kS), t.m), 0.0f);
        lb = __fmaf_rd(alpha, lb, __fmul_rd(__fmaf_rd(l2, l2, __fmaf_rd(l1, l1, __fmul_rd(l0, l0))), inv));
    }
    return __fmul_rd(lb, 1.0f - 0x1p-16f) >= e;
}
// The same bound for SF8F sources (float styles, e.g. blending-table cells): two 16-byte texels {G sums (exact),
// S.r sum} {S.g, S.b sums, their absolute margin ms}; the style delta loses both sums' margins.
template <int D, bool TWO>
__device__ __forceinline__ bool csb_reject_f(uint4 qa, uint4 qb, const TSums& t, float alpha, float e)
{
    const float d0 = __fsub_rn(t.g0, (float)qa.x), d1 = __fsub_rn(t.g1, (float)qa.y), d2 = __fsub_rn(t.g2, (float)qa.z);
    const float inv = __frcp_rd((float)(D * D));
    float lb = __fmul_rd(__fmaf_rd(d2, d2, __fmaf_rd(d1, d1, __fmul_rd(d0, d0))), inv);
    if (TWO) {
        constexpr float kS = 1.0f - 0x1p-22f;
        const float m = __fadd_ru(t.m, __uint_as_float(qb.z));
        const float l0 = fmaxf(__fsub_rd(__fmul_rd(fabsf(__fsub_rn(t.a0, __uint_as_float(qa.w))), kS), m), 0.0f);
        const float l1 = fmaxf(__fsub_rd(__fmul_rd(fabsf(__fsub_rn(t.a1, __uint_as_float(qb.x))), kS), m), 0.0f);
        const float l2 = fmaxf(__fsub_rd(__fmul_rd(fabsf(__fsub_rn(t.a2, __uint_as_float(qb.y))), kS), m), 0.0f);
        lb = __fmaf_rd(alpha, lb, __fmul_rd(__fmaf_rd(l2, l2, __fmaf_rd(l1, l1, __fmul_rd(l0, l0))), inv));
    }
    return __fmul_rd(lb, 1.0f - 0x1p-16f) >= e;
}
// Partial + remainder bound of the fused level-0 kernel: after the partial-distance check at row S1
// fails, the FP32 partial P (rows < S1) plus Cauchy-Schwarz on the NT tail taps' sums (SumJob::tail q, target tail
// sums tg01 = G.r | G.g << 16, tg2 = G.b (exact), a0..a2 (FP32, absolute error <= m: the whole patch's csb_margin
// bounds the tail's few roundings)) is a lower bound of the candidate's FP32 loss up to 46 u: P over-states the
// exact partial by <= 23 u, the full loss under-states the exact loss by <= 23 u (see the patch-sum bound above).
// So rd((P + LB) (1 - 2^-16)) >= E implies the FP32 loss is >= E and the candidate cannot win (D16).
template <int NT>
__device__ __forceinline__ bool tail_reject(uint4 q, uint32_t tg01, uint32_t tg2, float a0, float a1, float a2,
                                            float m, float alpha, float part, float e)
{
    const uint32_t d01 = __vabsdiffu2(tg01, q.x), d2 = __vabsdiffu2(tg2, q.y) & 0xFFFFu;
    const uint32_t d0 = d01 & 0xFFFFu, d1 = d01 >> 16;
    const uint32_t gg = d0 * d0 + d1 * d1 + d2 * d2;  // exact: < 3 * 2^32 / 2^8 for tail sums < 2^12
    constexpr float kS = 1.0f - 0x1p-22f;
    const float l0 = fmaxf(__fsub_rd(__fmul_rd(fabsf(__fsub_rn(a0, (float)(q.y >> 16))), kS), m), 0.0f);
    const float l1 = fmaxf(__fsub_rd(__fmul_rd(fabsf(__fsub_rn(a1, (float)(q.z & 0xFFFFu))), kS), m), 0.0f);
    const float l2 = fmaxf(__fsub_rd(__fmul_rd(fabsf(__fsub_rn(a2, (float)(q.z >> 16))), kS), m), 0.0f);
    const float ls = __fmaf_rd(l2, l2, __fmaf_rd(l1, l1, __fmul_rd(l0, l0)));
    const float lb = __fmul_rd(__fmaf_rd(alpha, __uint2float_rd(gg), ls), __frcp_rd((float)NT));
    return __fmul_rd(__fadd_rd(part, lb), 1.0f - 0x1p-16f) >= e;
}
// Target patch sums of the bound for lane (lx, ly) of a warp-per-tile-row layout (tile column lx + j, row ly + dr):
// column sums over the D rows (tile columns 32.. by lanes 0..2P-1), then the D columns by shuffles.  All 32 lanes
// must call it converged.  fetch(yy, xx, v) returns the tile texel's guide (v[0..2], level units) and aux
// (v[3..5]); guide sums are exact (multiples of 4^-k below 2^21 units), aux sums carry the margin of csb_margin.
template <int P, class Fetch>
__device__ __forceinline__ TSums tile_patch_sums(int lx, int ly, Fetch&& fetch)
{
    constexpr int D = 2 * P + 1;
    float cs[2][7];  // [main, extra] {g0, g1, g2, a0, a1, a2, max_c sum|a_c|}
#pragma unroll
    for (int x = 0; x < 2; ++x) {
#pragma unroll
        for (int q = 0; q < 7; ++q) cs[x][q] = 0.0f;
        if (x == 1 && lx >= 2 * P) break;
        float b0 = 0.f, b1 = 0.f, b2 = 0.f;
#pragma unroll
        for (int dr = 0; dr < D; ++dr) {
            float v[6];
            fetch(ly + dr, lx + 32 * x, v);
#pragma unroll
            for (int q = 0; q < 6; ++q) cs[x][q] = __fadd_rn(cs[x][q], v[q]);
            b0 = __fadd_ru(b0, fabsf(v[3])); b1 = __fadd_ru(b1, fabsf(v[4])); b2 = __fadd_ru(b2, fabsf(v[5]));
        }
        cs[x][6] = fmaxf(b0, fmaxf(b1, b2));
    }
    float acc[7];
#pragma unroll
    for (int q = 0; q < 7; ++q) acc[q] = cs[0][q];
#pragma unroll
    for (int j = 1; j < D; ++j) {
        const bool own = lx + j < 32;
        const int src = (lx + j) & 31;
#pragma unroll
        for (int q = 0; q < 7; ++q) {
            const float pv = __shfl_down_sync(0xffffffffu, cs[0][q], j), qv = __shfl_sync(0xffffffffu, cs[1][q], src);
            acc[q] = q == 6 ? __fadd_ru(acc[q], own ? pv : qv) : __fadd_rn(acc[q], own ? pv : qv);
        }
    }
    return TSums{acc[0], acc[1], acc[2], acc[3], acc[4], acc[5], csb_margin<D>(acc[6])};
}


__device__ __forceinline__ void store_tgt(char* out, int tfmt, int i, bool in, float4 g, float ar, float ag, float ab)
{
    if (tfmt == TF16 || tfmt == TF10) {
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (in) v = make_uint4(tfmt == TF16 ? pack_rgb(g.x, g.y, g.z) : pack10(g.x, g.y, g.z), __float_as_uint(ar),
                               __float_as_uint(ag), __float_as_uint(ab));
        reinterpret_cast<uint4*>(out)[i] = v;
    } else {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
        if (in) { a = make_float4(g.x, g.y, g.z, ar); b = make_float4(ag, ab, 0.0f, 0.0f); }
        reinterpret_cast<float4*>(out)[2 * i] = a;
        reinterpret_cast<float4*>(out)[2 * i + 1] = b;
    }
}

// BASE loss: the target operand is the target guide alone.
__global__ void k_pack_tgt_guide(const DTask* __restrict__ tasks, Lvl L, PLvl P, int tfmt)
{
    const DTask T = tasks[blockIdx.y];
    const int n = P.rows * P.pitch;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = i / P.pitch - B, c = i % P.pitch - B;
        const bool in = (unsigned)r < (unsigned)P.h && (unsigned)c < (unsigned)P.w;
        const float4 g = in ? T.tg[L.off + r * P.w + c] : make_float4(0.f, 0.f, 0.f, 0.f);
        store_tgt(T.tgt, tfmt, i, in, g, 0.0f, 0.0f, 0.0f);
    }
}

// ------------------------------------------------------------------------------------ NNF init / upsample
__global__ void k_init(const DTask* __restrict__ tasks, int2* __restrict__ F, long long fstride, Lvl L,
                       int identity, Rng rng, uint32_t level)
{
    const int t = blockIdx.y;
    const int n = L.h * L.w;
    const DTask T = tasks[t];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = i / L.w, c = i - r * L.w;
        int2 f;
        if (identity) {
            f = make_int2(r, c);
        } else {  // "Randomly initialize F": (mulhi(u0, h), mulhi(u1, w))
            const uint4 u = philox4x32_10(make_uint4((uint32_t)i, level << 22, T.c2, T.c3), rng.k0, rng.k1);
            f = make_int2((int)__umulhi(u.x, (uint32_t)L.h), (int)__umulhi(u.y, (uint32_t)L.w));
        }
        F[t * fstride + i] = f;
    }
}

// "Upsample F" (D7): F_f(r,c) = clamp(2 F_c(rc,cc) + (r - 2rc, c - 2cc)), rc = min(r>>1, h_c-1).
__global__ void k_upsample(const int2* __restrict__ Fc, int2* __restrict__ Ff, long long fstride, Lvl Lc, Lvl Lf)
{
    const int t = blockIdx.y;
    const int n = Lf.h * Lf.w;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = i / Lf.w, c = i - r * Lf.w;
        const int rc = min(r >> 1, Lc.h - 1), cc = min(c >> 1, Lc.w - 1);
        const int2 f = Fc[t * fstride + rc * Lc.w + cc];
        Ff[t * fstride + i] = make_int2(clampi(2 * f.x + (r - 2 * rc), 0, Lf.h - 1),
                                        clampi(2 * f.y + (c - 2 * cc), 0, Lf.w - 1));
    }
}

// ------------------------------------------------------------------------------------ remap (Alg. 2, D19)
// Sum over valid taps (target neighbour inside AND source texel inside), dr then dc ascending,
// then one IEEE division by the valid count.
template <int P>
__device__ __forceinline__ float3 remap_px(const float4* __restrict__ S, const int2* __restrict__ F, int h, int w,
                                           int r, int c)
{
    float ax = 0.0f, ay = 0.0f, az = 0.0f;
    int n = 0;
#pragma unroll
    for (int dr = -P; dr <= P; ++dr) {
        const int tr = r + dr;
        if ((unsigned)tr >= (unsigned)h) continue;
#pragma unroll
        for (int dc = -P; dc <= P; ++dc) {
            const int tc = c + dc;
            if ((unsigned)tc >= (unsigned)w) continue;
            const int2 f = __ldg(&F[tr * w + tc]);
            const int sr = f.x - dr, sc = f.y - dc;
            if ((unsigned)sr >= (unsigned)h || (unsigned)sc >= (unsigned)w) continue;
            const float4 v = __ldg(&S[sr * w + sc]);
            ax = __fadd_rn(ax, v.x);
            ay = __fadd_rn(ay, v.y);
            az = __fadd_rn(az, v.z);
            ++n;
        }
    }
    const float fn = (float)n;
    return make_float3(__fdiv_rn(ax, fn), __fdiv_rn(ay, fn), __fdiv_rn(az, fn));
}

// Same remap reading the style channels from a packed source slot (SF8: u8 word, SF10: 10-bit fields,
// SF16: two u16 words),
// a quarter / half of the bytes per tap of the float4 pyramid.  Exact integer form: a slot holds every
// style value as n * 4^-k with integer n (k = 0: u8; k = 1..4: SF16, D6), and a sum of at most (2P+1)^2
// such values has sum(n) < 2^24, so the FP32 chain of D19 is exact, order-free and equal to
// (float)sum(n) * 4^-k; the sums are kept in integers (SF8: r|b and g in 16-bit lanes) and the one IEEE
// division by the valid count is unchanged.  Branch-free: the zero border (>= P texels) makes every tap
// address valid (F is in bounds, so F - d lies within P of the image), and invalid taps are masked to 0.
// RU: patch rows unrolled (and their loads hoisted) at once: all for the single-member S^ refresh, one in
// the many-member combine, where hoisting every row's loads spills at the register cap (tbar.L0 44 -> 41 ms).
template <int P, int SFMT, int RU = 2 * P + 1>
__device__ __forceinline__ float3 remap_px_slot(const char* __restrict__ slot, int pitch, const int2* __restrict__ F,
                                                int h, int w, int r, int c, int k)
{
    uint32_t a0 = 0u, a1 = 0u, a2 = 0u;
    int n = 0;
#pragma unroll RU
    for (int dr = -P; dr <= P; ++dr) {
        const int tr = r + dr;
        const bool rin = (unsigned)tr < (unsigned)h;
        const int trc = clampi(tr, 0, h - 1);
#pragma unroll
        for (int dc = -P; dc <= P; ++dc) {
            const int tc = c + dc;
            const int2 f = __ldg(&F[trc * w + clampi(tc, 0, w - 1)]);
            const int sr = f.x - dr, sc = f.y - dc;
            const int idx = (sr + kBorder) * pitch + sc + kBorder;
            FB_ASSERT(sr >= -kBorder && sc >= -kBorder && sr < h + kBorder && sc < w + kBorder);
            if (SFMT == SF8) {  // the source-side validity is the texel's count byte (1 inside, 0 in the border)
                uint32_t sv = __ldg(reinterpret_cast<const uint32_t*>(slot) + 2 * idx + 1);
                sv = rin && (unsigned)tc < (unsigned)w ? sv : 0u;
                a0 += __byte_perm(sv, 0u, 0x4240u);  // r | b << 16
                a1 += __byte_perm(sv, 0u, 0x4341u);  // g | count << 16
                continue;
            }
            const bool v = rin && (unsigned)tc < (unsigned)w && (unsigned)sr < (unsigned)h && (unsigned)sc < (unsigned)w;
            if (SFMT == SF10) {
                uint32_t sv = __ldg(reinterpret_cast<const uint32_t*>(slot) + 2 * idx + 1);
                sv = v ? sv : 0u;
                a0 += sv & 0x3FFu;
                a1 += (sv >> 10) & 0x3FFu;
                a2 += sv >> 20;
            } else {
                uint2 sv = __ldg(reinterpret_cast<const uint2*>(slot) + 2 * idx + 1);
                if (!v) sv = make_uint2(0u, 0u);
                a0 += sv.x & 0xffffu;
                a1 += sv.x >> 16;
                a2 += sv.y;
            }
            n += v ? 1 : 0;
        }
    }
    float x, y, z;
    if (SFMT == SF8) {
        x = (float)(a0 & 0xffffu); y = (float)(a1 & 0xffffu); z = (float)(a0 >> 16);
        n = (int)(a1 >> 16);
    } else {
        const float sc = __int_as_float((127 - 2 * k) << 23);  // 4^-k, exact
        x = __fmul_rn((float)a0, sc); y = __fmul_rn((float)a1, sc); z = __fmul_rn((float)a2, sc);
    }
    const float fn = (float)n;
    return make_float3(__fdiv_rn(x, fn), __fdiv_rn(y, fn), __fdiv_rn(z, fn));
}

// S^ refresh (GUIDE_STYLE, D17/D18): packed target = {G_tgt, remap(S_src, F)} over the padded grid.
// SFMT = SF8 / SF16 reads the source style from the task's packed slot (exact integer form above); -1
// reads the float4 style pyramid (float-style sources such as blending-table cells).
#ifndef AUX_RU1
#define AUX_RU1 1    // p >= 3: remap one patch row at a time (config-5 shard: aux 204 ms -> < 120 ms)
#endif
#ifndef AUX3_MINB
#define AUX3_MINB 1
#endif
#ifndef AUX_MINB
#define AUX_MINB 5  // p = 2: 48 registers (balanced N=48: aux 62.5 -> 60.1 ms; 8 CTAs spill and lose)
#endif
template <int P, int SFMT>
__global__ void __launch_bounds__(256, P == 2 ? AUX_MINB : AUX3_MINB) k_aux_remap(const DTask* __restrict__ tasks, const int2* __restrict__ F, long long fstride, Lvl L,
                            PLvl PL, int tfmt, long long src_off)
{
    const int t = blockIdx.y;
    const DTask T = tasks[t];
    const float4* S = T.ss + L.off;
    const char* slot = T.src + src_off;
    const int2* Ft = F + t * fstride;
    const int n = PL.rows * PL.pitch;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = i / PL.pitch - B, c = i % PL.pitch - B;
        const bool in = (unsigned)r < (unsigned)L.h && (unsigned)c < (unsigned)L.w;
        float3 v = make_float3(0.f, 0.f, 0.f);
        float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
        if (in) {
            if (SFMT == SF8 || SFMT == SF10 || SFMT == SF16)
                v = remap_px_slot<P, SFMT, (P <= 2 || !AUX_RU1) ? 2 * P + 1 : 1>(slot, PL.pitch, Ft, L.h, L.w, r, c, PL.k);
            else v = remap_px<P>(S, Ft, L.h, L.w, r, c);
            g = __ldg(&T.tg[L.off + r * L.w + c]);
        }
        store_tgt(T.tgt, tfmt, i, in, g, v.x, v.y, v.z);
    }
}

// 5 CTAs/SM caps registers at 51: the unrolled 25-tap remap otherwise takes ~100 registers and halves the
// resident warps of this latency-bound gather (tbar.L0 66 -> 42 ms at N=48; 8 CTAs spill and lose again).
#ifndef COMBINE_MINB
#define COMBINE_MINB 5
#endif
template <int P, int FMT>
__global__ void __launch_bounds__(256, P <= 2 ? COMBINE_MINB : 1) k_combine(const DOut* __restrict__ outs, const DMember* __restrict__ mem, const int2* __restrict__ F,
                          long long fstride, int h, int w, PLvl PL)
{
    const DOut o = outs[blockIdx.y];
    const bool padded = FMT >= 2;
    const int n = padded ? PL.rows * PL.pitch : h * w;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int r, c;
        if (padded) { r = i / PL.pitch - B; c = i % PL.pitch - B; }
        else { r = i / w; c = i - r * w; }
        const bool in = (unsigned)r < (unsigned)h && (unsigned)c < (unsigned)w;
        float ax = 0.0f, ay = 0.0f, az = 0.0f;
        if (in) {
            const int j = r * w + c;
            for (int m = 0; m < o.nm; ++m) {
                const DMember mb = mem[o.m0 + m];
                float3 y;
                if (mb.task < 0) {
                    const float4 v = __ldg(&mb.img[j]);
                    y = make_float3(v.x, v.y, v.z);
                } else {
                    if (mb.sfmt == SF8)
                        y = remap_px_slot<P, SF8, 1>(mb.slot, PL.pitch, F + mb.task * fstride, h, w, r, c, 0);
                    else if (mb.sfmt == SF10)
                        y = remap_px_slot<P, SF10, 1>(mb.slot, PL.pitch, F + mb.task * fstride, h, w, r, c, PL.k);
                    else if (mb.sfmt == SF16)
                        y = remap_px_slot<P, SF16, 1>(mb.slot, PL.pitch, F + mb.task * fstride, h, w, r, c, PL.k);
                    else
                        y = remap_px<P>(mb.img, F + mb.task * fstride, h, w, r, c);
                }
                ax = __fmaf_rn(mb.w, y.x, ax);
                ay = __fmaf_rn(mb.w, y.y, ay);
                az = __fmaf_rn(mb.w, y.z, az);
            }
            ax = __fdiv_rn(ax, o.div);
            ay = __fdiv_rn(ay, o.div);
            az = __fdiv_rn(az, o.div);
        }
        if (FMT == 0) {
            static_cast<float4*>(o.out)[i] = make_float4(ax, ay, az, 0.0f);
        } else if (FMT == 1) {
            float* d = static_cast<float*>(o.out) + 3LL * i;
            d[0] = ax; d[1] = ay; d[2] = az;
        } else {
            const float4 g = in ? __ldg(&o.guide[r * w + c]) : make_float4(0.f, 0.f, 0.f, 0.f);
            store_tgt(static_cast<char*>(o.out), FMT == 2 ? TF16 : (FMT == 4 ? TF10 : TF32), i, in, g, ax, ay, az);
        }
    }
}

template <int P>
__global__ void k_remap_f3(const float* __restrict__ src, const int2* __restrict__ F, float* __restrict__ out, int h,
                           int w)
{
    const int b = blockIdx.y;
    const int n = h * w;
    const float* S = src + 3LL * b * n;
    const int2* Fb = F + (long long)b * n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = i / w, c = i - r * w;
        float ax = 0.0f, ay = 0.0f, az = 0.0f;
        int cnt = 0;
#pragma unroll
        for (int dr = -P; dr <= P; ++dr) {
            const int tr = r + dr;
            if ((unsigned)tr >= (unsigned)h) continue;
#pragma unroll
            for (int dc = -P; dc <= P; ++dc) {
                const int tc = c + dc;
                if ((unsigned)tc >= (unsigned)w) continue;
                const int2 f = Fb[tr * w + tc];
                const int sr = f.x - dr, sc = f.y - dc;
                if ((unsigned)sr >= (unsigned)h || (unsigned)sc >= (unsigned)w) continue;
                const float* v = S + 3LL * (sr * w + sc);
                ax = __fadd_rn(ax, v[0]);
                ay = __fadd_rn(ay, v[1]);
                az = __fadd_rn(az, v[2]);
                ++cnt;
            }
        }
        const float fn = (float)cnt;
        float* d = out + 3LL * ((long long)b * n + i);
        d[0] = __fdiv_rn(ax, fn); d[1] = __fdiv_rn(ay, fn); d[2] = __fdiv_rn(az, fn);
    }
}

// ------------------------------------------------------------------------------------ the field kernels
// One element of Alg. 1's updating sequence per launch, Jacobi over pixels:
//   PHASE 0: E <- L(F), then propagation (-1,0); 1: (+1,0); 2: (0,-1);
//   PHASE 3: propagation (0,+1), then the K random-search fields, pointwise in registers.
// Each candidate F' = clamp(.) is kept iff L(F') < E (strict, D16).
//
// Loss (Eq. 1 / Eq. 3 / Eq. 8): D = sum over rows dr of rho_dr, rho_dr = fma chain over dc then
// channel of (target - source)^2 (D20); two-term losses return fma(alpha, D_guide, D_style).

// Partial-distance elimination stages: rows [0,S1) then a bound check, rows [S1,S2) and a second check
// (skipped when S2 >= 2P+1), then the remaining rows.  Tuned on B200 (N=48 accurate proxy): the
// register-target kernel is best with one check after the first row, the smem-target kernel with
// checks after rows 1 and 3 (profiles/r01_pde_tuning.txt).
#define PDE_FAST_S1(P) 1
#define PDE_FAST_S2(P) (2 * (P) + 1)
// Fused fields 1-3: with the patch-sum bound in front, 91-94 % of the candidates it scores pass every partial
// check, so one check after three rows (p = 2) is best: N=48 field123.L0 318 -> 314 ms accurate, 261 -> 259
// balanced, 102 -> 100 fast (checks after rows 1 and 3: the round-1 optimum before the bound; 1 only, 2 only,
// none: 315-318 / 263-267 / 102-104).
#ifndef PDE_I13_S1
#define PDE_I13_S1(P) ((P) == 2 ? 3 : 1)
#endif
#ifndef PDE_I13_S2
#define PDE_I13_S2(P) (2 * (P) + 1)
#endif
#ifndef PDE_GEN_S1
#define PDE_GEN_S1(P) 1
#endif
#ifndef PDE_GEN_S2
#define PDE_GEN_S2(P) 3
#endif
__device__ __forceinline__ float partial_loss(float alpha, float dg, float ds, bool two)
{
    return two ? __fmaf_rn(alpha, dg, ds) : dg;
}

// Eq. 10 (PAIRWISE, D38/D39): the reference side of the second term is the counterpart keyframe's
// style patch centred at the counterpart's NNF (frozen at the iteration start), gathered once per pixel
// from its packed SF8 slot (zero border = zero padding, D9) and held in registers like a target patch.
template <int P>
__device__ __forceinline__ void load_pairwise_patch(const DTask& T, const FieldArgs& a, int i,
                                                    float (&pa)[2 * P + 1][2 * P + 1][3])
{
    const int2 q = __ldg(&T.pF[i]);
    FB_ASSERT((unsigned)q.x < (unsigned)a.L.h && (unsigned)q.y < (unsigned)a.L.w);
    const uint32_t* PS = reinterpret_cast<const uint32_t*>(T.psrc + a.src_off);
#pragma unroll
    for (int dr = 0; dr < 2 * P + 1; ++dr)
#pragma unroll
        for (int dc = 0; dc < 2 * P + 1; ++dc) {
            const uint32_t sv = __ldg(PS + 2 * ((q.x + dr - P + B) * a.L.pitch + (q.y + dc - P + B)) + 1);
            pa[dr][dc][0] = u8f(sv, 0);
            pa[dr][dc][1] = u8f(sv, 1);
            pa[dr][dc][2] = u8f(sv, 2);
        }
}

// ---- fast variant: SF8 source, TF16 target, target patch in registers (P <= 2) -------------------
// Guide term: at level 0 every guide value is an integer 0..255, every partial sum of the FP32 chain
// is an integer below 2^24 (p <= 4), so the chain is exact and equals the integer SSD computed with
// byte-wise |a-b| and dp4a; it is converted once, exactly.  Style term: the FP32 chain of D20 with the
// u8 source channel converted exactly (u8f).
template <int P, bool TWO, int PHASE, bool PW = false, int SFL = 0>
__global__ void __launch_bounds__(TILE_X* FAST_TY, 3) k_field_fast(FieldArgs a)
{
    constexpr int D = 2 * P + 1;
    constexpr int NCH = (D + 2) / 2;  // 16-byte chunks (texel pairs) covering D texels at either parity
    const int t = blockIdx.x / a.tiles_per_task;
    const int tile = blockIdx.x - t * a.tiles_per_task;
    const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
    const int c = tx * TILE_X + (threadIdx.x & (TILE_X - 1));
    const int r = ty * FAST_TY + (threadIdx.x / TILE_X);
    const int h = a.L.h, w = a.L.w, pitch = a.L.pitch;
    if (r >= h || c >= w) return;
    const DTask T = a.tasks[t];
    const uint2* S = reinterpret_cast<const uint2*>(T.src + a.src_off);
    const uint4* Tt = reinterpret_cast<const uint4*>(T.tgt);
    uint32_t tgG[D][D];
    float tgA[D][D][3];
#pragma unroll
    for (int dr = 0; dr < D; ++dr)
#pragma unroll
        for (int dc = 0; dc < D; ++dc) {
            const uint4 v = __ldg(&Tt[(r + dr - P + B) * pitch + (c + dc - P + B)]);
            tgG[dr][dc] = v.x;
            tgA[dr][dc][0] = __uint_as_float(v.y);
            tgA[dr][dc][1] = __uint_as_float(v.z);
            tgA[dr][dc][2] = __uint_as_float(v.w);
        }
    if (PW) load_pairwise_patch<P>(T, a, r * w + c, tgA);
    // One patch row of the loss (D20): exact integer guide SSD, FP32 style chain, row partial added.
    auto row = [&](int sr, int sc, int dr, uint32_t& dg, float& ds) {
        const int idx = (sr + dr - P + B) * pitch + (sc - P + B);
        FB_ASSERT((unsigned)sr < (unsigned)h && (unsigned)sc < (unsigned)w && FB_ROW_OK(idx, a.L, D));
        if (SFL == 1) {  // SF8F float style (blending-table cells): one 16-byte texel per tap
            const uint4* tp = reinterpret_cast<const uint4*>(S) + idx;
            float rs = 0.0f;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const uint4 v = __ldg(tp + j);
                const uint32_t d = __vabsdiffu4(v.x, tgG[dr][j]);
                dg = __dp4a(d, d, dg);
                if (TWO) {
                    float dl = __fsub_rn(tgA[dr][j][0], __uint_as_float(v.y)); rs = __fmaf_rn(dl, dl, rs);
                    dl = __fsub_rn(tgA[dr][j][1], __uint_as_float(v.z)); rs = __fmaf_rn(dl, dl, rs);
                    dl = __fsub_rn(tgA[dr][j][2], __uint_as_float(v.w)); rs = __fmaf_rn(dl, dl, rs);
                }
            }
            if (TWO) ds = __fadd_rn(ds, rs);
            return;
        }
        const int o = kSF8Copies == 2 ? 0 : (idx & 1);  // with two copies the row start is always even
        const uint4* cp = reinterpret_cast<const uint4*>(
            S + (kSF8Copies == 2 ? (size_t)(idx & 1) * (a.L.rows * pitch) + (idx & ~1) : (size_t)(idx - o)));
        uint32_t wd[4 * NCH];
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
            const uint4 v = __ldg(cp + k);
            wd[4 * k] = v.x; wd[4 * k + 1] = v.y; wd[4 * k + 2] = v.z; wd[4 * k + 3] = v.w;
        }
        float rs = 0.0f;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const uint32_t g = o ? wd[2 * j + 2] : wd[2 * j];
            const uint32_t d = __vabsdiffu4(g, tgG[dr][j]);
            dg = __dp4a(d, d, dg);
            if (TWO) {
                const uint32_t s = o ? wd[2 * j + 3] : wd[2 * j + 1];
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    const float dl = __fsub_rn(tgA[dr][j][ch], u8f(s, ch));
                    rs = __fmaf_rn(dl, dl, rs);
                }
            }
        }
        if (TWO) ds = __fadd_rn(ds, rs);
    };
    // Loss with partial-distance elimination: every term is >= 0 and round-to-nearest sums are
    // monotone, so once the partial loss after the first P rows is >= `bound` the full loss is too and
    // the candidate cannot win the strict select (D16); its remaining rows are never loaded.  Results
    // are unchanged: selected candidates are always evaluated in full, in the D20 order.
    auto loss = [&](int sr, int sc, float bound) -> float {
        uint32_t dg = 0u;
        float ds = 0.0f;
        constexpr int S1 = PDE_FAST_S1(P), S2 = PDE_FAST_S2(P);
#pragma unroll
        for (int dr = 0; dr < S1; ++dr) row(sr, sc, dr, dg, ds);
        if (partial_loss(a.alpha, __uint2float_rn(dg), ds, TWO) >= bound) return __int_as_float(0x7f800000);
        if (S2 < D) {
#pragma unroll
            for (int dr = S1; dr < S2; ++dr) row(sr, sc, dr, dg, ds);
            if (partial_loss(a.alpha, __uint2float_rn(dg), ds, TWO) >= bound) return __int_as_float(0x7f800000);
        }
#pragma unroll
        for (int dr = (S2 < D ? S2 : S1); dr < D; ++dr) row(sr, sc, dr, dg, ds);
        const float fg = __uint2float_rn(dg);
        return TWO ? __fmaf_rn(a.alpha, fg, ds) : fg;
    };
    const int2* Fi = a.Fin + t * a.fstride;
    const int i = r * w + c;
    int2 f = Fi[i];
    float e = PHASE == 0 && a.einit ? loss(f.x, f.y, __int_as_float(0x7f800000)) : a.E[t * a.fstride + i];
    {
        const int dx = (PHASE == 0 ? -1 : (PHASE == 1 ? 1 : 0)) * a.step;  // jump-flood step (D41)
        const int dy = (PHASE == 2 ? -1 : (PHASE == 3 ? 1 : 0)) * a.step;
        const int nr = clampi(r + dx, 0, h - 1), nc = clampi(c + dy, 0, w - 1);  // D11
        const int2 fn = Fi[nr * w + nc];
        const int sr = clampi(fn.x - dx, 0, h - 1), sc = clampi(fn.y - dy, 0, w - 1);  // D10
        if (sr != f.x || sc != f.y) {  // an incumbent-equal candidate cannot win (see select)
            const float e2 = loss(sr, sc, e);
            if (e2 < e) { f = make_int2(sr, sc); e = e2; }
        }
    }
    if (PHASE == 3 && a.do_rs) {
#pragma unroll
        for (int z = 0; z < 2; ++z)  // tracking fields T_{i-1}, T_{i+1} (D42)
            if (T.trk[z]) {
                const int2 g = __ldg(&T.trk[z][i]);
                if (g.x != f.x || g.y != f.y) {
                    const float e2 = loss(g.x, g.y, e);
                    if (e2 < e) { f = g; e = e2; }
                }
            }
        uint4 ru = make_uint4(0u, 0u, 0u, 0u);
        for (int s = 0; s < a.rs_k; ++s) {
            if (!(s & 1)) ru = rs_block(a, T, i, s);
            const int2 o = rs_offset(a, ru, s);
            const int sr = clampi(f.x + o.x, 0, h - 1), sc = clampi(f.y + o.y, 0, w - 1);
            if (sr != f.x || sc != f.y) {
                const float e2 = loss(sr, sc, e);
                if (e2 < e) { f = make_int2(sr, sc); e = e2; }
            }
        }
    }
    FB_ASSERT((unsigned)f.x < (unsigned)h && (unsigned)f.y < (unsigned)w);
    a.Fout[t * a.fstride + i] = f;
    a.E[t * a.fstride + i] = e;
}

// ---- fused iteration (fast operands): the whole updating sequence of one iteration in one launch ----
// Same arithmetic as k_field_fast, with the four propagation fields chained inside the CTA: a tile is
// IT_TX interior columns x IT_TY rows.  Each warp is one image row; lanes 0 and 31 are halo columns
// and warp IT_TY is the halo row below.  Field 0 (-1,0) reads F_in from global; its result goes to
// shared memory for field 1 (+1,0), which reads the row below; field 2 (0,-1) takes the left neighbour's
// field-1 result by shuffle and field 3 (0,+1) the right neighbour's field-2 result.  Halo pixels
// recompute exactly the fields their interior neighbours read, so every interior pixel sees the same
// Jacobi inputs as in the four-launch form and the results are identical.
static constexpr int IT_TX = 30, IT_TY = 4;
#ifndef IT_MINB
#define IT_MINB 2
#endif

template <int P, bool TWO>
__global__ void __launch_bounds__(32 * (IT_TY + 1), IT_MINB) k_iter_fast(FieldArgs a)
{
    constexpr bool PW = false;
    constexpr int SFL = 0;
    constexpr int D = 2 * P + 1;
    constexpr int NCH = (D + 2) / 2;
    __shared__ int2 sF0[IT_TY + 1][32];
    const int t = blockIdx.x / a.tiles_per_task;
    const int tile = blockIdx.x - t * a.tiles_per_task;
    const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
    const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
    const int c = tx * IT_TX - 1 + lane, r = ty * IT_TY + wy;
    const int h = a.L.h, w = a.L.w, pitch = a.L.pitch;
    const bool valid = (unsigned)r < (unsigned)h && (unsigned)c < (unsigned)w;
    const DTask T = a.tasks[t];
    const uint2* S = reinterpret_cast<const uint2*>(T.src + a.src_off);
    const uint4* Tt = reinterpret_cast<const uint4*>(T.tgt);
    uint32_t tgG[D][D];
    float tgA[D][D][3];
    if (valid) {
#pragma unroll
        for (int dr = 0; dr < D; ++dr)
#pragma unroll
            for (int dc = 0; dc < D; ++dc) {
                const uint4 v = __ldg(&Tt[(r + dr - P + B) * pitch + (c + dc - P + B)]);
                tgG[dr][dc] = v.x;
                tgA[dr][dc][0] = __uint_as_float(v.y);
                tgA[dr][dc][1] = __uint_as_float(v.z);
                tgA[dr][dc][2] = __uint_as_float(v.w);
            }
        if (PW) load_pairwise_patch<P>(T, a, r * w + c, tgA);
    }
    // One patch row of the loss (D20): exact integer guide SSD, FP32 style chain, row partial added.
    auto row = [&](int sr, int sc, int dr, uint32_t& dg, float& ds) {
        const int idx = (sr + dr - P + B) * pitch + (sc - P + B);
        FB_ASSERT((unsigned)sr < (unsigned)h && (unsigned)sc < (unsigned)w && FB_ROW_OK(idx, a.L, D));
        if (SFL == 1) {  // SF8F float style (blending-table cells): one 16-byte texel per tap
            const uint4* tp = reinterpret_cast<const uint4*>(S) + idx;
            float rs = 0.0f;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const uint4 v = __ldg(tp + j);
                const uint32_t d = __vabsdiffu4(v.x, tgG[dr][j]);
                dg = __dp4a(d, d, dg);
                if (TWO) {
                    float dl = __fsub_rn(tgA[dr][j][0], __uint_as_float(v.y)); rs = __fmaf_rn(dl, dl, rs);
                    dl = __fsub_rn(tgA[dr][j][1], __uint_as_float(v.z)); rs = __fmaf_rn(dl, dl, rs);
                    dl = __fsub_rn(tgA[dr][j][2], __uint_as_float(v.w)); rs = __fmaf_rn(dl, dl, rs);
                }
            }
            if (TWO) ds = __fadd_rn(ds, rs);
            return;
        }
        const int o = kSF8Copies == 2 ? 0 : (idx & 1);  // with two copies the row start is always even
        const uint4* cp = reinterpret_cast<const uint4*>(
            S + (kSF8Copies == 2 ? (size_t)(idx & 1) * (a.L.rows * pitch) + (idx & ~1) : (size_t)(idx - o)));
        uint32_t wd[4 * NCH];
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
            const uint4 v = __ldg(cp + k);
            wd[4 * k] = v.x; wd[4 * k + 1] = v.y; wd[4 * k + 2] = v.z; wd[4 * k + 3] = v.w;
        }
        float rs = 0.0f;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const uint32_t g = o ? wd[2 * j + 2] : wd[2 * j];
            const uint32_t d = __vabsdiffu4(g, tgG[dr][j]);
            dg = __dp4a(d, d, dg);
            if (TWO) {
                const uint32_t sv = o ? wd[2 * j + 3] : wd[2 * j + 1];
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    const float dl = __fsub_rn(tgA[dr][j][ch], u8f(sv, ch));
                    rs = __fmaf_rn(dl, dl, rs);
                }
            }
        }
        if (TWO) ds = __fadd_rn(ds, rs);
    };
    // Loss with partial-distance elimination: every term is >= 0 and round-to-nearest sums are
    // monotone, so once the partial loss after the first P rows is >= `bound` the full loss is too and
    // the candidate cannot win the strict select (D16); its remaining rows are never loaded.  Results
    // are unchanged: selected candidates are always evaluated in full, in the D20 order.
    auto loss = [&](int sr, int sc, float bound) -> float {
        uint32_t dg = 0u;
        float ds = 0.0f;
        constexpr int S1 = PDE_FAST_S1(P), S2 = PDE_FAST_S2(P);
#pragma unroll
        for (int dr = 0; dr < S1; ++dr) row(sr, sc, dr, dg, ds);
        if (partial_loss(a.alpha, __uint2float_rn(dg), ds, TWO) >= bound) return __int_as_float(0x7f800000);
        if (S2 < D) {
#pragma unroll
            for (int dr = S1; dr < S2; ++dr) row(sr, sc, dr, dg, ds);
            if (partial_loss(a.alpha, __uint2float_rn(dg), ds, TWO) >= bound) return __int_as_float(0x7f800000);
        }
#pragma unroll
        for (int dr = (S2 < D ? S2 : S1); dr < D; ++dr) row(sr, sc, dr, dg, ds);
        const float fg = __uint2float_rn(dg);
        return TWO ? __fmaf_rn(a.alpha, fg, ds) : fg;
    };
    // A candidate equal to the incumbent has exactly the incumbent's loss (same aux within the
    // iteration), so it cannot win the strict select (D16): skipping it changes nothing.
    auto select = [&](int2& f, float& e, int sr, int sc) {
        if (sr == f.x && sc == f.y) return;
        if (sr != f.x || sc != f.y) {  // an incumbent-equal candidate cannot win (see select)
            const float e2 = loss(sr, sc, e);
            if (e2 < e) { f = make_int2(sr, sc); e = e2; }
        }
    };
    const int2* Fi = a.Fin + t * a.fstride;
    const int i = r * w + c;
    int2 f = make_int2(0, 0);
    float e = 0.0f;
    // E <- L(F) and field 0: d = (-1,0), neighbour (r-1, c) of F_in (clamped, D11)
    if (valid) {
        f = Fi[i];
        e = loss(f.x, f.y, __int_as_float(0x7f800000));
        const int2 fn = r > 0 ? Fi[i - w] : f;
        select(f, e, min(fn.x + 1, h - 1), fn.y);
    }
    sF0[wy][lane] = f;
    __syncthreads();
    if (wy == IT_TY) return;  // the halo row only feeds field 1 of the last tile row
    // field 1: d = (+1,0), neighbour (r+1, c) of the field-0 result
    if (valid) {
        const int2 fn = r + 1 < h ? sF0[wy + 1][lane] : f;
        select(f, e, max(fn.x - 1, 0), fn.y);
    }
    // field 2: d = (0,-1), neighbour (r, c-1) of the field-1 result (lane - 1)
    {
        const int2 fl = make_int2(__shfl_up_sync(0xffffffffu, f.x, 1), __shfl_up_sync(0xffffffffu, f.y, 1));
        if (valid && lane > 0) {
            const int2 fn = c > 0 ? fl : f;
            select(f, e, fn.x, min(fn.y + 1, w - 1));
        }
    }
    // field 3: d = (0,+1), neighbour (r, c+1) of the field-2 result (lane + 1), then random search
    {
        const int2 fr = make_int2(__shfl_down_sync(0xffffffffu, f.x, 1), __shfl_down_sync(0xffffffffu, f.y, 1));
        if (!valid || lane == 0 || lane == 31) return;
        const int2 fn = c + 1 < w ? fr : f;
        select(f, e, fn.x, max(fn.y - 1, 0));
    }
#pragma unroll
    for (int z = 0; z < 2; ++z)  // tracking fields T_{i-1}, T_{i+1} (D42)
        if (T.trk[z]) {
            const int2 g = __ldg(&T.trk[z][i]);
            select(f, e, g.x, g.y);
        }
    uint4 ru = make_uint4(0u, 0u, 0u, 0u);
    for (int s = 0; s < a.rs_k; ++s) {
        if (!(s & 1)) ru = rs_block(a, T, i, s);
        const int2 o = rs_offset(a, ru, s);
        select(f, e, clampi(f.x + o.x, 0, h - 1), clampi(f.y + o.y, 0, w - 1));
    }
    FB_ASSERT((unsigned)f.x < (unsigned)h && (unsigned)f.y < (unsigned)w);
    a.Fout[t * a.fstride + i] = f;
    a.E[t * a.fstride + i] = e;
}

// ---- fields 1-3 + random search in one launch (fast operands) --------------------------------------
// Field 0 (E init and d = (-1,0)) runs as k_field_fast<PHASE 0>; this kernel then chains field 1
// (reads the row below from that launch's output), field 2 (left neighbour's field-1 result by shuffle)
// and field 3 (right neighbour's field-2 result by shuffle) and the random search.  Lanes 0 and 31 of
// each warp are halo columns that recompute the fields their interior neighbours read, so the interior
// pixels see exactly the Jacobi inputs of the per-field launches.  No shared memory, no barrier.
#ifndef FB_I13_TY
#define FB_I13_TY 4
#endif
static constexpr int I13_TY = FB_I13_TY;

// NR < D (hybrid target): only the first NR rows of each lane's target patch live in registers -- row 0 is
// read by every candidate, rows >= 1 only by candidates that survive row 0 -- and the rest is read from a
// shared-memory copy of the CTA's target tile.  Registers drop from 168 to <= 128: 4 CTAs/SM instead of 3.
template <int P, bool TWO, bool PW = false, int SFL = 0, int NR = 2 * P + 1, int SF = 0, bool TL = false>
#ifndef I13_HY_MINB
#define I13_HY_MINB 5  // 96 registers, no spills: 5 CTAs/SM (N=48: 388 -> 357 ms; 6 and 7 spill and lose)
#endif
#ifndef I13_SFL_MINB
#define I13_SFL_MINB 4  // SF8F (16-byte texel) queries spill at 5 CTAs/SM: fast N=48 field123.L0 126 -> 124 ms
#endif
#ifndef I13_HY1_MINB
#define I13_HY1_MINB 6  // one target row in registers
#endif
#ifndef I13_HY0_MINB
#define I13_HY0_MINB 10  // no target row in registers, u8 sources: 48 registers (N=48 accurate 308 -> 302 ms against 8
                         // CTAs at 64, 9: 305, 12: 315; balanced 247 -> 241 ms)
#endif
#ifndef I13_HY0X_MINB
#define I13_HY0X_MINB 8  // the same with SF8F cells (fast mode: 10 CTAs 97.4 vs 96.0 ms), SF10, the tail bound, p = 1
#endif
#ifndef I13_P3_MINB
#define I13_P3_MINB 10  // p = 3 (7-texel rows): config-5 shard field123.L0 6 / 8 / 10 CTAs: 339 / 330 / 324 ms (separate launches 333)
#endif
__global__ void __launch_bounds__(32 * I13_TY, NR < 2 * P + 1 ? (NR == 0 ? (P == 3 ? I13_P3_MINB : (P == 2 && !SFL && !SF && !TL ? I13_HY0_MINB : I13_HY0X_MINB)) : (SFL ? I13_SFL_MINB : (NR == 1 ? I13_HY1_MINB : I13_HY_MINB))) : 3) k_iter13_fast(FieldArgs a)
{
    constexpr int D = 2 * P + 1;
    constexpr bool HY = NR < D;
    static_assert(!(HY && PW), "the pairwise reference patch is per pixel: registers only");
    constexpr int NCH = (D + 2) / 2;
    const int t = blockIdx.x / a.tiles_per_task;
    const int tile = blockIdx.x - t * a.tiles_per_task;
    const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
    const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
    const int c = tx * IT_TX - 1 + lane, r = ty * I13_TY + wy;
    const int h = a.L.h, w = a.L.w, pitch = a.L.pitch;
    const bool valid = (unsigned)r < (unsigned)h && (unsigned)c < (unsigned)w;
    const DTask T = a.tasks[t];
    const uint2* S = reinterpret_cast<const uint2*>(T.src + a.src_off);
    const uint4* Tt = reinterpret_cast<const uint4*>(T.tgt);
    constexpr int NRR = HY ? NR : D;
    uint32_t tgG[NRR > 0 ? NRR : 1][D];
    float tgA[NRR > 0 ? NRR : 1][D][3];
    constexpr int TTY = HY ? I13_TY + 2 * P : 1, TTX = HY ? 32 + 2 * P : 1;
    __shared__ uint4 tT[TTY][TTX];
    if (HY) {  // the CTA's target tile (rows r0-P.., cols c0-P..), zero outside the padded plane
        const int pr0 = ty * I13_TY - P + B, pc0 = tx * IT_TX - 1 - P + B;
#if FB_TILE_TMA
        __shared__ uint64_t tbar;
        stage_tile_tma<TTY, TTX>(tT, Tt, pitch, a.L.rows, pr0, pc0, &tbar);
#else
        for (int k = threadIdx.x; k < TTY * TTX; k += 32 * I13_TY) {
            const int yy = k / TTX, xx = k - yy * TTX;
            const int pr = pr0 + yy, pc = pc0 + xx;
            tT[yy][xx] = (pr < a.L.rows && pc < pitch) ? __ldg(&Tt[pr * pitch + pc]) : make_uint4(0u, 0u, 0u, 0u);
        }
        __syncthreads();
#endif
    }
    constexpr bool CSB = (SFL == 0 || SFL == 1) && !PW && HY;  // patch-sum bound of the random search (csb_reject)
    const bool use_csb = CSB && a.sum_off >= 0;
    if (valid) {
#pragma unroll
        for (int dr = 0; dr < NRR; ++dr)
#pragma unroll
            for (int dc = 0; dc < D; ++dc) {
                const uint4 v = HY ? tT[wy + dr][lane + dc] : __ldg(&Tt[(r + dr - P + B) * pitch + (c + dc - P + B)]);
                tgG[dr][dc] = v.x;
                tgA[dr][dc][0] = __uint_as_float(v.y);
                tgA[dr][dc][1] = __uint_as_float(v.z);
                tgA[dr][dc][2] = __uint_as_float(v.w);
            }
        if constexpr (PW && !HY) load_pairwise_patch<P>(T, a, r * w + c, tgA);
    }
    // target texel (dr, j) of this lane's patch: registers for dr < NRR, else the shared tile
    auto tgt = [&](int dr, int j, uint32_t& g, float& a0, float& a1, float& a2) {
        if (dr < NRR) {
            const int d = dr < NRR ? dr : 0;
            g = tgG[d][j]; a0 = tgA[d][j][0]; a1 = tgA[d][j][1]; a2 = tgA[d][j][2];
        } else {
            const uint4 v = tT[HY ? wy + dr : 0][HY ? lane + j : 0];
            g = v.x; a0 = __uint_as_float(v.y); a1 = __uint_as_float(v.z); a2 = __uint_as_float(v.w);
        }
    };
    // One patch row of the loss (D20): exact integer guide SSD, FP32 style chain, row partial added.
    // SF = 1 (level 1, SF10 source + TF10 target): both terms are the literal FP32 chains of D20, with the
    // guide deltas of the exact biased values (b10_*) and the style converted exactly (f10_*); the guide rows
    // are added in FP32 (dgf), as the level-1 sum can exceed 2^24 sixteenths.
    auto row = [&](int sr, int sc, int dr, uint32_t& dg, float& dgf, float& ds) {
        const int idx = (sr + dr - P + B) * pitch + (sc - P + B);
        FB_ASSERT((unsigned)sr < (unsigned)h && (unsigned)sc < (unsigned)w && FB_ROW_OK(idx, a.L, D));
        if constexpr (SF == 1) {
            const uint4* cp = reinterpret_cast<const uint4*>(S + (size_t)(idx & 1) * (a.L.rows * pitch) + (idx & ~1));
            uint32_t wd[4 * NCH];
#pragma unroll
            for (int k = 0; k < NCH; ++k) {
                const uint4 v = __ldg(cp + k);
                wd[4 * k] = v.x; wd[4 * k + 1] = v.y; wd[4 * k + 2] = v.z; wd[4 * k + 3] = v.w;
            }
            float rg = 0.0f, rs = 0.0f;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const uint32_t gw = wd[2 * j], sw = wd[2 * j + 1];
                uint32_t tg; float ta[3];
                tgt(dr, j, tg, ta[0], ta[1], ta[2]);
                float dl;
                dl = __fsub_rn(b10_0(tg), b10_0(gw)); rg = __fmaf_rn(dl, dl, rg);
                dl = __fsub_rn(b10_1(tg), b10_1(gw)); rg = __fmaf_rn(dl, dl, rg);
                dl = __fsub_rn(b10_2(tg), b10_2(gw)); rg = __fmaf_rn(dl, dl, rg);
                if (TWO) {
                    dl = __fsub_rn(ta[0], f10_0(sw)); rs = __fmaf_rn(dl, dl, rs);
                    dl = __fsub_rn(ta[1], f10_1(sw)); rs = __fmaf_rn(dl, dl, rs);
                    dl = __fsub_rn(ta[2], f10_2(sw)); rs = __fmaf_rn(dl, dl, rs);
                }
            }
            dgf = __fadd_rn(dgf, rg);
            if (TWO) ds = __fadd_rn(ds, rs);
            return;
        }
        if (SFL == 1) {  // SF8F float style (blending-table cells): one 16-byte texel per tap
            const uint4* tp = reinterpret_cast<const uint4*>(S) + idx;
            float rs = 0.0f;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const uint4 v = __ldg(tp + j);
                uint32_t tg; float t0, t1, t2;
                tgt(dr, j, tg, t0, t1, t2);
                const uint32_t d = __vabsdiffu4(v.x, tg);
                dg = __dp4a(d, d, dg);
                if (TWO) {
                    float dl = __fsub_rn(t0, __uint_as_float(v.y)); rs = __fmaf_rn(dl, dl, rs);
                    dl = __fsub_rn(t1, __uint_as_float(v.z)); rs = __fmaf_rn(dl, dl, rs);
                    dl = __fsub_rn(t2, __uint_as_float(v.w)); rs = __fmaf_rn(dl, dl, rs);
                }
            }
            if (TWO) ds = __fadd_rn(ds, rs);
            return;
        }
        const int o = kSF8Copies == 2 ? 0 : (idx & 1);  // with two copies the row start is always even
        const uint4* cp = reinterpret_cast<const uint4*>(
            S + (kSF8Copies == 2 ? (size_t)(idx & 1) * (a.L.rows * pitch) + (idx & ~1) : (size_t)(idx - o)));
        uint32_t wd[4 * NCH];
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
            const uint4 v = __ldg(cp + k);
            wd[4 * k] = v.x; wd[4 * k + 1] = v.y; wd[4 * k + 2] = v.z; wd[4 * k + 3] = v.w;
        }
        float rs = 0.0f;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const uint32_t g = o ? wd[2 * j + 2] : wd[2 * j];
            uint32_t tg; float ta[3];
            tgt(dr, j, tg, ta[0], ta[1], ta[2]);
            const uint32_t d = __vabsdiffu4(g, tg);
            dg = __dp4a(d, d, dg);
            if (TWO) {
                const uint32_t sv = o ? wd[2 * j + 3] : wd[2 * j + 1];
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    const float dl = __fsub_rn(ta[ch], u8f(sv, ch));
                    rs = __fmaf_rn(dl, dl, rs);
                }
            }
        }
        if (TWO) ds = __fadd_rn(ds, rs);
    };
    // Loss with partial-distance elimination: every term is >= 0 and round-to-nearest sums are
    // monotone, so once the partial loss after the first P rows is >= `bound` the full loss is too and
    // the candidate cannot win the strict select (D16); its remaining rows are never loaded.  Results
    // are unchanged: selected candidates are always evaluated in full, in the D20 order.
    int cbase = 0;  // FB_COUNTERS: 0 propagation, 8 random search
    // partial + remainder bound (tail_reject) of the random search: the target's tail-row sums, set with the
    // patch-sum bound's target sums
    constexpr int S1 = PDE_I13_S1(P);
    constexpr bool TB = TL && CSB && SF == 0 && SFL == 0 && TWO && P == 2 && S1 < D;
    const bool use_tail = TB && use_csb && a.tail_off >= 0;
    const uint4* TAIL = use_tail ? reinterpret_cast<const uint4*>(T.src + a.tail_off) : nullptr;
    uint32_t tt01 = 0u, tt2 = 0u;
    float tta0 = 0.0f, tta1 = 0.0f, tta2 = 0.0f, ttm = 0.0f;
    auto loss = [&](int sr, int sc, float bound, bool tail) -> float {
        uint32_t dg = 0u;
        float dgf = 0.0f, ds = 0.0f;
        auto gsum = [&]() { return SF == 1 ? dgf : __uint2float_rn(dg); };
        constexpr int S2 = PDE_I13_S2(P);
        FB_CNT(cbase + 0);
        const uint4 q = TB && tail ? __ldg(TAIL + sr * w + sc) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int dr = 0; dr < S1; ++dr) row(sr, sc, dr, dg, dgf, ds);
        const float part = partial_loss(a.alpha, gsum(), ds, TWO);
        if (part >= bound) { FB_CNT(cbase + 1); return __int_as_float(0x7f800000); }
        if (TB && tail && tail_reject<(D - S1) * D>(q, tt01, tt2, tta0, tta1, tta2, ttm, a.alpha, part, bound)) {
            FB_CNT(21);
            return __int_as_float(0x7f800000);
        }
        if (S2 < D) {
#pragma unroll
            for (int dr = S1; dr < S2; ++dr) row(sr, sc, dr, dg, dgf, ds);
            if (partial_loss(a.alpha, gsum(), ds, TWO) >= bound) { FB_CNT(cbase + 2); return __int_as_float(0x7f800000); }
        }
#pragma unroll
        for (int dr = (S2 < D ? S2 : S1); dr < D; ++dr) row(sr, sc, dr, dg, dgf, ds);
        FB_CNT(cbase + 3);
        const float fg = gsum();
        return TWO ? __fmaf_rn(a.alpha, fg, ds) : fg;
    };
    // A candidate equal to the incumbent has exactly the incumbent's loss (same aux within the
    // iteration), so it cannot win the strict select (D16): skipping it changes nothing.
    auto select = [&](int2& f, float& e, int sr, int sc, bool tail) {
        if (sr == f.x && sc == f.y) { FB_CNT(cbase + 5); return; }
        if (sr != f.x || sc != f.y) {  // an incumbent-equal candidate cannot win (see select)
            const float e2 = loss(sr, sc, e, tail);
            if (e2 < e) { f = make_int2(sr, sc); e = e2; FB_CNT(cbase + 4); }
        }
    };
    const int2* Fi = a.Fin + t * a.fstride;
    const int i = r * w + c;
    int2 f = make_int2(0, 0);
    float e = 0.0f;
    // Fields 1-3 in one loop with one select site (smaller code: the fused kernel is sensitive to instruction-
    // cache misses), converged at the top of every iteration:
    //   fld 0: field 1, d = (+1,0), neighbour (r+1, c) of F_in (= the field-0 result), clamped (D11);
    //   fld 1: field 2, d = (0,-1), neighbour (r, c-1) of the field-1 result (lane - 1, by shuffle);
    //   fld 2: field 3, d = (0,+1), neighbour (r, c+1) of the field-2 result (lane + 1); halo lanes skip it.
    if (valid) {
        f = Fi[i];
        e = a.E[t * a.fstride + i];
    }
#pragma unroll 1
    for (int fld = 0; fld < 3; ++fld) {
        const int2 nb = make_int2(__shfl_sync(0xffffffffu, f.x, fld == 1 ? lane - 1 : lane + 1),
                                  __shfl_sync(0xffffffffu, f.y, fld == 1 ? lane - 1 : lane + 1));
        int2 cand;
        bool has;
        if (fld == 0) {
            has = valid;
            const int2 fn = valid && r + 1 < h ? Fi[i + w] : f;
            cand = make_int2(max(fn.x - 1, 0), fn.y);
        } else if (fld == 1) {
            has = valid && lane > 0;
            const int2 fn = c > 0 ? nb : f;
            cand = make_int2(fn.x, min(fn.y + 1, w - 1));
        } else {
            has = valid && lane > 0 && lane < 31;
            const int2 fn = c + 1 < w ? nb : f;
            cand = make_int2(fn.x, max(fn.y - 1, 0));
        }
        if (has) select(f, e, cand.x, cand.y, false);
    }
    TSums ts{};
    if (use_csb) {  // target patch sums of the bound, warp converged: column sums over the D rows of the shared
                    // tile (columns 32.. by lanes 0..2P-1), then the D columns of each lane's patch by shuffles
        uint32_t cg[2][2] = {{0u, 0u}, {0u, 0u}};  // [main, extra] {g0 | g1 << 16, g2}
        float ca[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};  // {a0, a1, a2, max_c sum|a_c|}
        uint32_t cgt[2][2] = {{0u, 0u}, {0u, 0u}};  // the same over the tail rows [S1, D) (tail_reject)
        float cat[2][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            float b0 = 0.f, b1 = 0.f, b2 = 0.f;
#pragma unroll
            for (int dr = 0; dr < D; ++dr) {
                if (x == 1 && lane >= 2 * P) break;  // tile columns 32.. only
                const uint4 v = tT[CSB ? wy + dr : 0][CSB ? lane + 32 * x : 0];
                if (SF == 1) { cg[x][0] += (v.x & 0x3FFu) | (((v.x >> 10) & 0x3FFu) << 16); cg[x][1] += v.x >> 20; }
                else { cg[x][0] += (v.x & 0xFFu) | (((v.x >> 8) & 0xFFu) << 16); cg[x][1] += (v.x >> 16) & 0xFFu; }
                const float t0 = __uint_as_float(v.y), t1 = __uint_as_float(v.z), t2 = __uint_as_float(v.w);
                ca[x][0] = __fadd_rn(ca[x][0], t0); ca[x][1] = __fadd_rn(ca[x][1], t1);
                ca[x][2] = __fadd_rn(ca[x][2], t2);
                b0 = __fadd_ru(b0, fabsf(t0)); b1 = __fadd_ru(b1, fabsf(t1)); b2 = __fadd_ru(b2, fabsf(t2));
                if (TB && dr >= S1) {
                    cgt[x][0] += (v.x & 0xFFu) | (((v.x >> 8) & 0xFFu) << 16); cgt[x][1] += (v.x >> 16) & 0xFFu;
                    cat[x][0] = __fadd_rn(cat[x][0], t0); cat[x][1] = __fadd_rn(cat[x][1], t1);
                    cat[x][2] = __fadd_rn(cat[x][2], t2);
                }
            }
            ca[x][3] = fmaxf(b0, fmaxf(b1, b2));
        }
        uint32_t g01 = cg[0][0], g2 = cg[0][1];  // 16-bit lanes: every sum <= D^2 * 1020 < 2^16
        float a0 = ca[0][0], a1 = ca[0][1], a2 = ca[0][2], m = ca[0][3];
        if (TB) { tt01 = cgt[0][0]; tt2 = cgt[0][1]; tta0 = cat[0][0]; tta1 = cat[0][1]; tta2 = cat[0][2]; }
#pragma unroll
        for (int j = 1; j < D; ++j) {
            const bool own = lane + j < 32;
            const int src = (lane + j) & 31;
            const uint32_t x0 = __shfl_down_sync(0xffffffffu, cg[0][0], j), y0 = __shfl_sync(0xffffffffu, cg[1][0], src);
            const uint32_t x1 = __shfl_down_sync(0xffffffffu, cg[0][1], j), y1 = __shfl_sync(0xffffffffu, cg[1][1], src);
            const float p0 = __shfl_down_sync(0xffffffffu, ca[0][0], j), q0 = __shfl_sync(0xffffffffu, ca[1][0], src);
            const float p1 = __shfl_down_sync(0xffffffffu, ca[0][1], j), q1 = __shfl_sync(0xffffffffu, ca[1][1], src);
            const float p2 = __shfl_down_sync(0xffffffffu, ca[0][2], j), q2 = __shfl_sync(0xffffffffu, ca[1][2], src);
            const float p3 = __shfl_down_sync(0xffffffffu, ca[0][3], j), q3 = __shfl_sync(0xffffffffu, ca[1][3], src);
            g01 += own ? x0 : y0; g2 += own ? x1 : y1;
            a0 = __fadd_rn(a0, own ? p0 : q0); a1 = __fadd_rn(a1, own ? p1 : q1); a2 = __fadd_rn(a2, own ? p2 : q2);
            m = __fadd_ru(m, own ? p3 : q3);
            if (TB) {
                const uint32_t u0 = __shfl_down_sync(0xffffffffu, cgt[0][0], j), v0 = __shfl_sync(0xffffffffu, cgt[1][0], src);
                const uint32_t u1 = __shfl_down_sync(0xffffffffu, cgt[0][1], j), v1 = __shfl_sync(0xffffffffu, cgt[1][1], src);
                const float r0 = __shfl_down_sync(0xffffffffu, cat[0][0], j), s0 = __shfl_sync(0xffffffffu, cat[1][0], src);
                const float r1 = __shfl_down_sync(0xffffffffu, cat[0][1], j), s1 = __shfl_sync(0xffffffffu, cat[1][1], src);
                const float r2 = __shfl_down_sync(0xffffffffu, cat[0][2], j), s2 = __shfl_sync(0xffffffffu, cat[1][2], src);
                tt01 += own ? u0 : v0; tt2 += own ? u1 : v1;
                tta0 = __fadd_rn(tta0, own ? r0 : s0); tta1 = __fadd_rn(tta1, own ? r1 : s1);
                tta2 = __fadd_rn(tta2, own ? r2 : s2);
            }
        }
        constexpr float gsc = SF == 1 ? 0.25f : 1.0f;
        ts = TSums{(float)(g01 & 0xFFFFu) * gsc, (float)(g01 >> 16) * gsc, (float)g2 * gsc, a0, a1, a2,
                   csb_margin<D>(m)};
        ttm = ts.m;
    }
    if (!valid || lane == 0 || lane == 31) return;  // halo lanes only fed fields 1-2
#pragma unroll
    for (int z = 0; z < 2; ++z)  // tracking fields T_{i-1}, T_{i+1} (D42)
        if (T.trk[z]) {
            const int2 g = __ldg(&T.trk[z][i]);
            select(f, e, g.x, g.y, false);
        }
    const uint4* SUMS = use_csb ? reinterpret_cast<const uint4*>(T.src + a.sum_off) : nullptr;
    constexpr float ssc = SF == 1 ? 0.25f : 1.0f;  // source sums: n = v (SF8) or n = 4 v (SF10)
    cbase = 8;
    uint4 ru = make_uint4(0u, 0u, 0u, 0u);
#if FB_RS_PREFETCH
    // Software-pipelined bound (exact): step s+1's candidate and its patch-sum texel are loaded before step s is
    // decided, from the incumbent as it stands; most steps are rejected by the bound and leave f unchanged, so
    // the load is the one step s+1 needs; when step s moves f the candidate is recomputed and reloaded.
    if (SFL == 0 && CSB && use_csb && a.rs_k > 0) {
        ru = rs_block(a, T, i, 0);
        int2 o = rs_offset(a, ru, 0);
        int sr = clampi(f.x + o.x, 0, h - 1), sc = clampi(f.y + o.y, 0, w - 1);
        uint4 sm = __ldg(SUMS + sr * w + sc);
        for (int s = 0; s < a.rs_k; ++s) {
            uint4 run = ru, smn = make_uint4(0u, 0u, 0u, 0u);
            int2 on = make_int2(0, 0);
            int srn = 0, scn = 0;
            const bool more = s + 1 < a.rs_k;
            if (more) {
                if (!((s + 1) & 1)) run = rs_block(a, T, i, s + 1);
                on = rs_offset(a, run, s + 1);
                srn = clampi(f.x + on.x, 0, h - 1); scn = clampi(f.y + on.y, 0, w - 1);
                smn = __ldg(SUMS + srn * w + scn);
            }
            if ((sr != f.x || sc != f.y) && csb_reject<D, TWO>(sm, ts, ssc, a.alpha, e)) {
                FB_CNT(14);
            } else {
                const int2 f0 = f;
                select(f, e, sr, sc, use_tail);
                if (more && (f.x != f0.x || f.y != f0.y)) {
                    srn = clampi(f.x + on.x, 0, h - 1); scn = clampi(f.y + on.y, 0, w - 1);
                    smn = __ldg(SUMS + srn * w + scn);
                }
            }
            ru = run; sr = srn; sc = scn; sm = smn;
        }
    } else
#endif
    for (int s = 0; s < a.rs_k; ++s) {
        if (!(s & 1)) ru = rs_block(a, T, i, s);
        const int2 o = rs_offset(a, ru, s);
        const int sr = clampi(f.x + o.x, 0, h - 1), sc = clampi(f.y + o.y, 0, w - 1);
        if (CSB && use_csb && (sr != f.x || sc != f.y) &&
            (SFL == 1 ? csb_reject_f<D, TWO>(__ldg(SUMS + 2 * (sr * w + sc)), __ldg(SUMS + 2 * (sr * w + sc) + 1), ts,
                                             a.alpha, e)
                      : csb_reject<D, TWO>(__ldg(SUMS + sr * w + sc), ts, ssc, a.alpha, e))) {
            FB_CNT(14);
            continue;
        }
        select(f, e, sr, sc, use_tail);
    }
    FB_ASSERT((unsigned)f.x < (unsigned)h && (unsigned)f.y < (unsigned)w);
    a.Fout[t * a.fstride + i] = f;
    if (a.Eout) a.Eout[t * a.fstride + i] = e;  // never a.E: halo lanes of other tiles read it
}

// ---- level-0 variant for p = 3, 4: SF8 source, TF16 target tile in shared memory -----------------
// The target patch of p >= 3 does not fit in registers, so it is staged per tile; the source rows and the
// exact integer guide term (every partial < 2^24 for p <= 4 at level 0) are those of k_field_fast.
template <int P, bool TWO, int PHASE, int SFL = 0, int SF = 0, bool PR = false>
// Source rows of the shared-memory-target kernel: 0 = from the aligned copy of the two SF8 copies (parity-free),
// 1 = from copy 0 with parity selects except in the paired accurate phase 0 (default), 2 = copy 0 everywhere.  Its
// candidates are coherent across lanes (the current F, the row-above neighbour's F), so reading one copy lets
// adjacent lanes share lines: N=48 balanced field0.L0 58.7 -> 54.1 ms, fast 22.3 -> 21.5, config-5 shard
// 107.3 -> 98.9 ms; the paired phase 0 loses with copy 0 (66.5 -> 74.0 ms: two rows of selects per tap), and so
// does the fused fields-1-3 kernel (issue-bound on its selects).
#ifndef FB_MID_COPY0
#define FB_MID_COPY0 1
#endif
#ifndef MID_MINB
#define MID_MINB 8  // p = 2 (phase 0): 8 CTAs/SM at 32 registers beats 5 at 44 (balanced N=48: 68 -> 62 ms)
#endif
#ifndef MID3_MINB
#define MID3_MINB 4  // p = 3: 64 registers, 4 CTAs/SM (config-5 shard 27.3 -> 30.6 G evals/s)
#endif
#ifndef MID10_MINB
#define MID10_MINB 4  // level-1 SF10 variant (more ALU per tap than the u8 one)
#endif
#ifndef MIDP_MINB
#define MIDP_MINB 6  // phase 0 with E init and field 0 scored together (accurate N=48: field0.L0 73.4 -> 67.8 ms)
#endif
__global__ void __launch_bounds__(TILE_X* TILE_Y, PR ? MIDP_MINB : (P == 2 ? (SF ? MID10_MINB : MID_MINB) : (P == 3 ? MID3_MINB : 1))) k_field_mid(FieldArgs a)
{
    constexpr int D = 2 * P + 1, SX = TILE_X + 2 * P, SY = TILE_Y + 2 * P;
    constexpr int NCH = (D + 2) / 2;  // 16-byte chunks covering D texels from an even start
    __shared__ uint4 tT[SY][SX];
    const int t = blockIdx.x / a.tiles_per_task;
    const int tile = blockIdx.x - t * a.tiles_per_task;
    const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
    const int h = a.L.h, w = a.L.w, pitch = a.L.pitch;
    const DTask T = a.tasks[t];
    {
        const uint4* Tt = reinterpret_cast<const uint4*>(T.tgt);
#if FB_TILE_TMA
        __shared__ uint64_t tbar;
        stage_tile_tma<SY, SX>(tT, Tt, pitch, a.L.rows, ty * TILE_Y - P + B, tx * TILE_X - P + B, &tbar);
#else
        for (int k = threadIdx.x; k < SX * SY; k += TILE_X * TILE_Y) {
            const int yy = k / SX, xx = k - yy * SX;
            const int pr = ty * TILE_Y + yy - P + B, pc = tx * TILE_X + xx - P + B;
            tT[yy][xx] = (pr < a.L.rows && pc < pitch) ? __ldg(&Tt[pr * pitch + pc]) : make_uint4(0u, 0u, 0u, 0u);
        }
        __syncthreads();
#endif
    }
    const int lx = threadIdx.x & (TILE_X - 1), ly = threadIdx.x / TILE_X;
    const int c = tx * TILE_X + lx, r = ty * TILE_Y + ly;
    // patch-sum bound of the random search (csb_reject): target sums while the warp is converged
    constexpr bool CSB = PHASE == 3 && SFL == 0;
    const bool use_csb = CSB && a.do_rs && a.sum_off >= 0;
    TSums ts{};
    if (use_csb)
        ts = tile_patch_sums<P>(lx, ly, [&](int yy, int xx, float (&v)[6]) {
            const uint4 q = tT[yy][xx];
            if (SF == 1) { v[0] = f10_0(q.x); v[1] = f10_1(q.x); v[2] = f10_2(q.x); }
            else { v[0] = (float)(q.x & 0xFFu); v[1] = (float)((q.x >> 8) & 0xFFu); v[2] = (float)((q.x >> 16) & 0xFFu); }
            v[3] = __uint_as_float(q.y); v[4] = __uint_as_float(q.z); v[5] = __uint_as_float(q.w);
        });
    if (r >= h || c >= w) return;
    const uint2* S = reinterpret_cast<const uint2*>(T.src + a.src_off);
    const int plane = a.L.rows * pitch;
    // SF = 1: level-1 SF10 source and TF10 target tile, the literal FP32 chains of D20 (see k_iter13_fast)
    auto row = [&](int sr, int sc, int dr, uint32_t& dg, float& dgf, float& ds) {
        const int idx = (sr + dr - P + B) * pitch + (sc - P + B);
        FB_ASSERT((unsigned)sr < (unsigned)h && (unsigned)sc < (unsigned)w && FB_ROW_OK(idx, a.L, D));
        if constexpr (SF == 1) {
            const uint4* cp = reinterpret_cast<const uint4*>(S + (size_t)(idx & 1) * plane + (idx & ~1));
            uint32_t wd[4 * NCH];
#pragma unroll
            for (int k = 0; k < NCH; ++k) {
                const uint4 v = __ldg(cp + k);
                wd[4 * k] = v.x; wd[4 * k + 1] = v.y; wd[4 * k + 2] = v.z; wd[4 * k + 3] = v.w;
            }
            float rg = 0.0f, rs = 0.0f;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const uint4 tv = tT[ly + dr][lx + j];
                const uint32_t gw = wd[2 * j], sw = wd[2 * j + 1];
                float dl;
                dl = __fsub_rn(b10_0(tv.x), b10_0(gw)); rg = __fmaf_rn(dl, dl, rg);
                dl = __fsub_rn(b10_1(tv.x), b10_1(gw)); rg = __fmaf_rn(dl, dl, rg);
                dl = __fsub_rn(b10_2(tv.x), b10_2(gw)); rg = __fmaf_rn(dl, dl, rg);
                if (TWO) {
                    dl = __fsub_rn(__uint_as_float(tv.y), f10_0(sw)); rs = __fmaf_rn(dl, dl, rs);
                    dl = __fsub_rn(__uint_as_float(tv.z), f10_1(sw)); rs = __fmaf_rn(dl, dl, rs);
                    dl = __fsub_rn(__uint_as_float(tv.w), f10_2(sw)); rs = __fmaf_rn(dl, dl, rs);
                }
            }
            dgf = __fadd_rn(dgf, rg);
            if (TWO) ds = __fadd_rn(ds, rs);
            return;
        }
        if (SFL == 1) {  // SF8F float style (blending-table cells): one 16-byte texel per tap
            const uint4* tp = reinterpret_cast<const uint4*>(T.src + a.src_off) + idx;
            float rs = 0.0f;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const uint4 v = __ldg(tp + j);
                const uint4 tv = tT[ly + dr][lx + j];
                const uint32_t d = __vabsdiffu4(v.x, tv.x);
                dg = __dp4a(d, d, dg);
                if (TWO) {
                    float dl = __fsub_rn(__uint_as_float(tv.y), __uint_as_float(v.y)); rs = __fmaf_rn(dl, dl, rs);
                    dl = __fsub_rn(__uint_as_float(tv.z), __uint_as_float(v.z)); rs = __fmaf_rn(dl, dl, rs);
                    dl = __fsub_rn(__uint_as_float(tv.w), __uint_as_float(v.w)); rs = __fmaf_rn(dl, dl, rs);
                }
            }
            if (TWO) ds = __fadd_rn(ds, rs);
            return;
        }
        constexpr bool C2 = kSF8Copies == 2 && (FB_MID_COPY0 == 0 || (FB_MID_COPY0 == 1 && PR));  // aligned copy, else
                                                                                                 // copy 0 + selects
        const uint4* cp = reinterpret_cast<const uint4*>(
            S + (C2 ? (size_t)(idx & 1) * plane + (idx & ~1) : (size_t)(idx & ~1)));
        const int o = C2 ? 0 : (idx & 1);
        uint32_t wd[4 * NCH];
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
            const uint4 v = __ldg(cp + k);
            wd[4 * k] = v.x; wd[4 * k + 1] = v.y; wd[4 * k + 2] = v.z; wd[4 * k + 3] = v.w;
        }
        float rs = 0.0f;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const uint4 tv = tT[ly + dr][lx + j];
            const uint32_t g = o ? wd[2 * j + 2] : wd[2 * j];
            const uint32_t d = __vabsdiffu4(g, tv.x);
            dg = __dp4a(d, d, dg);
            if (TWO) {
                const uint32_t sv = o ? wd[2 * j + 3] : wd[2 * j + 1];
                float dl = __fsub_rn(__uint_as_float(tv.y), u8f(sv, 0)); rs = __fmaf_rn(dl, dl, rs);
                dl = __fsub_rn(__uint_as_float(tv.z), u8f(sv, 1)); rs = __fmaf_rn(dl, dl, rs);
                dl = __fsub_rn(__uint_as_float(tv.w), u8f(sv, 2)); rs = __fmaf_rn(dl, dl, rs);
            }
        }
        if (TWO) ds = __fadd_rn(ds, rs);
    };
    auto loss = [&](int sr, int sc, float bound) -> float {
        uint32_t dg = 0u;
        float dgf = 0.0f, ds = 0.0f;
        auto gsum = [&]() { return SF == 1 ? dgf : __uint2float_rn(dg); };
        constexpr int S1 = PDE_GEN_S1(P), S2 = PDE_GEN_S2(P);
#pragma unroll
        for (int dr = 0; dr < S1; ++dr) row(sr, sc, dr, dg, dgf, ds);
        if (partial_loss(a.alpha, gsum(), ds, TWO) >= bound) return __int_as_float(0x7f800000);
        if (S2 < D) {
#pragma unroll
            for (int dr = S1; dr < S2; ++dr) row(sr, sc, dr, dg, dgf, ds);
            if (partial_loss(a.alpha, gsum(), ds, TWO) >= bound) return __int_as_float(0x7f800000);
        }
#pragma unroll
        for (int dr = (S2 < D ? S2 : S1); dr < D; ++dr) row(sr, sc, dr, dg, dgf, ds);
        const float fg = gsum();
        return TWO ? __fmaf_rn(a.alpha, fg, ds) : fg;
    };
    auto select = [&](int2& f, float& e, int sr, int sc) {
        if (sr == f.x && sc == f.y) return;  // incumbent-equal candidates cannot win
        const float e2 = loss(sr, sc, e);
        if (e2 < e) { f = make_int2(sr, sc); e = e2; }
    };
    const int2* Fi = a.Fin + t * a.fstride;
    const int i = r * w + c;
    int2 f = Fi[i];
    // PR (phase 0 of u8 sources, accurate mode): E <- L(F) and the field-0 candidate scored together, row by row,
    // so each target texel is read from the shared tile once for both (the kernel is bound by the L1/shared data
    // path).  Each loss keeps its own D20 chain, and the candidate is scored in full instead of with partial-
    // distance elimination, so the outcome equals E-init followed by the strict select.  Balanced mode keeps the
    // separate form: its propagation candidates are eliminated early more often (N=48: 61.9 vs 67.2 ms).
    constexpr bool PAIR0 = PR && PHASE == 0 && SF == 0 && SFL == 0;
    if (PAIR0 && a.einit) {
        const int dx = -a.step;  // field 0: d = (-1,0), jump-flood step (D41)
        const int nr = clampi(r + dx, 0, h - 1);  // D11
        const int2 fn = Fi[nr * w + c];
        const int cr = clampi(fn.x - dx, 0, h - 1), cc = clampi(fn.y, 0, w - 1);  // D10
        const bool two = cr != f.x || cc != f.y;
        uint32_t dgA = 0u, dgB = 0u;
        float dsA = 0.0f, dsB = 0.0f;
#pragma unroll
        for (int dr = 0; dr < D; ++dr) {
            uint32_t wa[4 * NCH], wb[4 * NCH];
            const int ia = (f.x + dr - P + B) * pitch + (f.y - P + B), ib = (cr + dr - P + B) * pitch + (cc - P + B);
            FB_ASSERT(FB_ROW_OK(ia, a.L, D) && FB_ROW_OK(ib, a.L, D));
            constexpr bool C2P = kSF8Copies == 2 && FB_MID_COPY0 < 2;  // aligned copy, else copy 0 + selects
            const uint4* pa = reinterpret_cast<const uint4*>(S + (C2P ? (size_t)(ia & 1) * plane : 0) + (ia & ~1));
            const uint4* pb = reinterpret_cast<const uint4*>(S + (C2P ? (size_t)(ib & 1) * plane : 0) + (ib & ~1));
            const int oa = C2P ? 0 : (ia & 1), ob = C2P ? 0 : (ib & 1);
#pragma unroll
            for (int k = 0; k < NCH; ++k) {
                const uint4 v = __ldg(pa + k);
                wa[4 * k] = v.x; wa[4 * k + 1] = v.y; wa[4 * k + 2] = v.z; wa[4 * k + 3] = v.w;
                const uint4 u = two ? __ldg(pb + k) : v;
                wb[4 * k] = u.x; wb[4 * k + 1] = u.y; wb[4 * k + 2] = u.z; wb[4 * k + 3] = u.w;
            }
            float ra = 0.0f, rb = 0.0f;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const uint4 tv = tT[ly + dr][lx + j];
                uint32_t d = __vabsdiffu4(oa ? wa[2 * j + 2] : wa[2 * j], tv.x);
                dgA = __dp4a(d, d, dgA);
                d = __vabsdiffu4(ob ? wb[2 * j + 2] : wb[2 * j], tv.x);
                dgB = __dp4a(d, d, dgB);
                if (TWO) {
                    const uint32_t sa = oa ? wa[2 * j + 3] : wa[2 * j + 1], sb = ob ? wb[2 * j + 3] : wb[2 * j + 1];
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) {
                        const float tc = __uint_as_float(ch == 0 ? tv.y : (ch == 1 ? tv.z : tv.w));
                        float dl = __fsub_rn(tc, u8f(sa, ch)); ra = __fmaf_rn(dl, dl, ra);
                        dl = __fsub_rn(tc, u8f(sb, ch)); rb = __fmaf_rn(dl, dl, rb);
                    }
                }
            }
            if (TWO) { dsA = __fadd_rn(dsA, ra); dsB = __fadd_rn(dsB, rb); }
        }
        const float eA = TWO ? __fmaf_rn(a.alpha, __uint2float_rn(dgA), dsA) : __uint2float_rn(dgA);
        const float eB = TWO ? __fmaf_rn(a.alpha, __uint2float_rn(dgB), dsB) : __uint2float_rn(dgB);
        float e = eA;
        if (two && eB < eA) { f = make_int2(cr, cc); e = eB; }
        a.Fout[t * a.fstride + i] = f;
        a.E[t * a.fstride + i] = e;
        return;
    }
    float e = PHASE == 0 && a.einit ? loss(f.x, f.y, __int_as_float(0x7f800000)) : a.E[t * a.fstride + i];
    {
        const int dx = (PHASE == 0 ? -1 : (PHASE == 1 ? 1 : 0)) * a.step;
        const int dy = (PHASE == 2 ? -1 : (PHASE == 3 ? 1 : 0)) * a.step;
        const int nr = clampi(r + dx, 0, h - 1), nc = clampi(c + dy, 0, w - 1);  // D11
        const int2 fn = Fi[nr * w + nc];
        select(f, e, clampi(fn.x - dx, 0, h - 1), clampi(fn.y - dy, 0, w - 1));  // D10
    }
    if (PHASE == 3 && a.do_rs) {
#pragma unroll
        for (int z = 0; z < 2; ++z)  // tracking fields (D42)
            if (T.trk[z]) {
                const int2 g = __ldg(&T.trk[z][i]);
                select(f, e, g.x, g.y);
            }
        const uint4* SUMS = use_csb ? reinterpret_cast<const uint4*>(T.src + a.sum_off) : nullptr;
        constexpr float ssc = SF == 1 ? 0.25f : 1.0f;  // source sums: n = v (SF8) or n = 4 v (SF10)
        uint4 ru = make_uint4(0u, 0u, 0u, 0u);
        for (int s = 0; s < a.rs_k; ++s) {
            if (!(s & 1)) ru = rs_block(a, T, i, s);
            const int2 o = rs_offset(a, ru, s);
            const int sr = clampi(f.x + o.x, 0, h - 1), sc = clampi(f.y + o.y, 0, w - 1);
            if (CSB && use_csb && (sr != f.x || sc != f.y) &&
                csb_reject<D, TWO>(__ldg(SUMS + sr * w + sc), ts, ssc, a.alpha, e))
                continue;
            select(f, e, sr, sc);
        }
    }
    FB_ASSERT((unsigned)f.x < (unsigned)h && (unsigned)f.y < (unsigned)w);
    a.Fout[t * a.fstride + i] = f;
    a.E[t * a.fstride + i] = e;
}

// ---- general variant: SF32 source, TF32 target staged in shared memory (any level, P <= 4) -------

template <int P, bool TWO, int PHASE, int SFMT, bool PW = false>
__global__ void __launch_bounds__(TILE_X* TILE_Y) k_field_gen(FieldArgs a)
{
    constexpr int D = 2 * P + 1, SX = TILE_X + 2 * P, SY = TILE_Y + 2 * P;
    __shared__ float4 t0[SY][SX];  // {G.r, G.g, G.b, aux.r}
    __shared__ float2 t1[SY][SX];  // {aux.g, aux.b}
    const int t = blockIdx.x / a.tiles_per_task;
    const int tile = blockIdx.x - t * a.tiles_per_task;
    const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
    const int h = a.L.h, w = a.L.w, pitch = a.L.pitch;
    const DTask T = a.tasks[t];
    // Exact packed sources (SF10 at level 1, SF16 at levels 2-4): the target guide is held in the tile biased by
    // the magic of the source decode (2^21 / 2^11 for SF10 channels 0, 2 / 1; 2^(23-2k) for SF16), so that the guide
    // delta of D20 is one FSUB of two biased values -- exact (same binade, Sterbenz) and equal to t - s -- and the
    // source guide needs no unbiasing FADD.  The bias is exact: level-k values are multiples of 4^-k below 256.
    constexpr bool GB = SFMT == SF10 || SFMT == SF16;
    const uint32_t ex = (uint32_t)(75 - a.L.k) << 24;
    const float gb0 = SFMT == SF10 ? 2097152.0f : __uint_as_float(ex), gb1 = SFMT == SF10 ? 2048.0f : gb0,
                gb2 = SFMT == SF10 ? 2097152.0f : gb0;
    {
        const float4* Tt = reinterpret_cast<const float4*>(T.tgt);
        for (int k = threadIdx.x; k < SX * SY; k += TILE_X * TILE_Y) {
            const int yy = k / SX, xx = k - yy * SX;
            const int pr = ty * TILE_Y + yy - P + B, pc = tx * TILE_X + xx - P + B;  // padded coords
            float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
            if (pr < a.L.rows && pc < pitch) {
                v0 = __ldg(&Tt[2 * (pr * pitch + pc)]);
                v1 = __ldg(&Tt[2 * (pr * pitch + pc) + 1]);
            }
            if (GB) { v0.x = __fadd_rn(v0.x, gb0); v0.y = __fadd_rn(v0.y, gb1); v0.z = __fadd_rn(v0.z, gb2); }
            t0[yy][xx] = v0;
            t1[yy][xx] = make_float2(v1.x, v1.y);
        }
    }
    __syncthreads();
    const int lx = threadIdx.x & (TILE_X - 1), ly = threadIdx.x / TILE_X;
    // Patch-sum bound of the random search (csb_reject, levels with exact packed sources): the target patch sums,
    // computed while the warp is converged -- column sums over the D rows of the tile (tile columns 32.. by lanes
    // 0..2P-1), then the D columns of each lane's patch by shuffles.  Guide sums are exact (multiples of 4^-k
    // below 2^21 units).
    constexpr bool CSB = PHASE == 3 && !PW && (SFMT == SF10 || SFMT == SF16);
    const bool use_csb = CSB && a.do_rs && a.sum_off >= 0;
    TSums ts{};
    if (use_csb)
        ts = tile_patch_sums<P>(lx, ly, [&](int yy, int xx, float (&v)[6]) {
            const float4 q0 = t0[yy][xx];
            const float2 q1 = t1[yy][xx];
            v[0] = __fsub_rn(q0.x, gb0); v[1] = __fsub_rn(q0.y, gb1); v[2] = __fsub_rn(q0.z, gb2);  // exact unbias
            v[3] = q0.w; v[4] = q1.x; v[5] = q1.y;
        });
    const int c = tx * TILE_X + lx, r = ty * TILE_Y + ly;
    if (r >= h || c >= w) return;
    const float4* S = reinterpret_cast<const float4*>(T.src + a.src_off);
    const uint4* S16 = reinterpret_cast<const uint4*>(T.src + a.src_off);
    float pa[PW ? D : 1][PW ? D : 1][3];  // PAIRWISE reference patch (Eq. 10, D39)
    if (PW) {
        const int2 q = __ldg(&T.pF[r * w + c]);
#pragma unroll
        for (int dr = 0; dr < D; ++dr)
#pragma unroll
            for (int dc = 0; dc < D; ++dc) {
                const int idx = (q.x + dr - P + B) * pitch + (q.y + dc - P + B);
                FB_ASSERT((unsigned)q.x < (unsigned)h && (unsigned)q.y < (unsigned)w);
                if (SFMT == SF10) {
                    const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(T.psrc + a.src_off) + 2 * idx + 1);
                    pa[PW ? dr : 0][PW ? dc : 0][0] = f10_0(v);
                    pa[PW ? dr : 0][PW ? dc : 0][1] = f10_1(v);
                    pa[PW ? dr : 0][PW ? dc : 0][2] = f10_2(v);
                } else if (SFMT == SF16) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4*>(T.psrc + a.src_off) + idx);
                    pa[PW ? dr : 0][PW ? dc : 0][0] = u16f(v.z, 0x7410u, ex);
                    pa[PW ? dr : 0][PW ? dc : 0][1] = u16f(v.z, 0x7432u, ex);
                    pa[PW ? dr : 0][PW ? dc : 0][2] = u16f(v.w, 0x7410u, ex);
                } else {
                    const float4 v0 = __ldg(reinterpret_cast<const float4*>(T.psrc + a.src_off) + 2 * idx);
                    const float4 v1 = __ldg(reinterpret_cast<const float4*>(T.psrc + a.src_off) + 2 * idx + 1);
                    pa[PW ? dr : 0][PW ? dc : 0][0] = v0.w;
                    pa[PW ? dr : 0][PW ? dc : 0][1] = v1.x;
                    pa[PW ? dr : 0][PW ? dc : 0][2] = v1.y;
                }
            }
    }
    // source texel dc of a patch row starting at padded texel `base` (SF10: from the row's preloaded words wd)
    auto texel = [&](const uint32_t* wd, int base, int dc, float4& s0, float4& s1) {
        if (SFMT == SF10) {  // guide biased (see GB), style exact
            const uint32_t gw = wd[SFMT == SF10 ? 2 * dc : 0], sw = wd[SFMT == SF10 ? 2 * dc + 1 : 0];
            s0 = make_float4(b10_0(gw), b10_1(gw), b10_2(gw), TWO ? f10_0(sw) : 0.0f);
            s1 = TWO ? make_float4(f10_1(sw), f10_2(sw), 0.0f, 0.0f) : s0;
        } else if (SFMT == SF16) {
            const uint4 v = __ldg(&S16[base + dc]);
            s0 = make_float4(__uint_as_float(__byte_perm(v.x, ex, 0x7410u)), __uint_as_float(__byte_perm(v.x, ex, 0x7432u)),
                             __uint_as_float(__byte_perm(v.y, ex, 0x7410u)), TWO ? u16f(v.z, 0x7410u, ex) : 0.0f);
            s1 = TWO ? make_float4(u16f(v.z, 0x7432u, ex), u16f(v.w, 0x7410u, ex), 0.0f, 0.0f) : s0;
        } else {
            s0 = __ldg(&S[2 * (base + dc)]);
            s1 = TWO ? __ldg(&S[2 * (base + dc) + 1]) : s0;
        }
    };
    constexpr int NCH = (D + 2) / 2;
    auto preload = [&](int base, uint32_t (&wd)[SFMT == SF10 ? 4 * NCH : 1]) {  // SF10: the row's aligned copy
        if (SFMT == SF10) {
            const uint4* cp = reinterpret_cast<const uint4*>(
                reinterpret_cast<const uint2*>(T.src + a.src_off) + (size_t)(base & 1) * (a.L.rows * pitch) + (base & ~1));
#pragma unroll
            for (int k = 0; k < NCH; ++k) {
                const uint4 v = __ldg(cp + k);
                wd[SFMT == SF10 ? 4 * k : 0] = v.x; wd[SFMT == SF10 ? 4 * k + 1 : 0] = v.y;
                wd[SFMT == SF10 ? 4 * k + 2 : 0] = v.z; wd[SFMT == SF10 ? 4 * k + 3 : 0] = v.w;
            }
        }
    };
    auto row = [&](int sr, int sc, int dr, float& dg, float& ds) {
        const int base = (sr + dr - P + B) * pitch + (sc - P + B);
        FB_ASSERT((unsigned)sr < (unsigned)h && (unsigned)sc < (unsigned)w && FB_ROW_OK(base, a.L, D));
        float rg = 0.0f, rs = 0.0f;
        // SF10: the row's texel pairs from the copy in which it starts 16-byte aligned (as SF8)
        uint32_t wd[SFMT == SF10 ? 4 * NCH : 1];
        preload(base, wd);
#pragma unroll
        for (int dc = 0; dc < D; ++dc) {
            float4 s0, s1;
            texel(wd, base, dc, s0, s1);
            const float4 q0 = t0[ly + dr][lx + dc];
            float dl;
            dl = __fsub_rn(q0.x, s0.x); rg = __fmaf_rn(dl, dl, rg);
            dl = __fsub_rn(q0.y, s0.y); rg = __fmaf_rn(dl, dl, rg);
            dl = __fsub_rn(q0.z, s0.z); rg = __fmaf_rn(dl, dl, rg);
            if (TWO) {
                float ar, ag, ab;
                if (PW) {
                    ar = pa[PW ? dr : 0][PW ? dc : 0][0]; ag = pa[PW ? dr : 0][PW ? dc : 0][1];
                    ab = pa[PW ? dr : 0][PW ? dc : 0][2];
                } else {
                    const float2 q1 = t1[ly + dr][lx + dc];
                    ar = q0.w; ag = q1.x; ab = q1.y;
                }
                dl = __fsub_rn(ar, s0.w); rs = __fmaf_rn(dl, dl, rs);
                dl = __fsub_rn(ag, s1.x); rs = __fmaf_rn(dl, dl, rs);
                dl = __fsub_rn(ab, s1.y); rs = __fmaf_rn(dl, dl, rs);
            }
        }
        dg = __fadd_rn(dg, rg);
        if (TWO) ds = __fadd_rn(ds, rs);
    };
    // Partial-distance elimination (see k_field_fast): monotone FP32 partial sums of non-negative terms.
    auto loss = [&](int sr, int sc, float bound) -> float {
        float dg = 0.0f, ds = 0.0f;
        constexpr int S1 = PDE_GEN_S1(P), S2 = PDE_GEN_S2(P);
#pragma unroll
        for (int dr = 0; dr < S1; ++dr) row(sr, sc, dr, dg, ds);
        if (partial_loss(a.alpha, dg, ds, TWO) >= bound) return __int_as_float(0x7f800000);
        if (S2 < D) {
#pragma unroll
            for (int dr = S1; dr < S2; ++dr) row(sr, sc, dr, dg, ds);
            if (partial_loss(a.alpha, dg, ds, TWO) >= bound) return __int_as_float(0x7f800000);
        }
#pragma unroll
        for (int dr = (S2 < D ? S2 : S1); dr < D; ++dr) row(sr, sc, dr, dg, ds);
        return TWO ? __fmaf_rn(a.alpha, dg, ds) : dg;
    };
    const int2* Fi = a.Fin + t * a.fstride;
    const int i = r * w + c;
    int2 f = Fi[i];
    // Accurate mode (a.pair0): E <- L(F) and the field-0 candidate scored together row by row, each target texel
    // read from the tile once for both (as k_field_mid's PR form; exact: the candidate is scored in full and
    // selected strictly).
    if (PHASE == 0 && TWO && !PW && a.einit && a.pair0) {
        const int dx = -a.step;  // field 0: d = (-1,0), jump-flood step (D41)
        const int2 fn = Fi[clampi(r + dx, 0, h - 1) * w + c];
        const int cr = clampi(fn.x - dx, 0, h - 1), cc = clampi(fn.y, 0, w - 1);  // D11, D10
        const bool two = cr != f.x || cc != f.y;
        float dgA = 0.0f, dsA = 0.0f, dgB = 0.0f, dsB = 0.0f;
#pragma unroll
        for (int dr = 0; dr < D; ++dr) {
            const int ba = (f.x + dr - P + B) * pitch + (f.y - P + B), bb = (cr + dr - P + B) * pitch + (cc - P + B);
            uint32_t wa[SFMT == SF10 ? 4 * NCH : 1], wb[SFMT == SF10 ? 4 * NCH : 1];
            preload(ba, wa);
            if (two) preload(bb, wb);
            float rga = 0.0f, rsa = 0.0f, rgb = 0.0f, rsb = 0.0f;
#pragma unroll
            for (int dc = 0; dc < D; ++dc) {
                const float4 q0 = t0[ly + dr][lx + dc];
                const float2 q1 = t1[ly + dr][lx + dc];
                float4 s0, s1;
                texel(wa, ba, dc, s0, s1);
                float dl;
                dl = __fsub_rn(q0.x, s0.x); rga = __fmaf_rn(dl, dl, rga);
                dl = __fsub_rn(q0.y, s0.y); rga = __fmaf_rn(dl, dl, rga);
                dl = __fsub_rn(q0.z, s0.z); rga = __fmaf_rn(dl, dl, rga);
                dl = __fsub_rn(q0.w, s0.w); rsa = __fmaf_rn(dl, dl, rsa);
                dl = __fsub_rn(q1.x, s1.x); rsa = __fmaf_rn(dl, dl, rsa);
                dl = __fsub_rn(q1.y, s1.y); rsa = __fmaf_rn(dl, dl, rsa);
                if (two) {
                    texel(wb, bb, dc, s0, s1);
                    dl = __fsub_rn(q0.x, s0.x); rgb = __fmaf_rn(dl, dl, rgb);
                    dl = __fsub_rn(q0.y, s0.y); rgb = __fmaf_rn(dl, dl, rgb);
                    dl = __fsub_rn(q0.z, s0.z); rgb = __fmaf_rn(dl, dl, rgb);
                    dl = __fsub_rn(q0.w, s0.w); rsb = __fmaf_rn(dl, dl, rsb);
                    dl = __fsub_rn(q1.x, s1.x); rsb = __fmaf_rn(dl, dl, rsb);
                    dl = __fsub_rn(q1.y, s1.y); rsb = __fmaf_rn(dl, dl, rsb);
                }
            }
            dgA = __fadd_rn(dgA, rga); dsA = __fadd_rn(dsA, rsa);
            dgB = __fadd_rn(dgB, rgb); dsB = __fadd_rn(dsB, rsb);
        }
        float e = __fmaf_rn(a.alpha, dgA, dsA);
        const float eB = __fmaf_rn(a.alpha, dgB, dsB);
        if (two && eB < e) { f = make_int2(cr, cc); e = eB; }
        a.Fout[t * a.fstride + i] = f;
        a.E[t * a.fstride + i] = e;
        return;
    }
    float e = PHASE == 0 && a.einit ? loss(f.x, f.y, __int_as_float(0x7f800000)) : a.E[t * a.fstride + i];
    {
        const int dx = (PHASE == 0 ? -1 : (PHASE == 1 ? 1 : 0)) * a.step;  // jump-flood step (D41)
        const int dy = (PHASE == 2 ? -1 : (PHASE == 3 ? 1 : 0)) * a.step;
        const int nr = clampi(r + dx, 0, h - 1), nc = clampi(c + dy, 0, w - 1);  // D11
        const int2 fn = Fi[nr * w + nc];
        const int sr = clampi(fn.x - dx, 0, h - 1), sc = clampi(fn.y - dy, 0, w - 1);  // D10
        if (sr != f.x || sc != f.y) {  // an incumbent-equal candidate cannot win (see select)
            const float e2 = loss(sr, sc, e);
            if (e2 < e) { f = make_int2(sr, sc); e = e2; }
        }
    }
    if (PHASE == 3 && a.do_rs) {
#pragma unroll
        for (int z = 0; z < 2; ++z)  // tracking fields T_{i-1}, T_{i+1} (D42)
            if (T.trk[z]) {
                const int2 g = __ldg(&T.trk[z][i]);
                if (g.x != f.x || g.y != f.y) {
                    const float e2 = loss(g.x, g.y, e);
                    if (e2 < e) { f = g; e = e2; }
                }
            }
        const uint4* SUMS = use_csb ? reinterpret_cast<const uint4*>(T.src + a.sum_off) : nullptr;
        const float scale = __uint_as_float((uint32_t)(127 - 2 * a.L.k) << 23);  // 4^-k: unit of the source sums
        uint4 ru = make_uint4(0u, 0u, 0u, 0u);
        for (int s = 0; s < a.rs_k; ++s) {
            if (!(s & 1)) ru = rs_block(a, T, i, s);
            const int2 o = rs_offset(a, ru, s);
            const int sr = clampi(f.x + o.x, 0, h - 1), sc = clampi(f.y + o.y, 0, w - 1);
            if (sr != f.x || sc != f.y) {
                if (CSB && use_csb && csb_reject<D, TWO>(__ldg(SUMS + sr * w + sc), ts, scale, a.alpha, e)) continue;
                const float e2 = loss(sr, sc, e);
                if (e2 < e) { f = make_int2(sr, sc); e = e2; }
            }
        }
    }
    FB_ASSERT((unsigned)f.x < (unsigned)h && (unsigned)f.y < (unsigned)w);
    a.Fout[t * a.fstride + i] = f;
    a.E[t * a.fstride + i] = e;
}

// ------------------------------------------------------------------------------------ launchers
static inline dim3 grid1d(long long n, int y, int threads = 256)
{
    long long b = (n + threads - 1) / threads;
    if (b > 148 * 16) b = 148 * 16;
    if (b < 1) b = 1;
    return dim3((unsigned)b, (unsigned)y);
}

// Launches with one grid row per frame / task / output (blockIdx.y) are split into chunks of at most 65535
// rows (the grid.y limit), each with its base pointers advanced by the chunk's first row.
constexpr int kMaxGridY = 65535;
template <class Launch>
static cudaError_t for_y_chunks(long long n, Launch&& launch)
{
    for (long long y0 = 0; y0 < n; y0 += kMaxGridY) {
        launch(y0, (int)std::min<long long>(kMaxGridY, n - y0));
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_u8_to_pyr0(const uint8_t* frames, float4* pyr, int Bn, int H, int W, long long pyr_stride,
                              cudaStream_t s)
{
    return for_y_chunks(Bn, [&](long long y0, int n) {
        k_u8_to_pyr0<<<grid1d((long long)H * W, n), 256, 0, s>>>(frames + y0 * 3LL * H * W, pyr + y0 * pyr_stride, H * W,
                                                              pyr_stride);
    });
}

cudaError_t launch_box(float4* pyr, int Bn, long long pyr_stride, Lvl prev, Lvl cur, cudaStream_t s)
{
    return for_y_chunks(Bn, [&](long long y0, int n) {
        k_box<<<grid1d((long long)cur.h * cur.w, n), 256, 0, s>>>(pyr + y0 * pyr_stride, pyr_stride, prev, cur);
    });
}

cudaError_t launch_pack_src(const PackSrc* jobs, int n, int fmt, PLvl L, cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    const int copies = fmt == SF8 ? kSF8Copies : (fmt == SF10 ? 2 : 1);
    return for_y_chunks(n, [&](long long y0, int m) {
        k_pack_src<<<grid1d((long long)L.rows * L.pitch * copies, m), 256, 0, s>>>(jobs + y0, fmt, L);
    });
}

cudaError_t launch_pack_tgt_guide(const DTask* tasks, int T, Lvl L, PLvl P, int tfmt, cudaStream_t s)
{
    return for_y_chunks(T, [&](long long y0, int n) {
        k_pack_tgt_guide<<<grid1d((long long)P.rows * P.pitch, n), 256, 0, s>>>(tasks + y0, L, P, tfmt);
    });
}

cudaError_t launch_init(const DTask* tasks, int T, int2* F, long long fstride, Lvl L, int identity, Rng rng,
                        uint32_t level, cudaStream_t s)
{
    return for_y_chunks(T, [&](long long y0, int n) {
        k_init<<<grid1d((long long)L.h * L.w, n), 256, 0, s>>>(tasks + y0, F + y0 * fstride, fstride, L, identity, rng,
                                                            level);
    });
}

cudaError_t launch_upsample(const int2* Fc, int2* Ff, int T, long long fstride, Lvl Lc, Lvl Lf, cudaStream_t s)
{
    return for_y_chunks(T, [&](long long y0, int n) {
        k_upsample<<<grid1d((long long)Lf.h * Lf.w, n), 256, 0, s>>>(Fc + y0 * fstride, Ff + y0 * fstride, fstride, Lc, Lf);
    });
}

#define FB_DISPATCH_P(p, CALL) \
    switch (p) {               \
    case 1: { constexpr int PP = 1; CALL; } break; \
    case 2: { constexpr int PP = 2; CALL; } break; \
    case 3: { constexpr int PP = 3; CALL; } break; \
    case 4: { constexpr int PP = 4; CALL; } break; \
    default: return cudaErrorInvalidValue;          \
    }

// Shared-memory carve-out of the gather kernels: the smallest that still holds the occupancy the registers
// allow (cudaOccupancyMaxActiveBlocksPerMultiprocessor) x (static shared memory + the 1 KB the driver reserves per
// CTA), so the rest of the SM's 256 KB stays L1 cache for the patch gathers.  The driver's default picks a larger
// carve-out (132 KB for the fused level-0 kernel, which needs 58): N=48 field123.L0 302 -> 299.5 ms; the maximum
// carve-out (100 %) costs 11 %.  Set once per kernel; -DFB_CARVEOUT=<percent> forces one value (A/B builds).
#ifndef FB_CARVEOUT
#define FB_CARVEOUT -2  // -2: computed per kernel, -1: driver default
#endif
static void carve(const void* fn, int threads)
{
#if FB_CARVEOUT == -1
    (void)fn; (void)threads;
#else
    static std::mutex mu;
    static std::unordered_map<const void*, int> done;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count(fn)) return;
    int pct = FB_CARVEOUT;
    if (pct < 0) {
        cudaFuncAttributes fa{};
        int dev = 0, smem_max = 0, n = 0;
        if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess || cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, 0) != cudaSuccess || smem_max <= 0) {
            (void)cudaGetLastError();
            done[fn] = -1;
            return;
        }
        const long long need = (long long)n * ((long long)fa.sharedSizeBytes + 1024);
        pct = (int)std::min<long long>(100, (need * 100 + smem_max - 1) / smem_max);
    }
    (void)cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    (void)cudaGetLastError();
    done[fn] = pct;
#endif
}

cudaError_t launch_patch_sums(const SumJob* jobs, int n, int fmt, PLvl L, int p, cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    if (fmt != SF8 && fmt != SF10 && fmt != SF16 && fmt != SF8F) return cudaErrorInvalidValue;
    cudaError_t e = cudaSuccess;
    FB_DISPATCH_P(p, (e = for_y_chunks(n, [&](long long y0, int m) {
        k_patch_sums<PP><<<grid1d((long long)L.h * L.w, m), 256, 0, s>>>(jobs + y0, fmt, L, tail_row0(p));
    })));
    return e;
}
int tail_row0(int p) { return PDE_I13_S1(p); }

template <int P>
static cudaError_t launch_aux_remap_t(const DTask* tasks, int T, const int2* F, long long fstride, Lvl L, PLvl PL,
                                      int tfmt, int sfmt, long long src_off, cudaStream_t s)
{
    return for_y_chunks(T, [&](long long y0, int n) {
        const dim3 g = grid1d((long long)PL.rows * PL.pitch, n);
        const DTask* tk = tasks + y0;
        const int2* Fy = F + y0 * fstride;
        if (sfmt == SF8) { carve((const void*)k_aux_remap<P, SF8>, (int)(256)); k_aux_remap<P, SF8><<<g, 256, 0, s>>>(tk, Fy, fstride, L, PL, tfmt, src_off); }
        else if (sfmt == SF10) { carve((const void*)k_aux_remap<P, SF10>, (int)(256)); k_aux_remap<P, SF10><<<g, 256, 0, s>>>(tk, Fy, fstride, L, PL, tfmt, src_off); }
        else if (sfmt == SF16) { carve((const void*)k_aux_remap<P, SF16>, (int)(256)); k_aux_remap<P, SF16><<<g, 256, 0, s>>>(tk, Fy, fstride, L, PL, tfmt, src_off); }
        else { carve((const void*)k_aux_remap<P, -1>, (int)(256)); k_aux_remap<P, -1><<<g, 256, 0, s>>>(tk, Fy, fstride, L, PL, tfmt, src_off); }
    });
}

cudaError_t launch_aux_remap(const DTask* tasks, int T, const int2* F, long long fstride, Lvl L, PLvl PL, int p,
                             int tfmt, int sfmt, long long src_off, cudaStream_t s)
{
    cudaError_t e = cudaSuccess;
    FB_DISPATCH_P(p, (e = launch_aux_remap_t<PP>(tasks, T, F, fstride, L, PL, tfmt, sfmt, src_off, s)));
    return e;
}

template <int P>
static cudaError_t launch_combine_t(const DOut* outs, int n_outs, const DMember* mem, const int2* F, long long fstride,
                                    int h, int w, int fmt, PLvl PL, cudaStream_t s)
{
    return for_y_chunks(n_outs, [&](long long y0, int n) {  // member task indices stay absolute (F is not offset)
        const dim3 g = grid1d(fmt >= 2 ? (long long)PL.rows * PL.pitch : (long long)h * w, n);
        const DOut* o = outs + y0;
        switch (fmt) {
        case 0: { carve((const void*)k_combine<P, 0>, (int)(256)); k_combine<P, 0><<<g, 256, 0, s>>>(o, mem, F, fstride, h, w, PL); } break;
        case 1: { carve((const void*)k_combine<P, 1>, (int)(256)); k_combine<P, 1><<<g, 256, 0, s>>>(o, mem, F, fstride, h, w, PL); } break;
        case 2: { carve((const void*)k_combine<P, 2>, (int)(256)); k_combine<P, 2><<<g, 256, 0, s>>>(o, mem, F, fstride, h, w, PL); } break;
        case 4: { carve((const void*)k_combine<P, 4>, (int)(256)); k_combine<P, 4><<<g, 256, 0, s>>>(o, mem, F, fstride, h, w, PL); } break;
        default: { carve((const void*)k_combine<P, 3>, (int)(256)); k_combine<P, 3><<<g, 256, 0, s>>>(o, mem, F, fstride, h, w, PL); } break;
        }
    });
}

cudaError_t launch_combine(const DOut* outs, int n_outs, const DMember* mem, const int2* F, long long fstride,
                           int h, int w, int p, int fmt, PLvl PL, cudaStream_t s)
{
    if (n_outs <= 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    FB_DISPATCH_P(p, (e = launch_combine_t<PP>(outs, n_outs, mem, F, fstride, h, w, fmt, PL, s)));
    return e;
}

cudaError_t launch_remap_f3(const float* src, const int2* F, float* out, int Bn, int H, int W, int p,
                            cudaStream_t s)
{
    const long long n = (long long)H * W;
    cudaError_t e = cudaSuccess;
    FB_DISPATCH_P(p, (e = for_y_chunks(Bn, [&](long long y0, int m) {
        k_remap_f3<PP><<<grid1d(n, m), 256, 0, s>>>(src + 3 * y0 * n, F + y0 * n, out + 3 * y0 * n, H, W);
    })));
    return e;
}

template <int P, bool TWO, int SFMT, bool PW = false>
static void launch_field_gen(const FieldArgs& a, int T, int phase, cudaStream_t s)
{
    const dim3 grid((unsigned)((long long)T * a.tiles_per_task)), block(TILE_X * TILE_Y);
    switch (phase) {
    case 0: { carve((const void*)k_field_gen<P, TWO, 0, SFMT, PW>, (int)(block.x * block.y * block.z)); k_field_gen<P, TWO, 0, SFMT, PW><<<grid, block, 0, s>>>(a); } break;
    case 1: { carve((const void*)k_field_gen<P, TWO, 1, SFMT, PW>, (int)(block.x * block.y * block.z)); k_field_gen<P, TWO, 1, SFMT, PW><<<grid, block, 0, s>>>(a); } break;
    case 2: { carve((const void*)k_field_gen<P, TWO, 2, SFMT, PW>, (int)(block.x * block.y * block.z)); k_field_gen<P, TWO, 2, SFMT, PW><<<grid, block, 0, s>>>(a); } break;
    default: { carve((const void*)k_field_gen<P, TWO, 3, SFMT, PW>, (int)(block.x * block.y * block.z)); k_field_gen<P, TWO, 3, SFMT, PW><<<grid, block, 0, s>>>(a); } break;
    }
}

template <int P, bool TWO, bool PW = false, int SFL = 0>
static void launch_field_fast(const FieldArgs& a, int T, int phase, cudaStream_t s)
{
    const dim3 grid((unsigned)((long long)T * a.tiles_per_task)), block(TILE_X * FAST_TY);
    switch (phase) {
    case 0: { carve((const void*)k_field_fast<P, TWO, 0, PW, SFL>, (int)(block.x * block.y * block.z)); k_field_fast<P, TWO, 0, PW, SFL><<<grid, block, 0, s>>>(a); } break;
    case 1: { carve((const void*)k_field_fast<P, TWO, 1, PW, SFL>, (int)(block.x * block.y * block.z)); k_field_fast<P, TWO, 1, PW, SFL><<<grid, block, 0, s>>>(a); } break;
    case 2: { carve((const void*)k_field_fast<P, TWO, 2, PW, SFL>, (int)(block.x * block.y * block.z)); k_field_fast<P, TWO, 2, PW, SFL><<<grid, block, 0, s>>>(a); } break;
    default: { carve((const void*)k_field_fast<P, TWO, 3, PW, SFL>, (int)(block.x * block.y * block.z)); k_field_fast<P, TWO, 3, PW, SFL><<<grid, block, 0, s>>>(a); } break;
    }
}

cudaError_t launch_iter_fast(const FieldArgs& a0, int T, int p, int loss, cudaStream_t s)
{
    FieldArgs a = a0;
    a.tiles_x = (a.L.w + IT_TX - 1) / IT_TX;
    a.tiles_per_task = a.tiles_x * ((a.L.h + IT_TY - 1) / IT_TY);
    const dim3 grid((unsigned)((long long)T * a.tiles_per_task)), block(32 * (IT_TY + 1));
    if (p == 1) { if (loss) k_iter_fast<1, true><<<grid, block, 0, s>>>(a); else k_iter_fast<1, false><<<grid, block, 0, s>>>(a); }
    else if (p == 2) { if (loss) k_iter_fast<2, true><<<grid, block, 0, s>>>(a); else k_iter_fast<2, false><<<grid, block, 0, s>>>(a); }
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

cudaError_t launch_iter13_fast(const FieldArgs& a0, int T, int p, int loss, cudaStream_t s)
{
    FieldArgs a = a0;
    a.tiles_x = (a.L.w + IT_TX - 1) / IT_TX;
    a.tiles_per_task = a.tiles_x * ((a.L.h + I13_TY - 1) / I13_TY);
    const dim3 grid((unsigned)((long long)T * a.tiles_per_task)), block(32 * I13_TY);
    const int hy = a.tgt_reg_rows;  // hybrid target (rows in registers: 1, 2; 3 = none; 0 = all)
    if (a.src_fmt == SF10) {  // level 1: SF10 source + TF10 target (GUIDE_STYLE / MEAN_ALIGN, p = 2)
        if (p != 2 || (loss != 1 && loss != 2)) return cudaErrorInvalidValue;
        if (hy == 3) { carve((const void*)k_iter13_fast<2, true, false, 0, 0, 1>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, true, false, 0, 0, 1><<<grid, block, 0, s>>>(a); }
        else if (hy == 1) { carve((const void*)k_iter13_fast<2, true, false, 0, 1, 1>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, true, false, 0, 1, 1><<<grid, block, 0, s>>>(a); }
        else { carve((const void*)k_iter13_fast<2, true, false, 0, 2, 1>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, true, false, 0, 2, 1><<<grid, block, 0, s>>>(a); }
        return cudaGetLastError();
    }
    if (a.src_fmt == SF8F) {
        if (loss != 1 && loss != 2) return cudaErrorInvalidValue;
        if (p == 1) { carve((const void*)k_iter13_fast<1, true, false, 1>, (int)(block.x * block.y * block.z)); k_iter13_fast<1, true, false, 1><<<grid, block, 0, s>>>(a); }
        else if (p == 2 && hy == 3) { carve((const void*)k_iter13_fast<2, true, false, 1, 0>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, true, false, 1, 0><<<grid, block, 0, s>>>(a); }
        else if (p == 2 && hy == 1) { carve((const void*)k_iter13_fast<2, true, false, 1, 1>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, true, false, 1, 1><<<grid, block, 0, s>>>(a); }
        else if (p == 2 && hy == 2) { carve((const void*)k_iter13_fast<2, true, false, 1, 2>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, true, false, 1, 2><<<grid, block, 0, s>>>(a); }
        else if (p == 2) { carve((const void*)k_iter13_fast<2, true, false, 1>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, true, false, 1><<<grid, block, 0, s>>>(a); }
        else return cudaErrorInvalidValue;
        return cudaGetLastError();
    }
    if (p == 1 && loss != 3 && hy == 3) {  // p = 1: every target row from the shared tile (patch-sum bound on)
        if (loss) { carve((const void*)k_iter13_fast<1, true, false, 0, 0>, (int)(block.x * block.y * block.z)); k_iter13_fast<1, true, false, 0, 0><<<grid, block, 0, s>>>(a); }
        else { carve((const void*)k_iter13_fast<1, false, false, 0, 0>, (int)(block.x * block.y * block.z)); k_iter13_fast<1, false, false, 0, 0><<<grid, block, 0, s>>>(a); }
        return cudaGetLastError();
    }
    if (p == 3 && loss != 3) {  // level 0 at p = 3 (config 5): every target row from the shared tile
        if (loss) { carve((const void*)k_iter13_fast<3, true, false, 0, 0>, (int)(block.x * block.y * block.z)); k_iter13_fast<3, true, false, 0, 0><<<grid, block, 0, s>>>(a); }
        else { carve((const void*)k_iter13_fast<3, false, false, 0, 0>, (int)(block.x * block.y * block.z)); k_iter13_fast<3, false, false, 0, 0><<<grid, block, 0, s>>>(a); }
        return cudaGetLastError();
    }
    if (p == 2 && loss != 3 && hy >= 1) {
        if (loss && hy == 3 && a.tail_off >= 0) { carve((const void*)k_iter13_fast<2, true, false, 0, 0, 0, true>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, true, false, 0, 0, 0, true><<<grid, block, 0, s>>>(a); }
        else if (loss && hy == 3) { carve((const void*)k_iter13_fast<2, true, false, 0, 0>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, true, false, 0, 0><<<grid, block, 0, s>>>(a); }
        else if (loss && hy == 1) { carve((const void*)k_iter13_fast<2, true, false, 0, 1>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, true, false, 0, 1><<<grid, block, 0, s>>>(a); }
        else if (loss) { carve((const void*)k_iter13_fast<2, true, false, 0, 2>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, true, false, 0, 2><<<grid, block, 0, s>>>(a); }
        else if (hy == 1) { carve((const void*)k_iter13_fast<2, false, false, 0, 1>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, false, false, 0, 1><<<grid, block, 0, s>>>(a); }
        else { carve((const void*)k_iter13_fast<2, false, false, 0, 2>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, false, false, 0, 2><<<grid, block, 0, s>>>(a); }
        return cudaGetLastError();
    }
    if (p == 1) {
        if (loss == 3) { carve((const void*)k_iter13_fast<1, true, true>, (int)(block.x * block.y * block.z)); k_iter13_fast<1, true, true><<<grid, block, 0, s>>>(a); }
        else if (loss) { carve((const void*)k_iter13_fast<1, true>, (int)(block.x * block.y * block.z)); k_iter13_fast<1, true><<<grid, block, 0, s>>>(a); }
        else { carve((const void*)k_iter13_fast<1, false>, (int)(block.x * block.y * block.z)); k_iter13_fast<1, false><<<grid, block, 0, s>>>(a); }
    } else if (p == 2) {
        if (loss == 3) { carve((const void*)k_iter13_fast<2, true, true>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, true, true><<<grid, block, 0, s>>>(a); }
        else if (loss) { carve((const void*)k_iter13_fast<2, true>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, true><<<grid, block, 0, s>>>(a); }
        else { carve((const void*)k_iter13_fast<2, false>, (int)(block.x * block.y * block.z)); k_iter13_fast<2, false><<<grid, block, 0, s>>>(a); }
    } else {
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <int P, bool TWO, int SFL = 0, int SF = 0>
static void launch_field_mid(const FieldArgs& a, int T, int phase, cudaStream_t s, bool pair0 = false)
{
    const dim3 grid((unsigned)((long long)T * a.tiles_per_task)), block(TILE_X * TILE_Y);
    switch (phase) {
    case 0:
        if constexpr (SF == 0 && SFL == 0) {
            if (pair0 && a.einit) { { carve((const void*)k_field_mid<P, TWO, 0, SFL, SF, true>, (int)(block.x * block.y * block.z)); k_field_mid<P, TWO, 0, SFL, SF, true><<<grid, block, 0, s>>>(a); } break; }
        }
        { carve((const void*)k_field_mid<P, TWO, 0, SFL, SF>, (int)(block.x * block.y * block.z)); k_field_mid<P, TWO, 0, SFL, SF><<<grid, block, 0, s>>>(a); }
        break;
    case 1: { carve((const void*)k_field_mid<P, TWO, 1, SFL, SF>, (int)(block.x * block.y * block.z)); k_field_mid<P, TWO, 1, SFL, SF><<<grid, block, 0, s>>>(a); } break;
    case 2: { carve((const void*)k_field_mid<P, TWO, 2, SFL, SF>, (int)(block.x * block.y * block.z)); k_field_mid<P, TWO, 2, SFL, SF><<<grid, block, 0, s>>>(a); } break;
    default: { carve((const void*)k_field_mid<P, TWO, 3, SFL, SF>, (int)(block.x * block.y * block.z)); k_field_mid<P, TWO, 3, SFL, SF><<<grid, block, 0, s>>>(a); } break;
    }
}

cudaError_t launch_field(const FieldArgs& a0, int T, int p, int loss, int phase, int kind, cudaStream_t s)
{
    const bool fast = kind == 1;
    FieldArgs a = a0;
    a.tiles_x = (a.L.w + TILE_X - 1) / TILE_X;
    a.tiles_per_task = a.tiles_x * ((a.L.h + (fast ? FAST_TY : TILE_Y) - 1) / (fast ? FAST_TY : TILE_Y));
    const bool pw = loss == 3;
    a.pair0 = loss == 2 && kind == 0 && phase == 0;  // accurate mode: paired E init + field 0 in the general kernel
    if (kind == 2) {  // level 0: SF8 (or, p = 2, SF8F) source, TF16 target tile; level 1: SF10 + TF10 (p = 2)
        if (pw) return cudaErrorInvalidValue;
        if (a.src_fmt == SF10) {
            if (p != 2 || !loss) return cudaErrorInvalidValue;
            launch_field_mid<2, true, 0, 1>(a, T, phase, s);
            return cudaGetLastError();
        }
        if (a.src_fmt == SF8F) {
            if (p != 2 || !loss) return cudaErrorInvalidValue;
            launch_field_mid<2, true, 1>(a, T, phase, s);
            return cudaGetLastError();
        }
        if (a.src_fmt != SF8) return cudaErrorInvalidValue;
        const bool pr = loss == 2;  // MEAN_ALIGN: paired phase 0
        if (p == 2) { if (loss) launch_field_mid<2, true>(a, T, phase, s, pr); else launch_field_mid<2, false>(a, T, phase, s); }
        else if (p == 3) { if (loss) launch_field_mid<3, true>(a, T, phase, s, pr); else launch_field_mid<3, false>(a, T, phase, s); }
        else if (p == 4) { if (loss) launch_field_mid<4, true>(a, T, phase, s, pr); else launch_field_mid<4, false>(a, T, phase, s); }
        else return cudaErrorInvalidValue;
        return cudaGetLastError();
    }
    if (fast && a.src_fmt == SF8F) {  // float-style level-0 sources (tree queries): GUIDE_STYLE only
        if (pw || !loss) return cudaErrorInvalidValue;
        if (p == 1) launch_field_fast<1, true, false, 1>(a, T, phase, s);
        else if (p == 2) launch_field_fast<2, true, false, 1>(a, T, phase, s);
        else return cudaErrorInvalidValue;
    } else if (fast) {
        if (p == 1) {
            if (pw) launch_field_fast<1, true, true>(a, T, phase, s);
            else if (loss) launch_field_fast<1, true>(a, T, phase, s);
            else launch_field_fast<1, false>(a, T, phase, s);
        } else if (p == 2) {
            if (pw) launch_field_fast<2, true, true>(a, T, phase, s);
            else if (loss) launch_field_fast<2, true>(a, T, phase, s);
            else launch_field_fast<2, false>(a, T, phase, s);
        } else {
            return cudaErrorInvalidValue;
        }
    } else if (a.src_fmt == SF10) {
        if (pw) {
            if (p == 1) launch_field_gen<1, true, SF10, true>(a, T, phase, s);
            else if (p == 2) launch_field_gen<2, true, SF10, true>(a, T, phase, s);
            else return cudaErrorInvalidValue;
        } else if (loss) {
            FB_DISPATCH_P(p, (launch_field_gen<PP, true, SF10>(a, T, phase, s)));
        } else {
            FB_DISPATCH_P(p, (launch_field_gen<PP, false, SF10>(a, T, phase, s)));
        }
    } else if (a.src_fmt == SF16) {
        if (pw) {
            if (p == 1) launch_field_gen<1, true, SF16, true>(a, T, phase, s);
            else if (p == 2) launch_field_gen<2, true, SF16, true>(a, T, phase, s);
            else return cudaErrorInvalidValue;
        } else if (loss) {
            FB_DISPATCH_P(p, (launch_field_gen<PP, true, SF16>(a, T, phase, s)));
        } else {
            FB_DISPATCH_P(p, (launch_field_gen<PP, false, SF16>(a, T, phase, s)));
        }
    } else if (pw) {
        FB_DISPATCH_P(p, (launch_field_gen<PP, true, SF32, true>(a, T, phase, s)));
    } else if (loss == 0) {
        FB_DISPATCH_P(p, (launch_field_gen<PP, false, SF32>(a, T, phase, s)));
    } else {
        FB_DISPATCH_P(p, (launch_field_gen<PP, true, SF32>(a, T, phase, s)));
    }
    return cudaGetLastError();
}

}  // namespace fbk

#ifdef FB_COUNTERS
extern "C" int fb_debug_counters(unsigned long long* out, int reset)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, fbk::g_fb_cnt, sizeof(unsigned long long) * 32);
    if (reset) {
        unsigned long long z[32] = {};
        cudaMemcpyToSymbol(fbk::g_fb_cnt, z, sizeof z);
    }
    return 0;
}
#endif
