// kernels.cu — sm_100a kernels of the FastBlend hot path (arXiv 2311.09265).
//
// No tensor cores: the method has no dense contraction (patch distances are gathers of data-dependent
// patches).  The bound resources are the L1/LSU gather path and the FP32 pipe.
//
// Every floating-point operation that decides a result is written with an explicit IEEE intrinsic
// (__fadd_rn, __fsub_rn, __fmaf_rn, __fdiv_rn) in the order DESIGN.md §3 fixes (D20), so the kernels
// are bit-identical to the contract regardless of scheduling or thread mapping.
#include "kernels.h"

namespace fbk {

static constexpr int TILE_X = 32, TILE_Y = 8;  // 256-thread 2D tiles: a warp is one row segment

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

template <int P>
__global__ void k_aux_remap(const DTask* __restrict__ tasks, const int2* __restrict__ F, long long fstride, Lvl L)
{
    const int t = blockIdx.y;
    const int n = L.h * L.w;
    const DTask T = tasks[t];
    const float4* S = T.ss + L.off;
    const int2* Ft = F + t * fstride;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = i / L.w, c = i - r * L.w;
        const float3 v = remap_px<P>(S, Ft, L.h, L.w, r, c);
        T.aux[i] = make_float4(v.x, v.y, v.z, 0.0f);
    }
}

template <int P>
__global__ void k_combine(const DOut* __restrict__ outs, const DMember* __restrict__ mem, const int2* __restrict__ F,
                          long long fstride, int h, int w)
{
    const DOut o = outs[blockIdx.y];
    const int n = h * w;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = i / w, c = i - r * w;
        float ax = 0.0f, ay = 0.0f, az = 0.0f;
        for (int m = 0; m < o.nm; ++m) {
            const DMember mb = mem[o.m0 + m];
            float3 y;
            if (mb.task < 0) {
                const float4 v = __ldg(&mb.img[i]);
                y = make_float3(v.x, v.y, v.z);
            } else {
                y = remap_px<P>(mb.img, F + mb.task * fstride, h, w, r, c);
            }
            ax = __fmaf_rn(mb.w, y.x, ax);
            ay = __fmaf_rn(mb.w, y.y, ay);
            az = __fmaf_rn(mb.w, y.z, az);
        }
        ax = __fdiv_rn(ax, o.div);
        ay = __fdiv_rn(ay, o.div);
        az = __fdiv_rn(az, o.div);
        if (o.fmt == 0) {
            static_cast<float4*>(o.out)[i] = make_float4(ax, ay, az, 0.0f);
        } else {
            float* d = static_cast<float*>(o.out) + 3LL * i;
            d[0] = ax; d[1] = ay; d[2] = az;
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

__global__ void k_f4_to_f3(const float4* __restrict__ in, long long in_stride, float* __restrict__ out, int npx)
{
    const int b = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npx; i += gridDim.x * blockDim.x) {
        const float4 v = in[(long long)b * in_stride + i];
        float* d = out + 3LL * ((long long)b * npx + i);
        d[0] = v.x; d[1] = v.y; d[2] = v.z;
    }
}

// ------------------------------------------------------------------------------------ patch loss
// D(A,(sr,sc),B,(r,c)) = sum_dr ( rho_dr ), rho_dr = fma chain over dc then channel of (B - A)^2, zero
// outside the image (Eq. 1, D9, D20).  GS = two-term loss fma(alpha, D_guide, D_style) (Eq. 3 / Eq. 8).
template <int P, bool GS>
__device__ __forceinline__ float patch_loss(const float4* __restrict__ sg, const float4* __restrict__ ss,
                                            const float4* __restrict__ tg, const float4* __restrict__ ax, int h,
                                            int w, int r, int c, int sr, int sc, float alpha)
{
    float dg = 0.0f, ds = 0.0f;
    const float4 z = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
    for (int dr = -P; dr <= P; ++dr) {
        const int tr = r + dr, ur = sr + dr;
        const bool tin_r = (unsigned)tr < (unsigned)h, sin_r = (unsigned)ur < (unsigned)h;
        float rg = 0.0f, rs = 0.0f;
#pragma unroll
        for (int dc = -P; dc <= P; ++dc) {
            const int tc = c + dc, uc = sc + dc;
            const bool tin = tin_r && (unsigned)tc < (unsigned)w;
            const bool sin = sin_r && (unsigned)uc < (unsigned)w;
            const int ti = tr * w + tc, si = ur * w + uc;
            const float4 b = tin ? __ldg(&tg[ti]) : z;
            const float4 a = sin ? __ldg(&sg[si]) : z;
            float d;
            d = __fsub_rn(b.x, a.x); rg = __fmaf_rn(d, d, rg);
            d = __fsub_rn(b.y, a.y); rg = __fmaf_rn(d, d, rg);
            d = __fsub_rn(b.z, a.z); rg = __fmaf_rn(d, d, rg);
            if (GS) {
                const float4 bb = tin ? __ldg(&ax[ti]) : z;
                const float4 aa = sin ? __ldg(&ss[si]) : z;
                d = __fsub_rn(bb.x, aa.x); rs = __fmaf_rn(d, d, rs);
                d = __fsub_rn(bb.y, aa.y); rs = __fmaf_rn(d, d, rs);
                d = __fsub_rn(bb.z, aa.z); rs = __fmaf_rn(d, d, rs);
            }
        }
        dg = __fadd_rn(dg, rg);
        if (GS) ds = __fadd_rn(ds, rs);
    }
    return GS ? __fmaf_rn(alpha, dg, ds) : dg;
}

// One element of Alg. 1's updating sequence per launch, Jacobi over pixels:
//   PHASE 0: E <- L(F), then propagation (-1,0); 1: (+1,0); 2: (0,-1);
//   PHASE 3: propagation (0,+1), then the K random-search fields, pointwise in registers.
// Each candidate F' = clamp(.) is kept iff L(F') < E (strict, D16).
template <int P, bool GS, int PHASE>
__global__ void __launch_bounds__(TILE_X* TILE_Y) k_field(FieldArgs a)
{
    const int t = blockIdx.x / a.tiles_per_task;
    const int tile = blockIdx.x - t * a.tiles_per_task;
    const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
    const int c = tx * TILE_X + (threadIdx.x & (TILE_X - 1));
    const int r = ty * TILE_Y + (threadIdx.x / TILE_X);
    const int h = a.L.h, w = a.L.w;
    if (r >= h || c >= w) return;
    const DTask T = a.tasks[t];
    const float4* sg = T.sg + a.L.off;
    const float4* tg = T.tg + a.L.off;
    const float4* ss = GS ? T.ss + a.L.off : nullptr;
    const float4* ax = GS ? T.aux : nullptr;
    const int2* Fi = a.Fin + t * a.fstride;
    const int i = r * w + c;
    int2 f = Fi[i];
    float e;
    if (PHASE == 0) e = patch_loss<P, GS>(sg, ss, tg, ax, h, w, r, c, f.x, f.y, a.alpha);
    else e = a.E[t * a.fstride + i];
    {
        constexpr int dx = PHASE == 0 ? -1 : (PHASE == 1 ? 1 : 0);
        constexpr int dy = PHASE == 2 ? -1 : (PHASE == 3 ? 1 : 0);
        const int nr = clampi(r + dx, 0, h - 1), nc = clampi(c + dy, 0, w - 1);  // D11
        const int2 fn = Fi[nr * w + nc];
        const int sr = clampi(fn.x - dx, 0, h - 1), sc = clampi(fn.y - dy, 0, w - 1);  // D10
        const float e2 = patch_loss<P, GS>(sg, ss, tg, ax, h, w, r, c, sr, sc, a.alpha);
        if (e2 < e) { f = make_int2(sr, sc); e = e2; }
    }
    if (PHASE == 3) {
        for (int s = 0; s < a.rs_k; ++s) {
            const int R = max(a.rs_r0 >> s, 1);
            const uint4 u = philox4x32_10(
                make_uint4((uint32_t)i, (1u << 28) | (a.level << 22) | (a.iter << 12) | (uint32_t)s, T.c2, T.c3),
                a.rng.k0, a.rng.k1);
            const uint32_t span = 2u * (uint32_t)R + 1u;
            const int ox = (int)__umulhi(u.x, span) - R, oy = (int)__umulhi(u.y, span) - R;
            const int sr = clampi(f.x + ox, 0, h - 1), sc = clampi(f.y + oy, 0, w - 1);
            const float e2 = patch_loss<P, GS>(sg, ss, tg, ax, h, w, r, c, sr, sc, a.alpha);
            if (e2 < e) { f = make_int2(sr, sc); e = e2; }
        }
    }
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

cudaError_t launch_u8_to_pyr0(const uint8_t* frames, float4* pyr, int B, int H, int W, long long pyr_stride,
                              cudaStream_t s)
{
    k_u8_to_pyr0<<<grid1d((long long)H * W, B), 256, 0, s>>>(frames, pyr, H * W, pyr_stride);
    return cudaGetLastError();
}

cudaError_t launch_box(float4* pyr, int B, long long pyr_stride, Lvl prev, Lvl cur, cudaStream_t s)
{
    k_box<<<grid1d((long long)cur.h * cur.w, B), 256, 0, s>>>(pyr, pyr_stride, prev, cur);
    return cudaGetLastError();
}

cudaError_t launch_init(const DTask* tasks, int T, int2* F, long long fstride, Lvl L, int identity, Rng rng,
                        uint32_t level, cudaStream_t s)
{
    k_init<<<grid1d((long long)L.h * L.w, T), 256, 0, s>>>(tasks, F, fstride, L, identity, rng, level);
    return cudaGetLastError();
}

cudaError_t launch_upsample(const int2* Fc, int2* Ff, int T, long long fstride, Lvl Lc, Lvl Lf, cudaStream_t s)
{
    k_upsample<<<grid1d((long long)Lf.h * Lf.w, T), 256, 0, s>>>(Fc, Ff, fstride, Lc, Lf);
    return cudaGetLastError();
}

#define FB_DISPATCH_P(p, CALL) \
    switch (p) {               \
    case 1: { constexpr int PP = 1; CALL; } break; \
    case 2: { constexpr int PP = 2; CALL; } break; \
    case 3: { constexpr int PP = 3; CALL; } break; \
    case 4: { constexpr int PP = 4; CALL; } break; \
    default: return cudaErrorInvalidValue;          \
    }

cudaError_t launch_aux_remap(const DTask* tasks, int T, const int2* F, long long fstride, Lvl L, int p,
                             cudaStream_t s)
{
    FB_DISPATCH_P(p, (k_aux_remap<PP><<<grid1d((long long)L.h * L.w, T), 256, 0, s>>>(tasks, F, fstride, L)));
    return cudaGetLastError();
}

cudaError_t launch_combine(const DOut* outs, int n_outs, const DMember* mem, const int2* F, long long fstride,
                           int h, int w, int p, cudaStream_t s)
{
    if (n_outs <= 0) return cudaSuccess;
    FB_DISPATCH_P(p, (k_combine<PP><<<grid1d((long long)h * w, n_outs), 256, 0, s>>>(outs, mem, F, fstride, h, w)));
    return cudaGetLastError();
}

cudaError_t launch_remap_f3(const float* src, const int2* F, float* out, int B, int H, int W, int p,
                            cudaStream_t s)
{
    FB_DISPATCH_P(p, (k_remap_f3<PP><<<grid1d((long long)H * W, B), 256, 0, s>>>(src, F, out, H, W)));
    return cudaGetLastError();
}

cudaError_t launch_f4_to_f3(const float4* in, long long in_stride, float* out, int B, int npx, cudaStream_t s)
{
    k_f4_to_f3<<<grid1d(npx, B), 256, 0, s>>>(in, in_stride, out, npx);
    return cudaGetLastError();
}

template <int P, bool GS>
static void launch_field_t(const FieldArgs& a, int T, int phase, cudaStream_t s)
{
    const dim3 grid((unsigned)((long long)T * a.tiles_per_task)), block(TILE_X * TILE_Y);
    switch (phase) {
    case 0: k_field<P, GS, 0><<<grid, block, 0, s>>>(a); break;
    case 1: k_field<P, GS, 1><<<grid, block, 0, s>>>(a); break;
    case 2: k_field<P, GS, 2><<<grid, block, 0, s>>>(a); break;
    default: k_field<P, GS, 3><<<grid, block, 0, s>>>(a); break;
    }
}

cudaError_t launch_field(const FieldArgs& a0, int T, int p, int loss, int phase, cudaStream_t s)
{
    FieldArgs a = a0;
    a.tiles_x = (a.L.w + TILE_X - 1) / TILE_X;
    a.tiles_per_task = a.tiles_x * ((a.L.h + TILE_Y - 1) / TILE_Y);
    if (loss == 0) {
        FB_DISPATCH_P(p, (launch_field_t<PP, false>(a, T, phase, s)));
    } else {
        FB_DISPATCH_P(p, (launch_field_t<PP, true>(a, T, phase, s)));
    }
    return cudaGetLastError();
}

}  // namespace fbk
