// engine.cu — host side of the B200 FastBlend path: C ABI (include/fb.h), workspace arena, the
// Alg. 1 batch driver and the three schedules (direct window blend, tree window blend, keyframe
// interpolation).  All arithmetic runs in kernels.cu; this file only plans and enqueues.
//
// Execution model: one context = one device + one stream.  Every call first plans in "dry" mode
// (same code path, no launches) to size the workspace, then runs for real.  All NNF tasks of a batch
// advance in lockstep (level, iteration, field), which is what MEAN_ALIGN's shared T-bar needs
// (Eq. 7) and what fills the 148 SMs: one launch covers every pixel of every pair.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/fb.h"
#include "kernels.h"

using fbk::DMember;
using fbk::DOut;
using fbk::DTask;
using fbk::Lvl;

struct fb_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    char* ws = nullptr;
    size_t ws_bytes = 0;
    int64_t max_pairs = 0;
    uint64_t launches = 0;
    // Kernel-schedule options (fb_set_option; per context, results identical for every setting):
    bool fused = false;  // FB_OPT_FUSED_ITER: a whole level-0 iteration per launch (measured slower)
    bool fuse13 = true;  // FB_OPT_FUSE13: fields 1-3 + random search fused on the fast path
    bool phase0_mid = true;  // FB_OPT_PHASE0_MID: E init + field 0 at level 0 through the shared-memory-target
                             // kernel (0: register target; 44 vs 163 registers: field0.L0 95 -> 76 ms at N=48)
    int tgt_reg_rows = 3;  // FB_OPT_TGT_REG_ROWS: fused fields 1-3 target rows in registers, rest in shared
                           // memory (0 = all in registers, 3 = none).  With the patch-sum bound most random-
                           // search candidates never read a target row, and occupancy wins: N=48 field123.L0
                           // two rows at 5 CTAs/SM 353 ms, one row at 6: 333, none at 8: 324 (accurate);
                           // 285 -> 268 balanced, 112 -> 102 fast
    bool sum_bound = true;  // FB_OPT_SUM_BOUND: random-search candidates rejected by the patch-sum bound (level 0,
                            // and level 1 with FB_OPT_L1_FAST) before any patch row is gathered
    bool p3_fused = true;  // FB_OPT_P3_FUSED: level-0 fields 1-3 + random search in one launch at p = 3 as well
    bool tail_bound = false;  // FB_OPT_TAIL_BOUND: the level-0 fused random search adds the partial + remainder
                              // bound (tail-row sums plane next to the patch sums, p = 2, SF8 sources); its
                              // registers keep the kernel at 8 CTAs/SM, which loses to 10 without it
    int l1_fast = 0;  // FB_OPT_L1_FAST: level 1 of u8 sources (SF10) through 16-byte TF10 targets and the
                      // level-0 kernels -- 1: E init + field 0 by the shared-tile kernel, fields 1-3 + random
                      // search fused; 2: every field by the shared-tile kernel.  Bit-identical; 1 measured slower
                      // (N=48 accurate: field123.L1 146 ms vs 102 for fields 1-3 of the general kernel)
    std::string err;
    // kernel timing (fb_profile_*)
    bool prof = false;
    struct Pending { int cls; cudaEvent_t a, b; uint64_t work; };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> pool;
    std::vector<std::string> cls_names;
    std::vector<fb_profile_entry> totals;
    int cls(const char* name)
    {
        for (size_t i = 0; i < cls_names.size(); ++i)
            if (cls_names[i] == name) return (int)i;
        cls_names.push_back(name);
        fb_profile_entry e{};
        snprintf(e.name, sizeof e.name, "%s", name);
        totals.push_back(e);
        return (int)cls_names.size() - 1;
    }
    cudaEvent_t ev()
    {
        if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    void drain()
    {
        for (auto& p : pending) {
            cudaEventSynchronize(p.b);
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, p.a, p.b);
            totals[p.cls].launches += 1;
            totals[p.cls].ms += ms;
            totals[p.cls].work += p.work;
            pool.push_back(p.a);
            pool.push_back(p.b);
        }
        pending.clear();
    }
    ~fb_ctx_s()
    {
        drain();
        for (auto e : pool) cudaEventDestroy(e);
    }
};

namespace {

constexpr size_t kAutoStateBudget = 64ull << 30;  // bytes of per-pair state in one auto-sized batch
constexpr int kMaxBatchPairs = 65535;              // pairs per batch (field grids T x tiles stay below 2^31)

struct Fail {
    fb_status st;
    std::string msg;
};

// ------------------------------------------------------------------------------------ arena
struct Arena {
    char* base = nullptr;  // nullptr in dry mode: pointers are offsets, never dereferenced
    size_t off = 0, peak = 0;
    template <class T>
    T* take(size_t n)
    {
        off = (off + 255) & ~size_t(255);
        T* p = reinterpret_cast<T*>(base + off);
        off += n * sizeof(T);
        peak = std::max(peak, off);
        return p;
    }
};

// NVTX range for profilers (nsys / ncu --nvtx): schedule phases, pyramid levels and iterations.  The
// calls are no-ops unless a tool is attached; dry (planning) runs emit nothing.
struct Nvtx {
    bool on;
    Nvtx(bool dry, const char* fmt, int a = 0, int b = 0) : on(!dry)
    {
        if (!on) return;
        char buf[64];
        snprintf(buf, sizeof buf, fmt, a, b);
        nvtxRangePushA(buf);
    }
    ~Nvtx() { if (on) nvtxRangePop(); }
};

struct Exec {
    fb_ctx ctx;
    bool dry;
    Arena ar;
    void check(cudaError_t e, const char* what)
    {
        if (e != cudaSuccess) throw Fail{FB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
    }
    template <class F>
    void launch(const char* what, F&& f, uint64_t work = 0)
    {
        if (dry) return;
        if (ctx->prof) {
            fb_ctx_s::Pending p{ctx->cls(what), ctx->ev(), ctx->ev(), work};
            cudaEventRecord(p.a, ctx->stream);
            check(f(), what);
            cudaEventRecord(p.b, ctx->stream);
            ctx->pending.push_back(p);
            if (ctx->pending.size() > 4096) ctx->drain();
        } else {
            check(f(), what);
        }
        ++ctx->launches;
    }
    template <class T>
    T* upload(const std::vector<T>& v)
    {
        T* d = ar.take<T>(std::max<size_t>(v.size(), 1));
        if (!dry && !v.empty())
            check(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream), "upload");
        return d;
    }
    void d2d(void* dst, const void* src, size_t bytes)
    {
        if (!dry && bytes) check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream), "d2d");
    }
};

// ------------------------------------------------------------------------------------ geometry
struct Geo {
    int H = 0, W = 0, Lv = 0, p = 0;
    Lvl L[24];
    fbk::PLvl PL[24];          // padded geometry of the packed PatchMatch operands
    long long pyr_texels = 0;  // texels of one pyramid
    long long npx0() const { return (long long)H * W; }
};

fbk::PLvl padded(int h, int w, int k)
{
    const int pitch = ((w + 2 * fbk::kBorder) + 3) & ~3;  // even (texel pairs are 16-byte aligned)
    return fbk::PLvl{h, w, pitch, h + 2 * fbk::kBorder, k};
}

// Packed source format of level k for a slot whose level-0 format is fmt0 (kernels.h): u8 styles use
// SF8 at level 0, the exact 10-bit form SF10 at level 1 (n = 4v < 2^10, 8 bytes per texel) and the exact
// 16-bit integer form SF16 at levels 2..4 (values n / 4^k, n < 2^16).
int src_fmt(int fmt0, int k)
{
    if (fmt0 == fbk::SF8F) return k == 0 ? fbk::SF8F : fbk::SF32;  // float styles: u8 guide + f32 style
    if (fmt0 != fbk::SF8) return fbk::SF32;
    if (k == 1) return fbk::SF10;
    return k == 0 ? fbk::SF8 : (k <= 4 ? fbk::SF16 : fbk::SF32);
}
size_t src_bytes(int fmt)
{
    return (fmt == fbk::SF8 || fmt == fbk::SF10) ? 8 : (fmt == fbk::SF16 || fmt == fbk::SF8F) ? 16 : 32;
}

int level_count(int H, int W, int p, int requested)  // D6, D32
{
    const int mn = std::min(H, W);
    if (mn < 2 * p + 1) return -1;
    if (requested > 0) {
        if (requested > 20) return -1;
        if (std::min(H >> (requested - 1), W >> (requested - 1)) < 2 * p + 1) return -1;
        return requested;
    }
    int lv = 1;
    for (int k = 1; k < 24; ++k)
        if ((mn >> k) >= 32) lv = k + 1;
    while (lv > 1 && (mn >> (lv - 1)) < 2 * p + 1) --lv;
    return lv;
}

Geo make_geo(const fb_match_cfg& cfg, int H, int W)
{
    Geo g;
    g.H = H; g.W = W; g.p = cfg.patch_radius;
    g.Lv = level_count(H, W, cfg.patch_radius, cfg.levels);
    if (g.Lv < 1) throw Fail{FB_ERR_SHAPE, "min(H,W) or the coarsest level is smaller than the patch (2p+1)"};
    long long off = 0;
    for (int k = 0; k < g.Lv; ++k) {
        g.L[k] = Lvl{H >> k, W >> k, off};
        g.PL[k] = padded(H >> k, W >> k, k);
        off += (long long)(H >> k) * (W >> k);
    }
    g.pyr_texels = off;
    return g;
}

int rs_r0(const fb_match_cfg& c, const Lvl& L) { return c.rs_radius0 > 0 ? c.rs_radius0 : std::max(L.h, L.w); }
int rs_count(const fb_match_cfg& c, const Lvl& L)  // D13, D33
{
    if (c.rs_steps > 0) return c.rs_steps;
    int n = 0, r0 = rs_r0(c, L);
    while ((r0 >> n) >= 1) ++n;
    return n;
}
uint64_t evals_per_pair(const fb_match_cfg& c, const Geo& g)
{
    uint64_t n = 0;
    for (int k = 0; k < g.Lv; ++k)
        n += (uint64_t)g.L[k].h * g.L[k].w * (uint64_t)c.iters_per_level *
             (uint64_t)(1 + 4 * std::max(1, c.prop_scales) + rs_count(c, g.L[k]));
    return n;
}

void validate_cfg(const fb_match_cfg* cfg)
{
    if (!cfg) throw Fail{FB_ERR_INVALID_ARG, "cfg is NULL"};
    if (cfg->patch_radius < 1) throw Fail{FB_ERR_INVALID_ARG, "patch_radius < 1"};
    if (cfg->patch_radius > 4) throw Fail{FB_ERR_UNSUPPORTED, "patch_radius > 4 is not compiled"};
    if (cfg->iters_per_level < 0 || cfg->levels < 0 || cfg->rs_radius0 < 0 || cfg->rs_steps < 0)
        throw Fail{FB_ERR_INVALID_ARG, "negative iteration / level / random-search parameter"};
    // the Philox counter word c1 packs purpose << 28 | level << 22 | iter << 12 | step (D21): wider values
    // would alias draws of different iterations / levels
    if (cfg->iters_per_level > 1023) throw Fail{FB_ERR_INVALID_ARG, "iters_per_level > 1023 (Philox counter field)"};
    if (cfg->rs_steps > 4095) throw Fail{FB_ERR_INVALID_ARG, "rs_steps > 4095 (Philox counter field)"};
    if (!(cfg->alpha >= 0.0f)) throw Fail{FB_ERR_INVALID_ARG, "alpha < 0"};
    if (cfg->loss < 0 || cfg->loss > 3) throw Fail{FB_ERR_INVALID_ARG, "unknown loss"};
    if (cfg->init < 0 || cfg->init > 1) throw Fail{FB_ERR_INVALID_ARG, "unknown init"};
    if (cfg->prop_scales < 0 || cfg->prop_scales > 12) throw Fail{FB_ERR_INVALID_ARG, "prop_scales not in [0, 12]"};
    if (cfg->tracking < 0 || cfg->tracking > 1) throw Fail{FB_ERR_INVALID_ARG, "tracking must be 0 or 1"};
}

// ------------------------------------------------------------------------------------ pyramids
struct Pyr {
    float4* base = nullptr;
    long long stride = 0;  // texels per frame
    const float4* frame(long long i) const { return base + i * stride; }
};

Pyr pyramid_u8(Exec& ex, const Geo& g, const uint8_t* frames, int B)
{
    Pyr P;
    P.stride = g.pyr_texels;
    P.base = ex.ar.take<float4>((size_t)B * P.stride);
    if (B == 0) return P;
    ex.launch("pyr0", [&] { return fbk::launch_u8_to_pyr0(frames, P.base, B, g.H, g.W, P.stride, ex.ctx->stream); });
    for (int k = 1; k < g.Lv; ++k)
        ex.launch("box", [&] { return fbk::launch_box(P.base, B, P.stride, g.L[k - 1], g.L[k], ex.ctx->stream); });
    return P;
}

void pyramid_levels_inplace(Exec& ex, const Geo& g, float4* base, int B, long long stride)
{
    for (int k = 1; k < g.Lv; ++k)
        ex.launch("box", [&] { return fbk::launch_box(base, B, stride, g.L[k - 1], g.L[k], ex.ctx->stream); });
}

// ------------------------------------------------------------------------------------ packed sources
// A source slot = (source guide, source style): the frame pair an NNF task matches from.  Slots are
// packed once per call (zero border) and shared by every task that reads them.
struct SlotSpec {
    const uint8_t* g8;  // uint8 [H,W,3] guide (SF8 level 0)
    const uint8_t* s8;  // uint8 [H,W,3] style (SF8 level 0; NULL = zeros, BASE loss)
    const float4* gp;   // guide float4 pyramid
    const float4* sp;   // style float4 pyramid (NULL = zeros, BASE loss)
};
struct Slots {
    char* base = nullptr;
    size_t stride = 0;  // bytes per slot
    size_t off[24] = {};
    long long sum_off[24];  // patch-sum plane of level k inside a slot (kernels.h SumJob), or -1
    long long tail_off[24];  // tail-row sums plane of level k (SumJob::tail), or -1
    int fmt0 = fbk::SF8;
    Slots() { std::fill(sum_off, sum_off + 24, -1LL); std::fill(tail_off, tail_off + 24, -1LL); }
    const char* slot(long long i) const { return base + (size_t)i * stride; }
};

Slots pack_sources(Exec& ex, const Geo& g, int fmt0, const std::vector<SlotSpec>& specs)
{
    Slots S;
    if (g.p > 2 && fmt0 == fbk::SF8F) fmt0 = fbk::SF32;  // float styles at p > 2: general kernel
    S.fmt0 = fmt0;
    size_t off = 0;
    const int D = 2 * g.p + 1;
    for (int k = 0; k < g.Lv; ++k) {
        S.off[k] = off;
        const int f = src_fmt(fmt0, k);
        const size_t copies = f == fbk::SF8 ? fbk::kSF8Copies : (f == fbk::SF10 ? 2 : 1);
        off = (off + copies * g.PL[k].rows * g.PL[k].pitch * src_bytes(f) + 255) & ~size_t(255);
        // patch sums for the random-search bound (exact packed sources: SF8 at level 0, SF10, SF16); every sum
        // must fit its 21-bit field (and, through the fused kernel at level 1, its 16-bit target sums)
        const bool sums = ex.ctx->sum_bound && (long long)D * D * 255 * (1LL << (2 * k)) < (1LL << 21) &&
                          (f == fbk::SF8 || f == fbk::SF10 || f == fbk::SF16 || (f == fbk::SF8F && g.p <= 2)) &&
                          (f != fbk::SF10 || !ex.ctx->l1_fast || D * D * 1020 < 65536);
        S.sum_off[k] = sums ? (long long)off : -1;
        if (sums) off = (off + (size_t)g.PL[k].h * g.PL[k].w * sizeof(uint4) * (f == fbk::SF8F ? 2 : 1) + 255) & ~size_t(255);
        // tail-row sums for the fused level-0 kernel's partial + remainder bound (p = 2, u8 sources)
        const bool tail = sums && ex.ctx->tail_bound && f == fbk::SF8 && k == 0 && g.p == 2;
        S.tail_off[k] = tail ? (long long)off : -1;
        if (tail) off = (off + (size_t)g.PL[k].h * g.PL[k].w * sizeof(uint4) + 255) & ~size_t(255);
    }
    S.stride = off;
    const int n = (int)specs.size();
    S.base = ex.ar.take<char>(std::max<size_t>(1, S.stride * (size_t)n));
    if (n == 0) return S;
    for (int k = 0; k < g.Lv; ++k) {
        std::vector<fbk::PackSrc> jobs(n);
        for (int i = 0; i < n; ++i) {
            const SlotSpec& sp = specs[i];
            jobs[i] = fbk::PackSrc{sp.g8, sp.s8, sp.gp ? sp.gp + g.L[k].off : nullptr,
                                   sp.sp ? sp.sp + g.L[k].off : nullptr, S.base + (size_t)i * S.stride + S.off[k]};
        }
        const fbk::PackSrc* dj = ex.upload(jobs);
        const int fmt = src_fmt(fmt0, k);
        ex.launch("pack_src", [&] { return fbk::launch_pack_src(dj, n, fmt, g.PL[k], ex.ctx->stream); },
                  (uint64_t)n * g.PL[k].rows * g.PL[k].pitch);
        if (S.sum_off[k] >= 0) {
            std::vector<fbk::SumJob> sj(n);
            for (int i = 0; i < n; ++i)
                sj[i] = fbk::SumJob{S.base + (size_t)i * S.stride + S.off[k],
                                    reinterpret_cast<uint4*>(S.base + (size_t)i * S.stride + S.sum_off[k]),
                                    S.tail_off[k] >= 0
                                        ? reinterpret_cast<uint4*>(S.base + (size_t)i * S.stride + S.tail_off[k])
                                        : nullptr};
            const fbk::SumJob* dsj = ex.upload(sj);
            ex.launch("patch_sums", [&] { return fbk::launch_patch_sums(dsj, n, fmt, g.PL[k], g.p, ex.ctx->stream); },
                      (uint64_t)n * g.PL[k].h * g.PL[k].w);
        }
    }
    return S;
}

// ------------------------------------------------------------------------------------ NNF batch (Alg. 1)
struct TaskSpec {
    const char* src;   // packed source slot
    const float4* ss;  // source style pyramid (the image being remapped, D22)
    const float4* tg;  // target guide pyramid
    int group;         // MEAN_ALIGN window index (into groups), else -1
    uint32_t src_id, tgt_id, tag;
    int partner = -1;  // PAIRWISE: index of the counterpart task in the batch (Eq. 10, D38)
    int track[2] = {-1, -1};  // tracking: batch indices of the tasks for T_{i-1}, T_{i+1} (D42)
};
struct GroupSpec {
    const float4* tstyle;  // target style pyramid (the self term of T-bar)
    const float4* tguide;  // target guide pyramid (the guide half of the packed target)
    uint32_t tgt_id;
};
struct BatchOut {
    int2* F = nullptr;  // final NNF of task t at F + t*fstride (level 0)
    float* E = nullptr;
    long long fstride = 0;
};

BatchOut run_nnf(Exec& ex, const fb_match_cfg& cfg, const Geo& g, const Slots& slots,
                 const std::vector<TaskSpec>& tasks, const std::vector<GroupSpec>& groups, fb_stats* st,
                 bool want_E = false)
{
    const int T = (int)tasks.size();
    const long long n0 = g.npx0();
    const cudaStream_t s = ex.ctx->stream;
    // level 0 uses packed u8 operands (TF16 targets) with SF8 / SF8F sources: in registers (fast kernels,
    // p <= 2) or as a shared-memory tile (mid kernel, p = 3, 4)
    const bool fast0 = slots.fmt0 == fbk::SF8 || slots.fmt0 == fbk::SF8F;
    const bool l1_fast_ok = ex.ctx->l1_fast && slots.fmt0 == fbk::SF8 && g.p == 2 && g.Lv > 1 &&
                            (cfg.loss == FB_LOSS_GUIDE_STYLE || cfg.loss == FB_LOSS_MEAN_ALIGN);
    BatchOut out;
    out.fstride = n0;
    int2* F[2] = {ex.ar.take<int2>((size_t)T * n0), ex.ar.take<int2>((size_t)T * n0)};
    out.E = ex.ar.take<float>((size_t)T * n0);
    // The fused fields-1-3 kernel must not overwrite E in place: its halo lanes read the field-0 E of pixels
    // owned by neighbouring tiles.  Its final E goes to a second buffer, needed only when the caller asks
    // for E (the next iteration recomputes E <- L(F) anyway, D17).
    float* E_final = want_E ? ex.ar.take<float>((size_t)T * n0) : nullptr;
    bool e_final_used = false;
    size_t tbytes = 0;  // one packed target operand, largest level
    for (int k = 0; k < g.Lv; ++k)
        tbytes = std::max(tbytes, (size_t)g.PL[k].rows * g.PL[k].pitch *
                                      (((k == 0 && fast0) || (k == 1 && l1_fast_ok)) ? 16 : 32));
    tbytes = (tbytes + 255) & ~size_t(255);
    const bool per_group = cfg.loss == FB_LOSS_MEAN_ALIGN;
    const bool pairwise = cfg.loss == FB_LOSS_PAIRWISE;
    bool tracking = false;
    uint64_t track_links = 0;
    for (const TaskSpec& k : tasks)
        for (int z = 0; z < 2; ++z)
            if (k.track[z] >= 0) { tracking = true; ++track_links; }
    char* tgt = ex.ar.take<char>(tbytes * (per_group ? groups.size() : (size_t)T));
    // NNFs frozen at the start of each iteration: counterparts (D39) and tracking neighbours (D42)
    int2* Fsnap = (pairwise || tracking) ? ex.ar.take<int2>((size_t)T * n0) : nullptr;
    std::vector<DTask> dt(T);
    for (int t = 0; t < T; ++t) {
        const TaskSpec& k = tasks[t];
        dt[t].src = k.src;
        dt[t].tgt = tgt + tbytes * (per_group ? (size_t)k.group : (size_t)t);
        dt[t].ss = k.ss;
        dt[t].tg = k.tg;
        dt[t].c2 = k.src_id;
        dt[t].c3 = (k.tag << 28) | k.tgt_id;
        dt[t].psrc = pairwise ? tasks[k.partner].src : nullptr;
        dt[t].pF = pairwise ? Fsnap + (long long)k.partner * n0 : nullptr;
        for (int z = 0; z < 2; ++z) dt[t].trk[z] = k.track[z] >= 0 ? Fsnap + (long long)k.track[z] * n0 : nullptr;
    }
    const DTask* d_tasks = ex.upload(dt);
    // T-bar member lists for every level (MEAN_ALIGN): ascending source id with the self term inserted.
    std::vector<const DOut*> d_outs(g.Lv, nullptr);
    std::vector<const DMember*> d_mem(g.Lv, nullptr);
    if (per_group) {
        std::vector<std::vector<int>> members(groups.size());
        for (int t = 0; t < T; ++t) members[tasks[t].group].push_back(t);
        for (auto& m : members)
            std::sort(m.begin(), m.end(), [&](int a, int b) { return tasks[a].src_id < tasks[b].src_id; });
        for (int k = 0; k < g.Lv; ++k) {
            std::vector<DOut> outs;
            std::vector<DMember> mem;
            for (size_t gi = 0; gi < groups.size(); ++gi) {
                DOut o;
                o.m0 = (int)mem.size();
                bool self_done = false;
                for (int t : members[gi]) {
                    if (!self_done && tasks[t].src_id > groups[gi].tgt_id) {
                        mem.push_back(DMember{groups[gi].tstyle + g.L[k].off, -1, 1.0f, nullptr, -1});
                        self_done = true;
                    }
                    const int sf = src_fmt(slots.fmt0, k);
                    mem.push_back(DMember{tasks[t].ss + g.L[k].off, t, 1.0f, tasks[t].src + slots.off[k],
                                          sf == fbk::SF32 ? -1 : sf});
                }
                if (!self_done) mem.push_back(DMember{groups[gi].tstyle + g.L[k].off, -1, 1.0f, nullptr, -1});
                o.nm = (int)mem.size() - o.m0;
                o.div = (float)o.nm;
                o.fmt = (k == 0 && fast0) ? 2 : 3;
                o.out = tgt + tbytes * gi;
                o.guide = groups[gi].tguide + g.L[k].off;
                outs.push_back(o);
            }
            d_outs[k] = ex.upload(outs);
            d_mem[k] = ex.upload(mem);
        }
    }
    const fbk::Rng rng{(uint32_t)(cfg.seed & 0xFFFFFFFFu), (uint32_t)(cfg.seed >> 32)};
    int cur = 0;
    Nvtx nv_nnf(ex.dry, "nnf batch (%d pairs)", T);
    for (int k = g.Lv - 1; k >= 0; --k) {
        Nvtx nv_level(ex.dry, "level %d", k);
        const Lvl L = g.L[k];
        const fbk::PLvl PL = g.PL[k];
        const bool tf16 = k == 0 && fast0;
        const bool fast = tf16 && g.p <= 2;                 // kernel kind 1
        // level 1 of u8 sources: SF10 source + TF10 target through the mid / fused kernels (p = 2)
        const bool l1 = l1_fast_ok && k == 1;
        const int kind = fast ? 1 : ((tf16 || l1) ? 2 : 0);  // 2: mid kernel (p = 3, 4 at level 0; level 1)
        const int tfmt = tf16 ? fbk::TF16 : (l1 ? fbk::TF10 : fbk::TF32);
        if (k == g.Lv - 1) {
            ex.launch("init", [&] { return fbk::launch_init(d_tasks, T, F[cur], n0, L, cfg.init == FB_INIT_IDENTITY,
                                                            rng, (uint32_t)k, s); });
        } else {
            ex.launch("upsample", [&] { return fbk::launch_upsample(F[cur], F[cur ^ 1], T, n0, g.L[k + 1], L, s); });
            cur ^= 1;
        }
        if (cfg.loss == FB_LOSS_BASE || pairwise)  // the target operand is the target guide alone
            ex.launch("pack_tgt", [&] { return fbk::launch_pack_tgt_guide(d_tasks, T, L, PL, tfmt, s); });
        const int rk = rs_count(cfg, L), r0 = rs_r0(cfg, L);
        for (int it = 0; it < cfg.iters_per_level; ++it) {
            Nvtx nv_iter(ex.dry, "iteration %d", it);
            if (Fsnap)  // freeze counterpart / tracking NNFs for this iteration (D39, D42)
                ex.d2d(Fsnap, F[cur], sizeof(int2) * (size_t)T * n0);
            if (cfg.loss == FB_LOSS_GUIDE_STYLE) {  // S^ refresh (D17/D18)
                ex.launch("aux", [&] { return fbk::launch_aux_remap(d_tasks, T, F[cur], n0, L, PL, g.p, tfmt,
                                                                       src_fmt(slots.fmt0, k), (long long)slots.off[k], s); },
                          (uint64_t)T * L.h * L.w);
                if (st) st->remap_pixels += (uint64_t)T * L.h * L.w;
            } else if (per_group) {  // T-bar refresh (Eq. 7, D27)
                ex.launch(k == 0 ? "tbar.L0" : "tbar.L1+", [&] { return fbk::launch_combine(d_outs[k], (int)groups.size(), d_mem[k], F[cur], n0,
                                                                   L.h, L.w, g.p, tf16 ? 2 : (l1 ? 4 : 3), PL, s); },
                          (uint64_t)T * L.h * L.w);
                if (st) st->remap_pixels += (uint64_t)T * L.h * L.w;
            }
            fbk::FieldArgs a{};
            a.tasks = d_tasks; a.E = out.E; a.fstride = n0; a.L = PL; a.src_off = (long long)slots.off[k];
            a.alpha = cfg.alpha; a.rng = rng; a.level = (uint32_t)k; a.iter = (uint32_t)it; a.rs_r0 = r0; a.rs_k = rk;
            a.src_fmt = src_fmt(slots.fmt0, k);
            a.tgt_reg_rows = ex.ctx->tgt_reg_rows;
            a.sum_off = slots.sum_off[k];
            a.tail_off = slots.tail_off[k];
            char names[4][32];
            for (int ph = 0; ph < 4; ++ph) snprintf(names[ph], sizeof names[ph], "field%d.L%d", ph, k);
            const int J = std::max(1, cfg.prop_scales);  // jump-flood scales (D41)
            a.einit = 1;
            a.do_rs = 0;
            if (fast && ex.ctx->fused && J == 1) {  // one fused launch per iteration (FB_FUSED=1)
                char nm[32];
                snprintf(nm, sizeof nm, "iter.L%d", k);
                a.step = 1;
                a.Fin = F[cur]; a.Fout = F[cur ^ 1];
                ex.launch(nm, [&] { return fbk::launch_iter_fast(a, T, g.p, cfg.loss, s); },
                          (uint64_t)(5 + rk) * T * L.h * L.w);
                cur ^= 1;
                continue;
            }
            for (int j = J - 1; j >= 0; --j) {
                a.step = 1 << j;
                const bool last = j == 0;
                // p = 3 at level 0 (u8 sources): fields 1-3 + random search fused as well (FB_OPT_P3_FUSED)
                const bool p3f = ex.ctx->p3_fused && tf16 && g.p == 3 && !pairwise && slots.fmt0 == fbk::SF8;
                if (last && (fast || p3f || (l1 && ex.ctx->l1_fast == 1)) && ex.ctx->fuse13) {  // field 0, then fields 1-3 + random search in one launch
                    a.Fin = F[cur]; a.Fout = F[cur ^ 1];
                    const int kind0 = (l1 || (ex.ctx->phase0_mid && !pairwise && g.p == 2 &&
                                              (a.src_fmt == fbk::SF8 || a.src_fmt == fbk::SF8F))) ? 2 : kind;
                    ex.launch(names[0], [&] { return fbk::launch_field(a, T, g.p, cfg.loss, 0, kind0, s); },
                              (1ull + (uint64_t)a.einit) * T * L.h * L.w);
                    cur ^= 1;
                    char nm[32];
                    snprintf(nm, sizeof nm, "field123.L%d", k);
                    a.Fin = F[cur]; a.Fout = F[cur ^ 1];
                    a.Eout = E_final;
                    e_final_used = k == 0 && it == cfg.iters_per_level - 1;
                    ex.launch(nm, [&] { return fbk::launch_iter13_fast(a, T, g.p, cfg.loss, s); },
                              (uint64_t)(3 + rk) * T * L.h * L.w);
                    cur ^= 1;
                    continue;
                }
                for (int ph = 0; ph < 4; ++ph) {
                    a.Fin = F[cur]; a.Fout = F[cur ^ 1];
                    a.do_rs = last && ph == 3;
                    const uint64_t per_px = 1 + (ph == 0 ? (uint64_t)a.einit : 0) + (a.do_rs ? (uint64_t)rk : 0);
                    ex.launch(names[ph], [&] { return fbk::launch_field(a, T, g.p, cfg.loss, ph, kind, s); },
                              per_px * (uint64_t)T * L.h * L.w);
                    cur ^= 1;
                    a.einit = 0;
                }
                a.einit = 0;
            }
        }
    }
    out.F = F[cur];
    if (e_final_used) out.E = E_final;
    if (st) {
        st->nnf_pairs += (uint64_t)T;
        st->candidate_evals += (uint64_t)T * evals_per_pair(cfg, g);
        for (int k = 0; k < g.Lv; ++k)  // tracking fields (D42)
            st->candidate_evals += track_links * (uint64_t)g.L[k].h * g.L[k].w * (uint64_t)cfg.iters_per_level;
    }
    return out;
}

// Final combine at level 0 into API-layout float [.., H, W, 3] rows.
struct CombineList {
    std::vector<DOut> outs;
    std::vector<DMember> mem;
    void begin() { outs.push_back(DOut{(int)mem.size(), 0, 1.0f, 1, nullptr, nullptr}); }
    void add_img(const float4* img, float w) { mem.push_back(DMember{img, -1, w, nullptr, -1}); ++outs.back().nm; }
    void add_remap(const float4* src_level_img, int task, float w)
    {
        mem.push_back(DMember{src_level_img, task, w, nullptr, -1});
        ++outs.back().nm;
    }
    // Remap read from the same image held exactly in a packed u8 slot (4 B per tap instead of 16; the
    // kernel's exact integer form gives identical values); other slot formats use the float image.
    void add_remap(const float4* src_level_img, int task, float w, const Slots& S, long long slot)
    {
        const bool u8 = src_fmt(S.fmt0, 0) == fbk::SF8;
        mem.push_back(DMember{src_level_img, task, w, u8 ? S.slot(slot) + S.off[0] : nullptr, u8 ? fbk::SF8 : -1});
        ++outs.back().nm;
    }
    void end(void* out, int fmt, float div) { outs.back().out = out; outs.back().fmt = fmt; outs.back().div = div; }
};

void run_combine(Exec& ex, const Geo& g, int k, const CombineList& cl, const int2* F, long long fstride)
{
    if (cl.outs.empty()) return;
    const DOut* o = ex.upload(cl.outs);
    const DMember* m = ex.upload(cl.mem);
    const int fmt = cl.outs[0].fmt;
    ex.launch("combine", [&] { return fbk::launch_combine(o, (int)cl.outs.size(), m, F, fstride, g.L[k].h, g.L[k].w,
                                                          g.p, fmt, g.PL[k], ex.ctx->stream); },
              (uint64_t)cl.outs.size() * g.L[k].h * g.L[k].w);
}

size_t per_pair_bytes(const Geo& g, int loss)
{
    // F ping-pong + E + (GS aux) per pair, plus descriptor slack
    const size_t tgt = (size_t)g.PL[0].rows * g.PL[0].pitch * 32;
    return (size_t)g.npx0() * (2 * sizeof(int2) + sizeof(float)) + (loss == FB_LOSS_MEAN_ALIGN ? 0 : tgt) + 4096;
}

int batch_pairs(fb_ctx ctx, const Geo& g, int loss)
{
    long long m = ctx->max_pairs > 0 ? ctx->max_pairs : (long long)(kAutoStateBudget / per_pair_bytes(g, loss));
    m = std::max<long long>(1, std::min<long long>(m, kMaxBatchPairs));
    return (int)m;
}

// Split consecutive units (each with `cost` pairs, never split) into batches of <= cap pairs.
std::vector<std::pair<int, int>> make_batches(const std::vector<int>& cost, int cap)
{
    std::vector<std::pair<int, int>> b;
    int start = 0, acc = 0;
    for (int i = 0; i < (int)cost.size(); ++i) {
        if (acc > 0 && acc + cost[i] > cap) { b.push_back({start, i}); start = i; acc = 0; }
        acc += cost[i];
    }
    if (start < (int)cost.size()) b.push_back({start, (int)cost.size()});
    return b;
}

// ------------------------------------------------------------------------------------ direct schedule
// Eq. 2 + Eq. 3 (balanced) or Eq. 7/8 (accurate), O(N*M) NNFs.
// Streaming ("Users can process long videos in accurate mode"): each batch of
// targets builds the pyramids and packed slots of only the frames its windows read, [first-M, last+M],
// inside the batch's arena region, so device memory is O(batch + 2M) frames, not O(N).
void blend_direct(Exec& ex, const fb_match_cfg& cfg, const Geo& g, int N_total, int f0, int N, int M,
                  const uint8_t* guide, const uint8_t* style, int t0, int t1, float* out, fb_stats* st)
{
    (void)N;
    const long long n0 = g.npx0();
    std::vector<int> cost;
    for (int i = t0; i < t1; ++i) cost.push_back(std::min(N_total - 1, i + M) - std::max(0, i - M));
    // tracking in blending (reading D44) couples every pair of the schedule: one batch
    long long total = 0;
    for (int c : cost) total += c;
    if (cfg.tracking && total > kMaxBatchPairs)
        throw Fail{FB_ERR_UNSUPPORTED, "tracking in blending needs all pairs of the schedule in one batch"};
    const auto batches = cfg.tracking ? std::vector<std::pair<int, int>>{{0, t1 - t0}}
                                      : make_batches(cost, batch_pairs(ex.ctx, g, cfg.loss));
    const size_t mark = ex.ar.off;
    for (auto [b0, b1] : batches) {
        Nvtx nv(ex.dry, "direct batch targets [%d, %d)", t0 + b0, t0 + b1);
        ex.ar.off = mark;
        // frames this batch reads (original ids), then their local (input) and batch indices
        const int lo_b = std::max(0, t0 + b0 - M), hi_b = std::min(N_total - 1, t0 + b1 - 1 + M);
        const int nb = hi_b - lo_b + 1;
        const uint8_t* gb = guide + 3 * n0 * (lo_b - f0);
        const uint8_t* sb = style + 3 * n0 * (lo_b - f0);
        const Pyr G = pyramid_u8(ex, g, gb, nb);
        const Pyr S = pyramid_u8(ex, g, sb, nb);
        std::vector<SlotSpec> specs;
        for (int j = 0; j < nb; ++j) specs.push_back(SlotSpec{gb + 3 * n0 * j, sb + 3 * n0 * j, G.frame(j), S.frame(j)});
        const Slots FR = pack_sources(ex, g, fbk::SF8, specs);
        std::vector<TaskSpec> tasks;
        std::vector<GroupSpec> groups;
        std::vector<int> first(b1 - b0);
        for (int q = b0; q < b1; ++q) {
            const int i = t0 + q, lo = std::max(0, i - M), hi = std::min(N_total - 1, i + M);
            first[q - b0] = (int)tasks.size();
            if (cfg.loss == FB_LOSS_MEAN_ALIGN) groups.push_back(GroupSpec{S.frame(i - lo_b), G.frame(i - lo_b), (uint32_t)i});
            for (int j = lo; j <= hi; ++j) {
                if (j == i) continue;
                tasks.push_back(TaskSpec{FR.slot(j - lo_b), S.frame(j - lo_b), G.frame(i - lo_b),
                                         cfg.loss == FB_LOSS_MEAN_ALIGN ? q - b0 : -1, (uint32_t)j, (uint32_t)i, 0u});
            }
        }
        if (cfg.tracking) {  // D44: NNF(G_j -> G_i) also tries NNF(G_j -> G_{i-1}) and NNF(G_j -> G_{i+1})
            std::map<std::pair<uint32_t, uint32_t>, int> idx;
            for (int k = 0; k < (int)tasks.size(); ++k) idx[{tasks[k].src_id, tasks[k].tgt_id}] = k;
            for (TaskSpec& tk : tasks)
                for (int z = 0; z < 2; ++z) {
                    const auto it = idx.find({tk.src_id, z == 0 ? tk.tgt_id - 1 : tk.tgt_id + 1});
                    if (it != idx.end()) tk.track[z] = it->second;
                }
        }
        BatchOut bo;
        if (!tasks.empty()) bo = run_nnf(ex, cfg, g, FR, tasks, groups, st);
        CombineList cl;  // out_i = (sum_{j asc} X_{j->i}) / |W_i|, X_{i->i} = S_i (D3, D4)
        for (int q = b0; q < b1; ++q) {
            const int i = t0 + q, lo = std::max(0, i - M), hi = std::min(N_total - 1, i + M);
            int t = first[q - b0];
            cl.begin();
            for (int j = lo; j <= hi; ++j) {
                if (j == i) cl.add_img(S.frame(i - lo_b), 1.0f);
                else cl.add_remap(S.frame(j - lo_b), t++, 1.0f, FR, j - lo_b);
            }
            cl.end(out + 3LL * n0 * q, 1, (float)(hi - lo + 1));
            if (st) st->remap_pixels += (uint64_t)(hi - lo) * n0;
        }
        run_combine(ex, g, 0, cl, bo.F, bo.fstride);
    }
}

// ------------------------------------------------------------------------------------ tree schedule
// Alg. 3 (remapping table), Alg. 4 (blending table), Alg. 5 (query) on the forward and the reversed
// frame order (D26), merged by Eq. 6.  Tables hold means (D25); levels capped at floor(log2(M+1))
// (D24); only the cells the requested targets' queries visit are built (the "task manager").

std::vector<std::pair<int, int>> query_nodes(int l, int r)  // Alg. 5 with i <- i - 2^L (D23)
{
    std::vector<std::pair<int, int>> v;
    int i = r;
    while (i >= l) {
        int L = 0;
        while ((i & (1 << L)) && i - (1 << (L + 1)) + 1 >= l) ++L;
        v.push_back({i, L});
        i -= 1 << L;
    }
    return v;
}

// Blending-table cells BT(j, L) (L >= 1) of one orientation, as float4 pyramids (g.pyr_texels each).
using CellMap = std::map<std::pair<int, int>, const float4*>;

// Alg. 3 + Alg. 4 for the cells (j, 1..top[j]) of orientation o (j in orientation order): RT sums of the
// remaps X_{v->j}, v in [j-2^L+1, j-2^(L-1)] ascending, then BT(j,L) = (BT(j,L-1) + RT(j,L)*2^-(L-1))*0.5
// level by level, then the BT pyramids.  The BT block stays in the arena (caller's mark).
CellMap tree_build(Exec& ex, const fb_match_cfg& cfg, const Geo& g, int N_total, int f0, const Pyr& G, const Pyr& S,
                   const Slots& FR, int o, const std::vector<int>& top, fb_stats* st)
{
    Nvtx nv(ex.dry, "tree build (orientation %d)", o);
    const long long n0 = g.npx0();
    auto orig = [&](int v) { return o == 0 ? v : N_total - 1 - v; };
    const uint32_t tag_build = o == 0 ? 1u : 3u;
    std::map<std::pair<int, int>, int> cell_id;  // (j, L) -> index
    std::vector<std::pair<int, int>> cells;
    int lmax = 0;
    for (int j = 0; j < (int)top.size(); ++j)
        for (int L = 1; L <= top[j]; ++L) { cell_id[{j, L}] = (int)cells.size(); cells.push_back({j, L}); lmax = std::max(lmax, L); }
    const int nc = (int)cells.size();
    float4* BT = ex.ar.take<float4>((size_t)nc * g.pyr_texels);  // BT cell pyramids (survive this call)
    const size_t mark0 = ex.ar.off;
    float4* RT = ex.ar.take<float4>((size_t)nc * n0);            // RT sums, level 0
    auto bt_pyr = [&](int v, int L) -> const float4* {
        return L == 0 ? S.frame(orig(v) - f0) : BT + (long long)cell_id.at({v, L}) * g.pyr_texels;
    };
    std::vector<int> cost(nc);
    for (int c = 0; c < nc; ++c) cost[c] = 1 << (cells[c].second - 1);
    const int cap = batch_pairs(ex.ctx, g, cfg.loss);
    const size_t mark = ex.ar.off;
    for (auto [c0, c1] : make_batches(cost, cap)) {
        ex.ar.off = mark;
        std::vector<TaskSpec> tasks;
        for (int c = c0; c < c1; ++c) {
            const auto [j, L] = cells[c];
            for (int v = j - (1 << L) + 1; v <= j - (1 << (L - 1)); ++v)
                tasks.push_back(TaskSpec{FR.slot(orig(v) - f0), S.frame(orig(v) - f0), G.frame(orig(j) - f0), -1,
                                         (uint32_t)orig(v), (uint32_t)orig(j), tag_build});
        }
        BatchOut bo = run_nnf(ex, cfg, g, FR, tasks, {}, st);
        CombineList cl;
        int t = 0;
        for (int c = c0; c < c1; ++c) {
            const auto [j, L] = cells[c];
            cl.begin();
            for (int v = j - (1 << L) + 1; v <= j - (1 << (L - 1)); ++v) cl.add_remap(S.frame(orig(v) - f0), t++, 1.0f);
            cl.end(RT + (long long)c * n0, 0, 1.0f);
        }
        if (st) st->remap_pixels += (uint64_t)tasks.size() * n0;
        run_combine(ex, g, 0, cl, bo.F, bo.fstride);
    }
    ex.ar.off = mark;
    for (int L = 1; L <= lmax; ++L) {
        CombineList cl;
        for (int c = 0; c < nc; ++c) {
            if (cells[c].second != L) continue;
            const int j = cells[c].first;
            cl.begin();
            cl.add_img(bt_pyr(j, L - 1), 1.0f);
            cl.add_img(RT + (long long)c * n0, 1.0f / (float)(1 << (L - 1)));
            cl.end(BT + (long long)c * g.pyr_texels, 0, 2.0f);
        }
        run_combine(ex, g, 0, cl, nullptr, 0);
    }
    if (nc) pyramid_levels_inplace(ex, g, BT, nc, g.pyr_texels);
    ex.ar.off = mark0;  // RT is dead; BT stays
    CellMap m;
    for (int c = 0; c < nc; ++c) m[cells[c]] = BT + (long long)c * g.pyr_texels;
    return m;
}

// Alg. 5 queries of targets [t0, t1) in orientation o into A (one float4 image per target):
// A = sum over the visited nodes of 2^L * (BT(node, L) -> S_r); the self node is BT itself; L = 0 nodes are
// frames.  Every visited (node, L >= 1) must be in `cells`.
void tree_query(Exec& ex, const fb_match_cfg& cfg, const Geo& g, int N_total, int f0, int M, const Pyr& G,
                const Pyr& S, int o, int t0, int t1, const CellMap& cells, float4* A, fb_stats* st)
{
    Nvtx nv(ex.dry, "tree queries (orientation %d)", o);
    const long long n0 = g.npx0();
    auto orig = [&](int v) { return o == 0 ? v : N_total - 1 - v; };
    const uint32_t tag_query = o == 0 ? 2u : 4u;
    auto bt_pyr = [&](int v, int L) -> const float4* {
        if (L == 0) return S.frame(orig(v) - f0);
        auto it = cells.find({v, L});
        if (it == cells.end()) throw Fail{FB_ERR_INVALID_ARG, "a query visits a blending-table cell that was not provided"};
        return it->second;
    };
    std::vector<int> qcost;
    std::vector<std::vector<std::pair<int, int>>> walks;
    for (int i = t0; i < t1; ++i) {
        const int v = o == 0 ? i : N_total - 1 - i;
        walks.push_back(query_nodes(std::max(0, v - M), v));
        qcost.push_back((int)walks.back().size() - 1);
    }
    const int cap = batch_pairs(ex.ctx, g, cfg.loss);
    const size_t mark2 = ex.ar.off;
    for (auto [q0, q1] : make_batches(qcost, cap)) {
        ex.ar.off = mark2;
        std::vector<TaskSpec> tasks;
        std::vector<SlotSpec> qspecs;  // query sources: (G_i, BT(i,L)) packed as SF8F (float style)
        for (int q = q0; q < q1; ++q) {
            const int i = t0 + q, v = o == 0 ? i : N_total - 1 - i;
            for (auto [node, L] : walks[q]) {
                if (node == v) continue;
                qspecs.push_back(SlotSpec{nullptr, nullptr, G.frame(orig(node) - f0), bt_pyr(node, L)});
                tasks.push_back(TaskSpec{nullptr, bt_pyr(node, L), G.frame(i - f0), -1, (uint32_t)orig(node),
                                         (uint32_t)i, tag_query});
            }
        }
        const Slots QS = pack_sources(ex, g, fbk::SF8F, qspecs);
        for (size_t t = 0; t < tasks.size(); ++t) tasks[t].src = QS.slot((long long)t);
        BatchOut bo;
        if (!tasks.empty()) bo = run_nnf(ex, cfg, g, QS, tasks, {}, st);
        CombineList cl;
        int t = 0;
        for (int q = q0; q < q1; ++q) {
            const int v = o == 0 ? t0 + q : N_total - 1 - (t0 + q);
            cl.begin();
            for (auto [node, L] : walks[q]) {
                const float wgt = (float)(1 << L);
                if (node == v) cl.add_img(bt_pyr(node, L), wgt);
                else cl.add_remap(bt_pyr(node, L), t++, wgt);
            }
            cl.end(A + (long long)q * n0, 0, 1.0f);
        }
        if (st) st->remap_pixels += (uint64_t)tasks.size() * n0;
        run_combine(ex, g, 0, cl, bo.F, bo.fstride);
    }
    ex.ar.off = mark2;
}

// Levels of the cells the queries of targets [t0, t1) visit, per node of orientation o.
std::vector<int> tree_top(int N_total, int M, int o, int t0, int t1)
{
    std::vector<int> top(N_total, 0);
    for (int i = t0; i < t1; ++i) {
        const int v = o == 0 ? i : N_total - 1 - i;
        for (auto [node, L] : query_nodes(std::max(0, v - M), v)) top[node] = std::max(top[node], L);
    }
    return top;
}

// Eq. 6: out_i = ((A_f + A_r) - S_i) / |W_i|
void tree_merge(Exec& ex, const Geo& g, int N_total, int f0, int M, const Pyr& S, int t0, int t1, float4* const A[2],
                float* out)
{
    const long long n0 = g.npx0();
    CombineList cl;
    for (int q = 0; q < t1 - t0; ++q) {
        const int i = t0 + q, lo = std::max(0, i - M), hi = std::min(N_total - 1, i + M);
        cl.begin();
        cl.add_img(A[0] + (long long)q * n0, 1.0f);
        cl.add_img(A[1] + (long long)q * n0, 1.0f);
        cl.add_img(S.frame(i - f0), -1.0f);
        cl.end(out + 3LL * n0 * q, 1, (float)(hi - lo + 1));
    }
    run_combine(ex, g, 0, cl, nullptr, 0);
}

// Whole tree schedule for targets [t0, t1), building every cell its queries visit locally.
void blend_tree(Exec& ex, const fb_match_cfg& cfg0, const Geo& g, int N_total, int f0, int N, int M,
                const uint8_t* guide, const uint8_t* style, int t0, int t1, float* out, fb_stats* st)
{
    fb_match_cfg cfg = cfg0;
    cfg.loss = FB_LOSS_GUIDE_STYLE;  // D22: the loss is taken on the image being remapped
    const Pyr G = pyramid_u8(ex, g, guide, N);
    const Pyr S = pyramid_u8(ex, g, style, N);
    const long long n0 = g.npx0();
    std::vector<SlotSpec> specs;
    for (int j = 0; j < N; ++j) specs.push_back(SlotSpec{guide + 3 * n0 * j, style + 3 * n0 * j, G.frame(j), S.frame(j)});
    const Slots FR = pack_sources(ex, g, fbk::SF8, specs);
    const int nt = t1 - t0;
    float4* A[2] = {ex.ar.take<float4>((size_t)nt * n0), ex.ar.take<float4>((size_t)nt * n0)};
    for (int o = 0; o < 2; ++o) {
        const size_t omark = ex.ar.off;  // this orientation's tables die once its A is written
        const CellMap cells = tree_build(ex, cfg, g, N_total, f0, G, S, FR, o, tree_top(N_total, M, o, t0, t1), st);
        tree_query(ex, cfg, g, N_total, f0, M, G, S, o, t0, t1, cells, A[o], st);
        ex.ar.off = omark;
    }
    tree_merge(ex, g, N_total, f0, M, S, t0, t1, A, out);
}

// Sharded tree schedule with cell exchange, phase 1: build the listed cells {o, j, L}
// (orientation order) into cell_out, one pyramid of g.pyr_texels float4 texels per listed cell.
void tree_build_cells(Exec& ex, const fb_match_cfg& cfg0, const Geo& g, int N_total, int f0, int N,
                      const uint8_t* guide, const uint8_t* style, int n_cells, const int32_t* cl, float* cell_out,
                      fb_stats* st)
{
    fb_match_cfg cfg = cfg0;
    cfg.loss = FB_LOSS_GUIDE_STYLE;
    const Pyr G = pyramid_u8(ex, g, guide, N);
    const Pyr S = pyramid_u8(ex, g, style, N);
    const long long n0 = g.npx0();
    std::vector<SlotSpec> specs;
    for (int j = 0; j < N; ++j) specs.push_back(SlotSpec{guide + 3 * n0 * j, style + 3 * n0 * j, G.frame(j), S.frame(j)});
    const Slots FR = pack_sources(ex, g, fbk::SF8, specs);
    for (int o = 0; o < 2; ++o) {
        std::vector<int> top(N_total, 0);
        bool any = false;
        for (int c = 0; c < n_cells; ++c)
            if (cl[3 * c] == o) { top[cl[3 * c + 1]] = std::max(top[cl[3 * c + 1]], cl[3 * c + 2]); any = true; }
        if (!any) continue;
        const size_t omark = ex.ar.off;
        const CellMap cells = tree_build(ex, cfg, g, N_total, f0, G, S, FR, o, top, st);
        for (int c = 0; c < n_cells; ++c)
            if (cl[3 * c] == o)
                ex.d2d(cell_out + (size_t)c * 4 * g.pyr_texels, cells.at({cl[3 * c + 1], cl[3 * c + 2]}),
                       sizeof(float4) * (size_t)g.pyr_texels);
        ex.ar.off = omark;
    }
}

// Phase 2: the queries of targets [t0, t1) from local frames plus the given cells, then Eq. 6.
void tree_query_cells(Exec& ex, const fb_match_cfg& cfg0, const Geo& g, int N_total, int f0, int N, int M,
                      const uint8_t* guide, const uint8_t* style, int t0, int t1, int n_cells, const int32_t* cl,
                      const float* const* cell_ptrs, float* out, fb_stats* st)
{
    fb_match_cfg cfg = cfg0;
    cfg.loss = FB_LOSS_GUIDE_STYLE;
    const Pyr G = pyramid_u8(ex, g, guide, N);
    const Pyr S = pyramid_u8(ex, g, style, N);
    const long long n0 = g.npx0();
    const int nt = t1 - t0;
    float4* A[2] = {ex.ar.take<float4>((size_t)nt * n0), ex.ar.take<float4>((size_t)nt * n0)};
    for (int o = 0; o < 2; ++o) {
        CellMap cells;
        for (int c = 0; c < n_cells; ++c)
            if (cl[3 * c] == o)
                cells[{cl[3 * c + 1], cl[3 * c + 2]}] = cell_ptrs ? reinterpret_cast<const float4*>(cell_ptrs[c]) : nullptr;
        tree_query(ex, cfg, g, N_total, f0, M, G, S, o, t0, t1, cells, A[o], st);
    }
    tree_merge(ex, g, N_total, f0, M, S, t0, t1, A, out);
}

// ------------------------------------------------------------------------------------ interpolation
// Eq. 9 (D28).
// Targets [t0, t1) of an N-frame video: guide holds frames t0..t1-1; key_guide the K keyframes' guides
// (nullptr: taken from guide, which then must hold every keyframe, i.e. the full call).
void interpolate(Exec& ex, const fb_match_cfg& cfg0, const Geo& g, int N, int t0, int t1, const uint8_t* guide,
                 int K, const int32_t* keys, const uint8_t* key_guide, const uint8_t* key_style, float* out,
                 fb_stats* st)
{
    // cfg.loss == PAIRWISE: frames between two keys estimate both NNFs jointly with the alignment loss
    // of Eq. 10 (D38-D40); single-key frames and all other losses use Eq. 3 (GUIDE_STYLE).
    const bool align = cfg0.loss == FB_LOSS_PAIRWISE;
    const Pyr G = pyramid_u8(ex, g, guide, t1 - t0);
    const Pyr KS = pyramid_u8(ex, g, key_style, K);
    const long long n0 = g.npx0();
    Pyr GK;
    if (key_guide) GK = pyramid_u8(ex, g, key_guide, K);
    auto kg8 = [&](int k) { return key_guide ? key_guide + 3 * n0 * k : guide + 3 * n0 * (keys[k] - t0); };
    auto kgp = [&](int k) { return key_guide ? GK.frame(k) : G.frame(keys[k] - t0); };
    std::vector<SlotSpec> specs;
    for (int k = 0; k < K; ++k) specs.push_back(SlotSpec{kg8(k), key_style + 3 * n0 * k, kgp(k), KS.frame(k)});
    const Slots KSl = pack_sources(ex, g, (align && g.p > 2) ? fbk::SF32 : fbk::SF8, specs);
    struct Tgt { int m, left, right, key; };  // key indices (or -1)
    std::vector<Tgt> tg[2];  // [0]: keys and GUIDE_STYLE targets, [1]: aligned (two-key) targets
    for (int m = t0; m < t1; ++m) {
        Tgt t{m, -1, -1, -1};
        for (int k = 0; k < K; ++k) {
            if (keys[k] == m) t.key = k;
            if (keys[k] < m) t.left = k;
            if (keys[k] > m && t.right < 0) t.right = k;
        }
        tg[align && t.key < 0 && t.left >= 0 && t.right >= 0 ? 1 : 0].push_back(t);
    }
    const size_t mark = ex.ar.off;
    for (int pass = 0; pass < 2; ++pass) {
        Nvtx nv(ex.dry, "interpolation pass %d", pass);
        fb_match_cfg cfg = cfg0;
        cfg.loss = pass == 1 ? FB_LOSS_PAIRWISE : FB_LOSS_GUIDE_STYLE;
        std::vector<int> cost;
        for (const Tgt& t : tg[pass]) cost.push_back(t.key >= 0 ? 0 : (t.left >= 0) + (t.right >= 0));
        // with tracking every frame of a pass is coupled to its neighbours (D42): one batch per pass
        int cap = batch_pairs(ex.ctx, g, cfg.loss);
        if (cfg0.tracking) {
            long long total = 0;
            for (int c : cost) total += c;
            if (total > kMaxBatchPairs) throw Fail{FB_ERR_UNSUPPORTED, "tracking needs all pairs of a key span in one batch"};
            cap = (int)std::max<long long>(cap, total);
        }
        for (auto [b0, b1] : make_batches(cost, cap)) {
            ex.ar.off = mark;
            std::vector<TaskSpec> tasks;
            std::vector<int> tl(b1 - b0, -1), tr(b1 - b0, -1);
            for (int q = b0; q < b1; ++q) {
                const Tgt& t = tg[pass][q];
                if (t.key >= 0) continue;
                if (t.left >= 0) {
                    tl[q - b0] = (int)tasks.size();
                    tasks.push_back(TaskSpec{KSl.slot(t.left), KS.frame(t.left), G.frame(t.m - t0), -1,
                                             (uint32_t)keys[t.left], (uint32_t)t.m, 5u});
                }
                if (t.right >= 0) {
                    tr[q - b0] = (int)tasks.size();
                    tasks.push_back(TaskSpec{KSl.slot(t.right), KS.frame(t.right), G.frame(t.m - t0), -1,
                                             (uint32_t)keys[t.right], (uint32_t)t.m, 5u});
                }
                if (pass == 1) {  // counterparts (Eq. 10)
                    tasks[tl[q - b0]].partner = tr[q - b0];
                    tasks[tr[q - b0]].partner = tl[q - b0];
                }
            }
            if (cfg0.tracking) {  // D42: same keyframe, targets m-1 / m+1 (tasks of this pass)
                std::map<std::pair<uint32_t, uint32_t>, int> by;  // (key frame id, target id) -> task
                for (int t = 0; t < (int)tasks.size(); ++t) by[{tasks[t].src_id, tasks[t].tgt_id}] = t;
                for (auto& tk : tasks) {
                    auto p = by.find({tk.src_id, tk.tgt_id - 1});
                    auto n = by.find({tk.src_id, tk.tgt_id + 1});
                    tk.track[0] = p != by.end() ? p->second : -1;
                    tk.track[1] = n != by.end() ? n->second : -1;
                }
            }
            BatchOut bo;
            if (!tasks.empty()) bo = run_nnf(ex, cfg, g, KSl, tasks, {}, st);
            CombineList cl;
            for (int q = b0; q < b1; ++q) {
                const Tgt& t = tg[pass][q];
                cl.begin();
                if (t.key >= 0) {
                    cl.add_img(KS.frame(t.key), 1.0f);  // keyframes are not modified
                } else if (t.left < 0 || t.right < 0) {
                    const int k = t.left >= 0 ? t.left : t.right;
                    cl.add_remap(KS.frame(k), t.left >= 0 ? tl[q - b0] : tr[q - b0], 1.0f, KSl, k);
                } else {
                    const int l = keys[t.left], r = keys[t.right], m = t.m;
                    const float wl = (float)(r - m) / (float)(r - l), wr = (float)(m - l) / (float)(r - l);
                    cl.add_remap(KS.frame(t.right), tr[q - b0], wr, KSl, t.right);  // A = X_r w_r, fma(X_l, w_l, A)
                    cl.add_remap(KS.frame(t.left), tl[q - b0], wl, KSl, t.left);
                }
                cl.end(out + 3LL * n0 * (t.m - t0), 1, 1.0f);
            }
            if (st) st->remap_pixels += (uint64_t)tasks.size() * n0;
            run_combine(ex, g, 0, cl, bo.F, bo.fstride);
        }
    }
}

// ------------------------------------------------------------------------------------ NNF API
void nnf_api(Exec& ex, const fb_match_cfg& cfg, const Geo& g, int B, const uint8_t* sg, const uint8_t* tg,
             const uint8_t* ss, const uint8_t* ts, const int32_t* group, const fb_pair_key* keys, int32_t* nnf_out,
             float* err_out, float* rem_out, fb_stats* st)
{
    const Pyr SG = pyramid_u8(ex, g, sg, B), TG = pyramid_u8(ex, g, tg, B);
    Pyr SS, TS;
    if (cfg.loss != FB_LOSS_BASE) SS = pyramid_u8(ex, g, ss, B);
    if (cfg.loss == FB_LOSS_MEAN_ALIGN) TS = pyramid_u8(ex, g, ts, B);
    const long long np = g.npx0();
    std::vector<SlotSpec> specs;
    for (int b = 0; b < B; ++b)
        specs.push_back(SlotSpec{sg + 3 * np * b, cfg.loss != FB_LOSS_BASE ? ss + 3 * np * b : nullptr, SG.frame(b),
                                 cfg.loss != FB_LOSS_BASE ? SS.frame(b) : nullptr});
    const Slots SL = pack_sources(ex, g, (cfg.loss == FB_LOSS_PAIRWISE && g.p > 2) ? fbk::SF32 : fbk::SF8, specs);
    std::vector<TaskSpec> tasks;
    std::vector<GroupSpec> groups;
    std::map<int32_t, int> gidx;
    for (int b = 0; b < B; ++b) {
        int gi = -1;
        if (cfg.loss == FB_LOSS_MEAN_ALIGN) {
            auto it = gidx.find(group[b]);
            if (it == gidx.end()) {
                gi = (int)groups.size();
                gidx[group[b]] = gi;
                groups.push_back(GroupSpec{TS.frame(b), TG.frame(b), (uint32_t)keys[b].tgt_id});
            } else {
                gi = it->second;
                if (groups[gi].tgt_id != (uint32_t)keys[b].tgt_id)
                    throw Fail{FB_ERR_INVALID_ARG, "pairs of one MEAN_ALIGN group must share tgt_id"};
            }
        }
        tasks.push_back(TaskSpec{SL.slot(b), cfg.loss != FB_LOSS_BASE ? SS.frame(b) : nullptr, TG.frame(b), gi,
                                 (uint32_t)keys[b].src_id, (uint32_t)keys[b].tgt_id, (uint32_t)keys[b].task_tag});
        if (cfg.loss == FB_LOSS_PAIRWISE) {
            if (group[b] < 0 || group[b] >= B || group[group[b]] != b || group[b] == b)
                throw Fail{FB_ERR_INVALID_ARG, "PAIRWISE: group[b] must name a distinct counterpart pair (mutual)"};
            tasks.back().partner = group[b];
        }
    }
    BatchOut bo = run_nnf(ex, cfg, g, SL, tasks, groups, st, err_out != nullptr);
    const long long n0 = g.npx0();
    ex.d2d(nnf_out, bo.F, sizeof(int2) * (size_t)B * n0);
    if (err_out) ex.d2d(err_out, bo.E, sizeof(float) * (size_t)B * n0);
    if (rem_out) {
        if (cfg.loss == FB_LOSS_BASE) throw Fail{FB_ERR_INVALID_ARG, "remapped_out needs src_style (loss != BASE)"};
        CombineList cl;
        for (int b = 0; b < B; ++b) {
            cl.begin();
            cl.add_remap(SS.frame(b), b, 1.0f);
            cl.end(rem_out + 3LL * n0 * b, 1, 1.0f);
        }
        if (st) st->remap_pixels += (uint64_t)B * n0;
        run_combine(ex, g, 0, cl, bo.F, bo.fstride);
    }
}

// Runs `body` twice: dry (to size the workspace) then for real.
template <class Body>
fb_status guarded(fb_ctx ctx, fb_stats* stats, Body&& body, size_t* need_only = nullptr)
{
    if (!ctx) return FB_ERR_INVALID_ARG;
    try {
        Exec dry{ctx, true, Arena{}};
        fb_stats tmp{};
        body(dry, &tmp);
        if (need_only) { *need_only = dry.ar.peak; return FB_OK; }
        if (dry.ar.peak > 0 && (!ctx->ws || ctx->ws_bytes < dry.ar.peak)) {
            char buf[160];
            snprintf(buf, sizeof buf, "workspace too small: need %zu bytes, have %zu", dry.ar.peak, ctx->ws_bytes);
            throw Fail{FB_ERR_WORKSPACE, buf};
        }
        cudaError_t e = cudaSetDevice(ctx->device);
        if (e != cudaSuccess) throw Fail{FB_ERR_CUDA, cudaGetErrorString(e)};
        e = cudaGetLastError();  // surface a pending fault from earlier work
        if (e != cudaSuccess) throw Fail{FB_ERR_CUDA, std::string("pending: ") + cudaGetErrorString(e)};
        Exec run{ctx, false, Arena{ctx->ws}};
        fb_stats st{};
        body(run, &st);
        if (stats) *stats = st;
        ctx->err.clear();
        return FB_OK;
    } catch (const Fail& f) {
        ctx->err = f.msg;
        return f.st;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return FB_ERR_INVALID_ARG;
    }
}

void check_frames(int N, int H, int W)
{
    if (N < 1 || H < 1 || W < 1) throw Fail{FB_ERR_INVALID_ARG, "N, H, W must be >= 1"};
}

}  // namespace

// ==================================================================================== C ABI
extern "C" {

fb_status fb_ctx_create(int device, void* cuda_stream, fb_ctx* out)
{
    if (!out) return FB_ERR_INVALID_ARG;
    *out = nullptr;
    if (cudaSetDevice(device) != cudaSuccess) return FB_ERR_CUDA;
    fb_ctx c = new fb_ctx_s;
    c->device = device;
    c->stream = static_cast<cudaStream_t>(cuda_stream);
    *out = c;
    return FB_OK;
}

void fb_ctx_destroy(fb_ctx ctx) { delete ctx; }

const char* fb_last_error(fb_ctx ctx) { return ctx ? ctx->err.c_str() : "null context"; }

fb_status fb_set_workspace(fb_ctx ctx, void* dev_ptr, size_t bytes)
{
    if (!ctx || (!dev_ptr && bytes)) return FB_ERR_INVALID_ARG;
    ctx->ws = static_cast<char*>(dev_ptr);
    ctx->ws_bytes = bytes;
    return FB_OK;
}

fb_status fb_set_max_batch_pairs(fb_ctx ctx, int64_t max_pairs)
{
    if (!ctx || max_pairs < 0) return FB_ERR_INVALID_ARG;
    ctx->max_pairs = max_pairs;
    return FB_OK;
}

fb_status fb_set_option(fb_ctx ctx, int option, int value)
{
    if (!ctx) return FB_ERR_INVALID_ARG;
    switch (option) {
    case FB_OPT_FUSED_ITER: ctx->fused = value != 0; break;
    case FB_OPT_FUSE13: ctx->fuse13 = value != 0; break;
    case FB_OPT_PHASE0_MID: ctx->phase0_mid = value != 0; break;
    case FB_OPT_L1_FAST:
        if (value < 0 || value > 2) { ctx->err = "l1_fast must be 0, 1 or 2"; return FB_ERR_INVALID_ARG; }
        ctx->l1_fast = value;
        break;
    case FB_OPT_SUM_BOUND: ctx->sum_bound = value != 0; break;
    case FB_OPT_P3_FUSED: ctx->p3_fused = value != 0; break;
    case FB_OPT_TAIL_BOUND: ctx->tail_bound = value != 0; break;
    case FB_OPT_TGT_REG_ROWS:
        if (value < 0 || value > 3) { ctx->err = "tgt_reg_rows must be 0 (all), 1, 2 or 3 (none)"; return FB_ERR_INVALID_ARG; }
        ctx->tgt_reg_rows = value;
        break;
    default: ctx->err = "unknown option"; return FB_ERR_INVALID_ARG;
    }
    return FB_OK;
}

uint64_t fb_launch_count(fb_ctx ctx) { return ctx ? ctx->launches : 0; }

fb_status fb_profile_enable(fb_ctx ctx, int on)
{
    if (!ctx) return FB_ERR_INVALID_ARG;
    ctx->prof = on != 0;
    return FB_OK;
}

int fb_profile_read(fb_ctx ctx, fb_profile_entry* out, int cap)
{
    if (!ctx) return 0;
    ctx->drain();
    const int n = (int)ctx->totals.size();
    for (int i = 0; i < n && i < cap && out; ++i) out[i] = ctx->totals[i];
    return n;
}

void fb_profile_reset(fb_ctx ctx)
{
    if (!ctx) return;
    ctx->drain();
    for (auto& e : ctx->totals) { e.launches = 0; e.ms = 0; e.work = 0; }
}

size_t fb_pyramid_elems(int B, int H, int W, int levels)
{
    if (B < 0 || H < 1 || W < 1 || levels < 1) return 0;
    size_t n = 0;
    for (int k = 0; k < levels; ++k) n += (size_t)(H >> k) * (size_t)(W >> k);
    return 4 * n * (size_t)B;
}

fb_status fb_build_pyramid(fb_ctx ctx, const uint8_t* frames, int B, int H, int W, int levels, float* out)
{
    return guarded(ctx, nullptr, [&](Exec& ex, fb_stats*) {
        if (!frames || !out || B < 1 || H < 1 || W < 1 || levels < 1 || levels > 20)
            throw Fail{FB_ERR_INVALID_ARG, "bad pyramid arguments"};
        if (std::min(H >> (levels - 1), W >> (levels - 1)) < 1) throw Fail{FB_ERR_SHAPE, "too many levels"};
        Geo g;
        g.H = H; g.W = W; g.Lv = levels;
        long long off = 0;
        for (int k = 0; k < levels; ++k) { g.L[k] = Lvl{H >> k, W >> k, off}; off += (long long)(H >> k) * (W >> k); }
        g.pyr_texels = off;
        float4* base = reinterpret_cast<float4*>(out);
        ex.launch("pyr0", [&] { return fbk::launch_u8_to_pyr0(frames, base, B, H, W, off, ex.ctx->stream); });
        pyramid_levels_inplace(ex, g, base, B, off);
    });
}

fb_status fb_remap(fb_ctx ctx, int B, int H, int W, int p, const float* src, const int32_t* nnf, float* out)
{
    return guarded(ctx, nullptr, [&](Exec& ex, fb_stats*) {
        if (!src || !nnf || !out || B < 0 || H < 1 || W < 1 || p < 1) throw Fail{FB_ERR_INVALID_ARG, "bad remap arguments"};
        if (p > 4) throw Fail{FB_ERR_UNSUPPORTED, "patch_radius > 4 is not compiled"};
        if (B == 0) return;
        ex.launch("remap", [&] { return fbk::launch_remap_f3(src, reinterpret_cast<const int2*>(nnf), out, B, H, W, p,
                                                             ex.ctx->stream); });
    });
}

static void validate_nnf(const fb_match_cfg* cfg, int B, int H, int W, const uint8_t* sg, const uint8_t* tg,
                         const uint8_t* ss, const uint8_t* ts, const int32_t* group, const fb_pair_key* keys,
                         const int32_t* nnf_out)
{
    validate_cfg(cfg);
    if (B < 1 || H < 1 || W < 1) throw Fail{FB_ERR_INVALID_ARG, "B, H, W must be >= 1"};
    if (B > kMaxBatchPairs) throw Fail{FB_ERR_INVALID_ARG, "B exceeds 65535 pairs per call"};
    if (!sg || !tg || !keys || !nnf_out) throw Fail{FB_ERR_INVALID_ARG, "NULL required pointer"};
    if (cfg->loss != FB_LOSS_BASE && !ss) throw Fail{FB_ERR_INVALID_ARG, "src_style required for this loss"};
    if (cfg->loss == FB_LOSS_MEAN_ALIGN && (!ts || !group)) throw Fail{FB_ERR_INVALID_ARG, "MEAN_ALIGN needs tgt_style and group"};
    if (cfg->loss == FB_LOSS_PAIRWISE && !group) throw Fail{FB_ERR_INVALID_ARG, "PAIRWISE needs group (counterparts)"};
    for (int b = 0; b < B; ++b)
        if (keys[b].src_id < 0 || keys[b].tgt_id < 0 || keys[b].tgt_id >= (1 << 28) || keys[b].task_tag < 0 ||
            keys[b].task_tag > 15)
            throw Fail{FB_ERR_INVALID_ARG, "pair key out of range"};
}

fb_status fb_nnf_estimate(fb_ctx ctx, const fb_match_cfg* cfg, int B, int H, int W, const uint8_t* src_guide,
                          const uint8_t* tgt_guide, const uint8_t* src_style, const uint8_t* tgt_style,
                          const int32_t* group, const fb_pair_key* pair_keys, int32_t* nnf_out, float* err_out,
                          float* remapped_out, fb_stats* stats)
{
    return guarded(ctx, stats, [&](Exec& ex, fb_stats* st) {
        validate_nnf(cfg, B, H, W, src_guide, tgt_guide, src_style, tgt_style, group, pair_keys, nnf_out);
        const Geo g = make_geo(*cfg, H, W);
        nnf_api(ex, *cfg, g, B, src_guide, tgt_guide, src_style, tgt_style, group, pair_keys, nnf_out, err_out,
                remapped_out, st);
    });
}

static void blend_range_body(Exec& ex, fb_stats* st, const fb_match_cfg* cfg, int schedule, int N_total, int f0,
                             int N, int H, int W, int M, const uint8_t* guide, const uint8_t* style, int t0, int t1,
                             float* out)
{
    validate_cfg(cfg);
    check_frames(N_total, H, W);
    if (M < 0) throw Fail{FB_ERR_INVALID_ARG, "M < 0"};
    if (schedule != FB_SCHED_DIRECT && schedule != FB_SCHED_TREE) throw Fail{FB_ERR_INVALID_ARG, "unknown schedule"};
    if (schedule == FB_SCHED_TREE && cfg->loss == FB_LOSS_MEAN_ALIGN)
        throw Fail{FB_ERR_UNSUPPORTED, "accurate mode (MEAN_ALIGN) is defined only for the direct schedule (P:249)"};
    if (cfg->loss == FB_LOSS_BASE || cfg->loss == FB_LOSS_PAIRWISE)
        throw Fail{FB_ERR_INVALID_ARG, "blending needs GUIDE_STYLE or MEAN_ALIGN"};
    if (!guide || !style || !out) throw Fail{FB_ERR_INVALID_ARG, "NULL required pointer"};
    if (t0 < 0 || t1 > N_total || t0 >= t1) throw Fail{FB_ERR_INVALID_ARG, "bad target range"};
    if (f0 < 0 || N < 1 || f0 + N > N_total || f0 > std::max(0, t0 - M) || f0 + N < std::min(N_total, t1 + M))
        throw Fail{FB_ERR_INVALID_ARG, "local frames must cover the targets plus a halo of M"};
    if (cfg->tracking && schedule == FB_SCHED_TREE)
        throw Fail{FB_ERR_UNSUPPORTED, "tracking in blending is defined for the direct schedule (D44)"};
    if (cfg->tracking && (t0 > 0 || t1 < N_total))
        throw Fail{FB_ERR_UNSUPPORTED, "tracking couples every pair of the schedule (D44): use the full call"};
    const Geo g = make_geo(*cfg, H, W);
    if (schedule == FB_SCHED_DIRECT) blend_direct(ex, *cfg, g, N_total, f0, N, M, guide, style, t0, t1, out, st);
    else blend_tree(ex, *cfg, g, N_total, f0, N, M, guide, style, t0, t1, out, st);
}

fb_status fb_blend_window_range(fb_ctx ctx, const fb_match_cfg* cfg, int schedule, int N_total, int f0, int N,
                                int H, int W, int M, const uint8_t* guide, const uint8_t* style, int t0, int t1,
                                float* out, fb_stats* stats)
{
    return guarded(ctx, stats, [&](Exec& ex, fb_stats* st) {
        blend_range_body(ex, st, cfg, schedule, N_total, f0, N, H, W, M, guide, style, t0, t1, out);
    });
}

size_t fb_tree_cell_texels(const fb_match_cfg* cfg, int H, int W)
{
    try {
        if (!cfg) return 0;
        validate_cfg(cfg);
        return (size_t)make_geo(*cfg, H, W).pyr_texels;
    } catch (...) {
        return 0;
    }
}

static void tree_common_checks(const fb_match_cfg* cfg, int N_total, int f0, int N, int H, int W,
                               const uint8_t* guide, const uint8_t* style, int n_cells, const int32_t* cells)
{
    validate_cfg(cfg);
    check_frames(N_total, H, W);
    if (cfg->loss != FB_LOSS_GUIDE_STYLE) throw Fail{FB_ERR_INVALID_ARG, "the tree schedule uses GUIDE_STYLE"};
    if (!guide || !style) throw Fail{FB_ERR_INVALID_ARG, "NULL frames"};
    if (f0 < 0 || N < 1 || f0 + N > N_total) throw Fail{FB_ERR_INVALID_ARG, "bad local frame range"};
    if (n_cells < 0 || (n_cells > 0 && !cells)) throw Fail{FB_ERR_INVALID_ARG, "bad cell list"};
    for (int c = 0; c < n_cells; ++c) {
        const int o = cells[3 * c], j = cells[3 * c + 1], L = cells[3 * c + 2];
        if ((o != 0 && o != 1) || j < 0 || j >= N_total || L < 1 || L > 30 || j - (1 << L) + 1 < 0)
            throw Fail{FB_ERR_INVALID_ARG, "bad cell {orient, j, L}"};
    }
}

fb_status fb_tree_build_cells(fb_ctx ctx, const fb_match_cfg* cfg, int N_total, int f0, int N, int H, int W,
                              const uint8_t* guide, const uint8_t* style, int n_cells, const int32_t* cells,
                              float* cell_out, fb_stats* stats, size_t* ws_needed)
{
    return guarded(ctx, stats, [&](Exec& ex, fb_stats* st) {
        tree_common_checks(cfg, N_total, f0, N, H, W, guide, style, n_cells, cells);
        if (n_cells > 0 && !cell_out && !ex.dry) throw Fail{FB_ERR_INVALID_ARG, "NULL cell_out"};
        for (int c = 0; c < n_cells; ++c) {  // every frame a cell reads is local
            const int o = cells[3 * c], j = cells[3 * c + 1], L = cells[3 * c + 2];
            const int a = j - (1 << L) + 1, b = j;
            const int lo = o == 0 ? a : N_total - 1 - b, hi = o == 0 ? b : N_total - 1 - a;
            if (lo < f0 || hi >= f0 + N) throw Fail{FB_ERR_INVALID_ARG, "a cell reads frames outside the local range"};
        }
        const Geo g = make_geo(*cfg, H, W);
        tree_build_cells(ex, *cfg, g, N_total, f0, N, guide, style, n_cells, cells, cell_out, st);
    }, ws_needed);
}

fb_status fb_tree_query(fb_ctx ctx, const fb_match_cfg* cfg, int N_total, int f0, int N, int H, int W, int M,
                        const uint8_t* guide, const uint8_t* style, int t0, int t1, int n_cells,
                        const int32_t* cells, const float* const* cell_ptrs, float* out, fb_stats* stats,
                        size_t* ws_needed)
{
    return guarded(ctx, stats, [&](Exec& ex, fb_stats* st) {
        tree_common_checks(cfg, N_total, f0, N, H, W, guide, style, n_cells, cells);
        if (M < 0) throw Fail{FB_ERR_INVALID_ARG, "M < 0"};
        if (t0 < 0 || t1 > N_total || t0 >= t1) throw Fail{FB_ERR_INVALID_ARG, "bad target range"};
        if (f0 > std::max(0, t0 - M) || f0 + N < std::min(N_total, t1 + M))
            throw Fail{FB_ERR_INVALID_ARG, "local frames must cover the targets plus a halo of M"};
        if (!ex.dry && (!out || (n_cells > 0 && !cell_ptrs))) throw Fail{FB_ERR_INVALID_ARG, "NULL pointer"};
        const Geo g = make_geo(*cfg, H, W);
        tree_query_cells(ex, *cfg, g, N_total, f0, N, M, guide, style, t0, t1, n_cells, cells, cell_ptrs, out, st);
    }, ws_needed);
}

fb_status fb_blend_window(fb_ctx ctx, const fb_match_cfg* cfg, int schedule, int N, int H, int W, int M,
                          const uint8_t* guide, const uint8_t* style, float* out, fb_stats* stats)
{
    return fb_blend_window_range(ctx, cfg, schedule, N, 0, N, H, W, M, guide, style, 0, N, out, stats);
}

fb_status fb_interpolate_keyframes(fb_ctx ctx, const fb_match_cfg* cfg, int N, int H, int W, const uint8_t* guide,
                                   int K, const int32_t* key_index, const uint8_t* key_style, float* out,
                                   fb_stats* stats)
{
    return guarded(ctx, stats, [&](Exec& ex, fb_stats* st) {
        validate_cfg(cfg);
        check_frames(N, H, W);
        if (!guide || !key_index || !key_style || !out || K < 1) throw Fail{FB_ERR_INVALID_ARG, "NULL pointer or K < 1"};
        for (int k = 0; k < K; ++k)
            if (key_index[k] < 0 || key_index[k] >= N || (k && key_index[k] <= key_index[k - 1]))
                throw Fail{FB_ERR_INVALID_ARG, "key_index must be strictly increasing in [0, N)"};
        const Geo g = make_geo(*cfg, H, W);
        interpolate(ex, *cfg, g, N, 0, N, guide, K, key_index, nullptr, key_style, out, st);
    });
}

fb_status fb_interpolate_keyframes_range(fb_ctx ctx, const fb_match_cfg* cfg, int N, int H, int W, int t0, int t1,
                                         const uint8_t* guide, int K, const int32_t* key_index,
                                         const uint8_t* key_guide, const uint8_t* key_style, float* out,
                                         fb_stats* stats, size_t* ws_needed)
{
    return guarded(ctx, stats, [&](Exec& ex, fb_stats* st) {
        validate_cfg(cfg);
        check_frames(N, H, W);
        if (!guide || !key_index || !key_guide || !key_style || (!out && !ex.dry) || K < 1)
            throw Fail{FB_ERR_INVALID_ARG, "NULL pointer or K < 1"};
        if (t0 < 0 || t1 > N || t0 >= t1) throw Fail{FB_ERR_INVALID_ARG, "bad target range"};
        for (int k = 0; k < K; ++k)
            if (key_index[k] < 0 || key_index[k] >= N || (k && key_index[k] <= key_index[k - 1]))
                throw Fail{FB_ERR_INVALID_ARG, "key_index must be strictly increasing in [0, N)"};
        if (cfg->tracking && (t0 > 0 || t1 < N))
            throw Fail{FB_ERR_UNSUPPORTED, "tracking couples every frame of a key span (D42): use the full call"};
        const Geo g = make_geo(*cfg, H, W);
        interpolate(ex, *cfg, g, N, t0, t1, guide, K, key_index, key_guide, key_style, out, st);
    }, ws_needed);
}

size_t fb_workspace_size_range(fb_ctx ctx, int schedule, const fb_match_cfg* cfg, int N_total, int f0, int N, int H,
                               int W, int M, int t0, int t1)
{
    if (!ctx || !cfg) return 0;
    size_t need = 0;
    const uint8_t* fake = reinterpret_cast<const uint8_t*>(16);  // dry run: pointers are never dereferenced
    float* fout = reinterpret_cast<float*>(16);
    std::string saved = ctx->err;
    const fb_status s = guarded(ctx, nullptr, [&](Exec& ex, fb_stats* st) {
        blend_range_body(ex, st, cfg, schedule, N_total, f0, N, H, W, M, fake, fake, t0, t1, fout);
    }, &need);
    ctx->err = saved;
    return s == FB_OK ? std::max<size_t>(need, 256) : 0;
}

size_t fb_workspace_size(fb_ctx ctx, int op, const fb_match_cfg* cfg, int n, int H, int W, int M)
{
    if (!ctx || !cfg || n < 1 || H < 1 || W < 1) return 0;
    size_t need = 0;
    const uint8_t* fake = reinterpret_cast<const uint8_t*>(16);  // dry run: pointers are never dereferenced
    float* fout = reinterpret_cast<float*>(16);
    std::string saved = ctx->err;
    fb_status s = FB_OK;
    if (op == FB_OP_NNF) {
        // worst case: every MEAN_ALIGN pair its own group (one packed T-bar target per group)
        std::vector<fb_pair_key> keys(n, fb_pair_key{0, 0, 6});
        std::vector<int32_t> grp(n, 0);
        for (int b = 0; b < n; ++b) {
            grp[b] = cfg->loss == FB_LOSS_PAIRWISE ? ((b ^ 1) < n ? (b ^ 1) : b) : b;
            keys[b].tgt_id = b;
        }
        s = guarded(ctx, nullptr, [&](Exec& ex, fb_stats* st) {
            validate_cfg(cfg);
            const Geo g = make_geo(*cfg, H, W);
            nnf_api(ex, *cfg, g, n, fake, fake, fake, fake, grp.data(), keys.data(),
                    reinterpret_cast<int32_t*>(16), fout, cfg->loss == FB_LOSS_BASE ? nullptr : fout, st);
        }, &need);
    } else if (op == FB_OP_BLEND_DIRECT || op == FB_OP_BLEND_TREE) {
        s = guarded(ctx, nullptr, [&](Exec& ex, fb_stats* st) {
            blend_range_body(ex, st, cfg, op == FB_OP_BLEND_TREE ? FB_SCHED_TREE : FB_SCHED_DIRECT, n, 0, n, H, W, M,
                             fake, fake, 0, n, fout);
        }, &need);
    } else if (op == FB_OP_INTERPOLATE) {
        // upper bound: every non-key frame has two keys; the key placement does not change the size
        std::vector<int32_t> keys;
        const int K = std::max(1, std::min(M, n));
        for (int k = 0; k < K; ++k) keys.push_back((int)((long long)k * (n - 1) / std::max(1, K - 1)));
        keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
        s = guarded(ctx, nullptr, [&](Exec& ex, fb_stats* st) {
            validate_cfg(cfg);
            const Geo g = make_geo(*cfg, H, W);
            interpolate(ex, *cfg, g, n, 0, n, fake, (int)keys.size(), keys.data(), nullptr, fake, fout, st);
        }, &need);
    } else {
        return 0;
    }
    ctx->err = saved;
    return s == FB_OK ? std::max<size_t>(need, 256) : 0;
}

}  // extern "C"
