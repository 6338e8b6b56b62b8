/*
 * fb_oracle.c — CPU ORACLE for FastBlend's data-parallel hot path (arXiv 2311.09265).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or helper with the
 * CUDA product path (paper_2311_09265_b200/csrc); the two meet only at seeded inputs.
 *
 * This is a plain, slow, obviously-correct transcription of the paper's method, step by step, in
 * the paper's order and notation.  Citations "P:n" are lines of PAPER.md; "Dn" are the readings in
 * DESIGN.md §3 (the ambiguity ledger inherited from SURVEY.md §8(c)).
 *
 * Arithmetic contract (D5/D20): IEEE FP32, round-to-nearest-even, compiled with
 * -ffp-contract=off and no fast-math.  Images are floats in 8-bit units (0..255).  The only fused
 * operations are the explicit fmaf() calls written below.  Summation orders are the ones written
 * in the loops; nothing is blocked, fused or reordered.
 *
 * Parity pins: every function here is pinned by tests/test_oracle_*.py against closed forms,
 * library routines, brute force or invariants.  The only "parity unpinned" item is
 * the quality of the accurate/fast modes on real content (P14), which has no closed form.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------------------------------
 * Configuration (mirrors the meaning of fb_match_cfg in include/fb.h but is declared separately:
 * the oracle includes no product header).
 * ---------------------------------------------------------------------------------------------- */
typedef struct {
    int32_t patch_radius;    /* p: a patch is (2p+1)^2 pixels                          */
    int32_t levels;          /* pyramid levels, 0 = auto (D6, D32)                            */
    int32_t iters_per_level; /* n in Alg. 1                                            */
    int32_t rs_radius0;      /* initial random-search radius, 0 = max(h_k, w_k) (D13, D33)  */
    int32_t rs_steps;        /* random-search steps, 0 = until radius < 1 (D13, D33)          */
    float alpha;             /* guide weight alpha (Eq. 3; Eq. 8)               */
    int32_t loss;            /* 0 BASE (Eq. 1), 1 GUIDE_STYLE (Eq. 3), 2 MEAN_ALIGN (Eq. 8), 3 PAIRWISE (Eq. 10) */
    int32_t init;            /* 0 random, 1 identity (D8)                              */
    uint64_t seed;           /* Philox key (D21)                                              */
    int32_t prop_scales;     /* J propagation scales, steps 2^(J-1)..1 (jump flood, D41); 0/1 = P:72 */
    int32_t tracking;        /* interpolation: NNF(S,T_{i-1}), NNF(S,T_{i+1}) as candidates (D42) */
} orc_cfg;

enum { ORC_BASE = 0, ORC_GUIDE_STYLE = 1, ORC_MEAN_ALIGN = 2, ORC_PAIRWISE = 3 };
enum { ORC_TAG_DIRECT = 0, ORC_TAG_TREE_BUILD_F = 1, ORC_TAG_TREE_QUERY_F = 2,
       ORC_TAG_TREE_BUILD_R = 3, ORC_TAG_TREE_QUERY_R = 4, ORC_TAG_INTERP = 5 };

/* ------------------------------------------------------------------------------------------------
 * Philox4x32-10 (Salmon et al. 2011), the counter-based generator of D21.  Pinned by the Random123
 * known-answer vectors in tests/golden/philox_kat.txt.
 * ---------------------------------------------------------------------------------------------- */
static inline uint32_t mulhi32(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) >> 32); }

void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint32_t p0 = 0xD2511F53u, p1 = 0xCD9E8D57u;
        uint32_t hi0 = mulhi32(p0, c0), lo0 = p0 * c0;
        uint32_t hi1 = mulhi32(p1, c2), lo1 = p1 * c2;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* The counter layout of D21: c0 = pixel, c1 = purpose|level|iteration|step, c2 = source frame id,
 * c3 = task tag|target frame id.  Purpose 0 = initialisation, 1 = random search. */
static void orc_draw(uint64_t seed, uint32_t pixel, uint32_t purpose, uint32_t level, uint32_t iter,
                     uint32_t step, uint32_t src_id, uint32_t tag, uint32_t tgt_id, uint32_t out[4])
{
    uint32_t key[2] = { (uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32) };
    uint32_t ctr[4] = { pixel, (purpose << 28) | (level << 22) | (iter << 12) | step, src_id,
                        (tag << 28) | tgt_id };
    orc_philox4x32_10(ctr, key, out);
}

/* ------------------------------------------------------------------------------------------------
 * Pyramid (Alg. 1 "Resize images S, T"; reading D6): level k is the 2x2 box mean of
 * level k-1 with floor dimensions; P_k(r,c) = ((a+b)+(d+e)) * 0.25.
 * ---------------------------------------------------------------------------------------------- */
int orc_level_count(int H, int W, int p, int requested)
{
    int mn = H < W ? H : W;
    if (mn < 2 * p + 1) return -1;
    if (requested > 0) {
        int hk = H >> (requested - 1), wk = W >> (requested - 1);
        if ((hk < wk ? hk : wk) < 2 * p + 1) return -1; /* D32: explicit levels must fit */
        return requested;
    }
    int lv = 1; /* D6: Lv = 1 + max{k : min(H,W) >> k >= 32} */
    for (int k = 1; k < 30; ++k)
        if ((mn >> k) >= 32) lv = k + 1;
    while (lv > 1 && (mn >> (lv - 1)) < 2 * p + 1) --lv; /* D32 */
    return lv;
}

static size_t level_offset(int H, int W, int k) /* in pixels */
{
    size_t off = 0;
    for (int i = 0; i < k; ++i) off += (size_t)(H >> i) * (size_t)(W >> i);
    return off;
}

size_t orc_pyramid_pixels(int H, int W, int levels) { return level_offset(H, W, levels); }

/* img0: [H,W,3] float; out: all levels packed level-major, each [h_k, w_k, 3]. */
void orc_pyramid(const float* img0, int H, int W, int levels, float* out)
{
    memcpy(out, img0, sizeof(float) * 3 * (size_t)H * W);
    for (int k = 1; k < levels; ++k) {
        const float* prev = out + 3 * level_offset(H, W, k - 1);
        float* cur = out + 3 * level_offset(H, W, k);
        int hp = H >> (k - 1), wp = W >> (k - 1), hk = H >> k, wk = W >> k;
        (void)hp;
        for (int r = 0; r < hk; ++r)
            for (int c = 0; c < wk; ++c)
                for (int ch = 0; ch < 3; ++ch) {
                    float a = prev[3 * ((size_t)(2 * r) * wp + 2 * c) + ch];
                    float b = prev[3 * ((size_t)(2 * r) * wp + 2 * c + 1) + ch];
                    float d = prev[3 * ((size_t)(2 * r + 1) * wp + 2 * c) + ch];
                    float e = prev[3 * ((size_t)(2 * r + 1) * wp + 2 * c + 1) + ch];
                    cur[3 * ((size_t)r * wk + c) + ch] = ((a + b) + (d + e)) * 0.25f;
                }
    }
}

/* ------------------------------------------------------------------------------------------------
 * Patch distance (Eq. 1): ||S[F(x,y)] - T[x,y]||^2 over the (2p+1)^2 patch.
 * Order (D20): for each dr a row partial rho = fma(delta, delta, rho) over dc then channel, then
 * D = D + rho with rows in increasing dr.  Pixels outside the image read 0 (D9).
 * ---------------------------------------------------------------------------------------------- */
static inline float px(const float* I, int h, int w, int r, int c, int ch)
{
    if (r < 0 || r >= h || c < 0 || c >= w) return 0.0f;
    return I[3 * ((size_t)r * w + c) + ch];
}

float orc_patch_dist(const float* A, const float* B, int h, int w, int sr, int sc, int r, int c, int p)
{
    float D = 0.0f;
    for (int dr = -p; dr <= p; ++dr) {
        float rho = 0.0f;
        for (int dc = -p; dc <= p; ++dc)
            for (int ch = 0; ch < 3; ++ch) {
                float delta = px(B, h, w, r + dr, c + dc, ch) - px(A, h, w, sr + dr, sc + dc, ch);
                rho = fmaf(delta, delta, rho);
            }
        D = D + rho;
    }
    return D;
}

/* ------------------------------------------------------------------------------------------------
 * Remap, Alg. 2 with the valid-tap average of P:101 (reading D19):
 * T^(x,y) = (sum over valid (dx,dy), increasing dx then dy, of S(F(x+dx,y+dy) - (dx,dy))) / n_valid.
 * F is int32 [h,w,2] holding (row, col) of the source patch centre.
 * ---------------------------------------------------------------------------------------------- */
void orc_remap(const float* S, int h, int w, const int32_t* F, int p, float* out)
{
#pragma omp parallel for schedule(static)
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            float acc[3] = { 0.0f, 0.0f, 0.0f };
            int n = 0;
            for (int dr = -p; dr <= p; ++dr)
                for (int dc = -p; dc <= p; ++dc) {
                    int tr = r + dr, tc = c + dc;
                    if (tr < 0 || tr >= h || tc < 0 || tc >= w) continue;
                    int sr = F[2 * ((size_t)tr * w + tc)] - dr;
                    int sc = F[2 * ((size_t)tr * w + tc) + 1] - dc;
                    if (sr < 0 || sr >= h || sc < 0 || sc >= w) continue;
                    for (int ch = 0; ch < 3; ++ch) acc[ch] = acc[ch] + S[3 * ((size_t)sr * w + sc) + ch];
                    ++n;
                }
            for (int ch = 0; ch < 3; ++ch) out[3 * ((size_t)r * w + c) + ch] = acc[ch] / (float)n;
        }
}

/* ------------------------------------------------------------------------------------------------
 * One NNF estimation task set (Alg. 1), run in lockstep so that MEAN_ALIGN groups can
 * share their average remapped image T-bar (Eq. 7; reading D27).
 * ---------------------------------------------------------------------------------------------- */
typedef struct {
    int src_guide, tgt_guide, src_style, tgt_style; /* indices into the frame stack (-1 = none) */
    int group;                                       /* MEAN_ALIGN window id                     */
    int src_id, tgt_id, tag;                         /* RNG key (D21)                            */
    int partner;                                     /* PAIRWISE: the counterpart task (D38)     */
    int track_prev, track_next;                      /* tracking neighbours (tasks for T_{i-1}, T_{i+1}), -1 */
} orc_task;

typedef struct {
    int h, w;        /* level dims */
    size_t off;      /* level offset in pixels */
} lvl_t;

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* random-search radius schedule at level k ("r declines exponentially to zero"; D13, D33) */
static int rs_count(const orc_cfg* cfg, int hk, int wk)
{
    int r0 = cfg->rs_radius0 > 0 ? cfg->rs_radius0 : (hk > wk ? hk : wk);
    if (cfg->rs_steps > 0) return cfg->rs_steps;
    int n = 0;
    while ((r0 >> n) >= 1) ++n;
    return n;
}
static int rs_radius(const orc_cfg* cfg, int hk, int wk, int s)
{
    int r0 = cfg->rs_radius0 > 0 ? cfg->rs_radius0 : (hk > wk ? hk : wk);
    int R = r0 >> s;
    return R < 1 ? 1 : R;
}

/* D41: number of propagation scales (1 = the paper's unit-step propagation) */
static int prop_scales(const orc_cfg* cfg) { return cfg->prop_scales > 1 ? cfg->prop_scales : 1; }

uint64_t orc_evals_per_task(const orc_cfg* cfg, int H, int W)
{
    int lv = orc_level_count(H, W, cfg->patch_radius, cfg->levels);
    if (lv < 1) return 0;
    uint64_t n = 0;
    for (int k = 0; k < lv; ++k) {
        int hk = H >> k, wk = W >> k;
        n += (uint64_t)hk * wk * cfg->iters_per_level * (uint64_t)(1 + 4 * prop_scales(cfg) + rs_count(cfg, hk, wk));
    }
    return n;
}

/* Everything the loss of one task needs at one pyramid level. */
typedef struct {
    int h, w, p, loss;
    float alpha;
    const float *sg, *tg, *ss, *aux; /* source guide, target guide, source style, aux (S^ or T-bar) */
    const float* pss;                /* PAIRWISE: counterpart's source style (the other keyframe)   */
    const int32_t* pF;               /* PAIRWISE: counterpart's NNF at the start of the iteration   */
} orc_level_ctx;

/* The loss L(S', T', F)(x,y) of a candidate (sr, sc) for target pixel (r, c):
 * BASE = Eq. 1; GUIDE_STYLE = Eq. 3, alpha*D(G_src,G_tgt) + D(S_src, S^);
 * MEAN_ALIGN = Eq. 8 (reading D27), alpha*D(G_src,G_tgt) + D(S_src, T-bar);
 * PAIRWISE = Eq. 10 (reading D38/D39), alpha*D(G_src,G_tgt) + ||S_l[F_l(x)] - S_r[F_r(x)]||^2:
 * the second term compares the candidate's patch of this task's keyframe style with the patch of
 * the counterpart keyframe's style at the counterpart's NNF (frozen at the iteration start). */
static float level_loss(const orc_level_ctx* L, int r, int c, int sr, int sc)
{
    float dg = orc_patch_dist(L->sg, L->tg, L->h, L->w, sr, sc, r, c, L->p);
    if (L->loss == ORC_BASE) return dg;
    float ds;
    if (L->loss == ORC_PAIRWISE) {
        const int32_t* q = L->pF + 2 * ((size_t)r * L->w + c);
        ds = orc_patch_dist(L->ss, L->pss, L->h, L->w, sr, sc, q[0], q[1], L->p);
    } else {
        ds = orc_patch_dist(L->ss, L->aux, L->h, L->w, sr, sc, r, c, L->p);
    }
    return fmaf(L->alpha, dg, ds);
}

/* One element of Alg. 1's loop body at one level.
 *   field = -1: E <- L(F)
 *   field = 0..3: propagation F'(x,y) = F(x+dx, y+dy) - (dx,dy) with (dx,dy) = (-1,0),(1,0),(0,-1),(0,1)
 *                 (P:72), neighbour index clamped (D11), candidate clamped to the source (D10);
 *                 Jacobi: every pixel reads the F of the previous field.  With a jump-flood
 *                 step s (D41) the neighbour is x + s*d and the candidate F(x + s*d) - s*d.
 *   field = 4+s: random search step s: F'(x,y) = F(x,y) + (dx,dy), dx,dy uniform integers in [-R_s, R_s]
 *                 with R_s = r0 >> s (D13) from the Philox stream of D21
 * followed by the strict-min select F(E'<E) <- F'(E'<E), E(E'<E) <- E'(E'<E).
 * F, E are updated in place; Fo/Eo are scratch of the same size. */
static const int PROP_DIRS[4][2] = { { -1, 0 }, { 1, 0 }, { 0, -1 }, { 0, 1 } };

static void level_field(const orc_level_ctx* L, const orc_cfg* cfg, int field, int step, int k, int it, int src_id,
                        int tgt_id, int tag, int32_t* F, float* E, int32_t* Fo, float* Eo)
{
    int h = L->h, w = L->w;
    size_t n = (size_t)h * w;
    if (field < 0) {
#pragma omp parallel for schedule(static)
        for (int r = 0; r < h; ++r)
            for (int c = 0; c < w; ++c) {
                size_t i = (size_t)r * w + c;
                E[i] = level_loss(L, r, c, F[2 * i], F[2 * i + 1]);
            }
        return;
    }
    if (field < 4) {
        int dx = step * PROP_DIRS[field][0], dy = step * PROP_DIRS[field][1];
#pragma omp parallel for schedule(static)
        for (int r = 0; r < h; ++r)
            for (int c = 0; c < w; ++c) {
                size_t i = (size_t)r * w + c;
                int nr = clampi(r + dx, 0, h - 1), nc = clampi(c + dy, 0, w - 1);
                size_t j = (size_t)nr * w + nc;
                int sr = clampi(F[2 * j] - dx, 0, h - 1), sc = clampi(F[2 * j + 1] - dy, 0, w - 1);
                float e = level_loss(L, r, c, sr, sc);
                if (e < E[i]) { Fo[2 * i] = sr; Fo[2 * i + 1] = sc; Eo[i] = e; }
                else { Fo[2 * i] = F[2 * i]; Fo[2 * i + 1] = F[2 * i + 1]; Eo[i] = E[i]; }
            }
        memcpy(F, Fo, sizeof(int32_t) * 2 * n);
        memcpy(E, Eo, sizeof(float) * n);
        return;
    }
    int s = field - 4, R = rs_radius(cfg, h, w, s);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            size_t i = (size_t)r * w + c;
            /* D21: one Philox block per two steps (counter step field s >> 1); step s uses words 0, 1 when even,
             * 2, 3 when odd */
            uint32_t u[4];
            orc_draw(cfg->seed, (uint32_t)i, 1, (uint32_t)k, (uint32_t)it, (uint32_t)(s >> 1), (uint32_t)src_id,
                     (uint32_t)tag, (uint32_t)tgt_id, u);
            int ox = (int)mulhi32(u[2 * (s & 1)], (uint32_t)(2 * R + 1)) - R;
            int oy = (int)mulhi32(u[2 * (s & 1) + 1], (uint32_t)(2 * R + 1)) - R;
            int sr = clampi(F[2 * i] + ox, 0, h - 1), sc = clampi(F[2 * i + 1] + oy, 0, w - 1);
            float e = level_loss(L, r, c, sr, sc);
            if (e < E[i]) { F[2 * i] = sr; F[2 * i + 1] = sc; E[i] = e; } /* pointwise: in place is Jacobi */
        }
}

/* Tracking field (D42): the whole field of a neighbouring frame's NNF (frozen at the start
 * of the iteration) as the candidate, F'(x) = G(x), followed by the strict-min select. */
static void level_track_field(const orc_level_ctx* L, const int32_t* G, int32_t* F, float* E)
{
    int h = L->h, w = L->w;
#pragma omp parallel for schedule(static)
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            size_t i = (size_t)r * w + c;
            int sr = G[2 * i], sc = G[2 * i + 1];
            float e = level_loss(L, r, c, sr, sc);
            if (e < E[i]) { F[2 * i] = sr; F[2 * i + 1] = sc; E[i] = e; } /* pointwise: in place is Jacobi */
        }
}

/* Tracking-field entry for the pins: one level, explicit candidate field G. */
void orc_track_field(const orc_cfg* cfg, int h, int w, const float* sg, const float* tg, const float* ss,
                     const float* aux, const int32_t* G, int32_t* F, float* E)
{
    orc_level_ctx L = { h, w, cfg->patch_radius, cfg->loss, cfg->alpha, sg, tg, ss, aux, NULL, NULL };
    level_track_field(&L, G, F, E);
}

/* Single-field entry for the pins (tests/test_oracle_pins.py): one level, explicit F/E/aux. */
void orc_field(const orc_cfg* cfg, int h, int w, const float* sg, const float* tg, const float* ss,
               const float* aux, int field, int k, int it, int src_id, int tgt_id, int tag, int32_t* F, float* E)
{
    orc_level_ctx L = { h, w, cfg->patch_radius, cfg->loss, cfg->alpha, sg, tg, ss, aux, NULL, NULL };
    int32_t* Fo = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)h * w);
    float* Eo = (float*)malloc(sizeof(float) * (size_t)h * w);
    level_field(&L, cfg, field, 1, k, it, src_id, tgt_id, tag, F, E, Fo, Eo);
    free(Fo); free(Eo);
}

/* Same with a propagation step (jump flood, D41). */
void orc_field_step(const orc_cfg* cfg, int h, int w, const float* sg, const float* tg, const float* ss,
                    const float* aux, int field, int step, int k, int it, int src_id, int tgt_id, int tag,
                    int32_t* F, float* E)
{
    orc_level_ctx L = { h, w, cfg->patch_radius, cfg->loss, cfg->alpha, sg, tg, ss, aux, NULL, NULL };
    int32_t* Fo = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)h * w);
    float* Eo = (float*)malloc(sizeof(float) * (size_t)h * w);
    level_field(&L, cfg, field, step, k, it, src_id, tgt_id, tag, F, E, Fo, Eo);
    free(Fo); free(Eo);
}

typedef struct {
    const orc_cfg* cfg;
    int T, H, W, lv;
    const orc_task* tasks;
    float** pyr_sg; float** pyr_tg; float** pyr_ss; float** pyr_ts; /* per task pyramids */
    float** aux;     /* per task aux at current level [h_k, w_k, 3] */
    int32_t** F; float** E;
    int32_t** Fn; float** En;
    int32_t** Fsnap;  /* PAIRWISE: every task's NNF at the start of the current iteration (D39) */
    lvl_t L[32];
} orc_state;

static int cmp_int_pair(const void* a, const void* b)
{
    const int* x = (const int*)a; const int* y = (const int*)b;
    return (x[0] > y[0]) - (x[0] < y[0]);
}

/* Aux refresh "once at the beginning of each iteration" (D17/D18/D27). */
static void refresh_aux(orc_state* st, int k)
{
    const orc_cfg* cfg = st->cfg;
    int h = st->L[k].h, w = st->L[k].w, p = cfg->patch_radius;
    size_t npx = (size_t)h * w;
    if (cfg->loss == ORC_PAIRWISE || cfg->tracking) {
        /* counterpart (D39) and tracking (D42) NNFs are frozen at the start of the iteration */
        for (int t = 0; t < st->T; ++t) memcpy(st->Fsnap[t], st->F[t], sizeof(int32_t) * 2 * npx);
    }
    if (cfg->loss == ORC_GUIDE_STYLE) {
        /* S^_i = remap of the task's source style with the current F at this level (D18) */
        for (int t = 0; t < st->T; ++t)
            orc_remap(st->pyr_ss[t] + 3 * st->L[k].off, h, w, st->F[t], p, st->aux[t]);
    } else if (cfg->loss == ORC_MEAN_ALIGN) {
        /* T-bar_i = (sum over j in W_i ascending of Y_j) / |W_i|, Y_i = S_i, Y_j = (S_j -> T)
         * (Eq. 7; D27).  Pairs sharing a group id form one window. */
        float** rem = (float**)malloc(sizeof(float*) * st->T);
        for (int t = 0; t < st->T; ++t) {
            rem[t] = (float*)malloc(sizeof(float) * 3 * npx);
            orc_remap(st->pyr_ss[t] + 3 * st->L[k].off, h, w, st->F[t], p, rem[t]);
        }
        int* done = (int*)calloc(st->T, sizeof(int));
        int* members = (int*)malloc(sizeof(int) * 2 * (st->T + 1));
        float* mean = (float*)malloc(sizeof(float) * 3 * npx);
        for (int t = 0; t < st->T; ++t) {
            if (done[t]) continue;
            int g = st->tasks[t].group, nm = 0;
            for (int u = 0; u < st->T; ++u)
                if (st->tasks[u].group == g) { members[2 * nm] = st->tasks[u].src_id; members[2 * nm + 1] = u; ++nm; done[u] = 1; }
            members[2 * nm] = st->tasks[t].tgt_id; members[2 * nm + 1] = -1; ++nm; /* self: Y_i = S_i */
            qsort(members, nm, 2 * sizeof(int), cmp_int_pair);
            const float* self = st->pyr_ts[t] + 3 * st->L[k].off;
            for (size_t i = 0; i < 3 * npx; ++i) {
                float a = 0.0f;
                for (int m = 0; m < nm; ++m) {
                    int u = members[2 * m + 1];
                    a = a + (u < 0 ? self[i] : rem[u][i]);
                }
                mean[i] = a / (float)nm;
            }
            for (int u = 0; u < st->T; ++u)
                if (st->tasks[u].group == g) memcpy(st->aux[u], mean, sizeof(float) * 3 * npx);
        }
        for (int t = 0; t < st->T; ++t) free(rem[t]);
        free(rem); free(done); free(members); free(mean);
    }
}

/* Alg. 1 loop body for one task at level k, iteration it, after the aux refresh:
 * E <- L(F), the four propagation fields, then the K_k random-search fields. */
static void iterate_task(orc_state* st, int t, int k, int it, uint64_t* evals)
{
    const orc_cfg* cfg = st->cfg;
    const orc_task* tk = &st->tasks[t];
    size_t off = 3 * st->L[k].off;
    orc_level_ctx L = { st->L[k].h, st->L[k].w, cfg->patch_radius, cfg->loss, cfg->alpha,
                        st->pyr_sg[t] + off, st->pyr_tg[t] + off, st->pyr_ss[t] ? st->pyr_ss[t] + off : NULL,
                        st->aux[t], NULL, NULL };
    if (cfg->loss == ORC_PAIRWISE) {
        L.pss = st->pyr_ss[tk->partner] + off;
        L.pF = st->Fsnap[tk->partner];
    }
    int K = rs_count(cfg, L.h, L.w);
    /* E <- L(F); propagation at every scale (descending steps, D41; one unit-step scale = P:72); then
     * the K random-search fields */
    const int J = prop_scales(cfg);
    level_field(&L, cfg, -1, 1, k, it, tk->src_id, tk->tgt_id, tk->tag, st->F[t], st->E[t], st->Fn[t], st->En[t]);
    *evals += (uint64_t)L.h * L.w;
    for (int j = J - 1; j >= 0; --j)
        for (int d = 0; d < 4; ++d) {
            level_field(&L, cfg, d, 1 << j, k, it, tk->src_id, tk->tgt_id, tk->tag, st->F[t], st->E[t], st->Fn[t],
                        st->En[t]);
            *evals += (uint64_t)L.h * L.w;
        }
    if (cfg->tracking) /* tracking candidates T_{i-1} then T_{i+1} (D42) */
        for (int z = 0; z < 2; ++z) {
            int nb = z == 0 ? tk->track_prev : tk->track_next;
            if (nb < 0) continue;
            level_track_field(&L, st->Fsnap[nb], st->F[t], st->E[t]);
            *evals += (uint64_t)L.h * L.w;
        }
    for (int field = 4; field < 4 + K; ++field) {
        level_field(&L, cfg, field, 1, k, it, tk->src_id, tk->tgt_id, tk->tag, st->F[t], st->E[t], st->Fn[t],
                    st->En[t]);
        *evals += (uint64_t)L.h * L.w;
    }
}

/* "Upsample F" (Alg. 1; reading D7): the coarse field Fc [hc, wc, 2] (level k+1) to the fine grid
 * [h, w, 2] (level k, h = 2hc or 2hc+1):
 *   F_f(r,c) = clamp(2 F_c(rc,cc) + (r - 2rc, c - 2cc)),  rc = min(r>>1, hc-1),  cc = min(c>>1, wc-1),
 * clamped to [0,h-1] x [0,w-1] (D10).  The last odd row / column reuses the last coarse cell. */
void orc_upsample(const int32_t* Fc, int hc, int wc, int32_t* Ff, int h, int w)
{
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            int rc = (r >> 1) < hc - 1 ? (r >> 1) : hc - 1;
            int cc = (c >> 1) < wc - 1 ? (c >> 1) : wc - 1;
            size_t j = (size_t)rc * wc + cc, i = (size_t)r * w + c;
            Ff[2 * i] = clampi(2 * Fc[2 * j] + (r - 2 * rc), 0, h - 1);
            Ff[2 * i + 1] = clampi(2 * Fc[2 * j + 1] + (c - 2 * cc), 0, w - 1);
        }
}

/* frames: stack [NF, H, W, 3] float (8-bit units).  Outputs per task (nullable):
 * F_out int32 [T,H,W,2], E_out float [T,H,W], X_out float [T,H,W,3] = remap of src style (Alg. 2). */
int orc_nnf(const orc_cfg* cfg, int T, int H, int W, const float* frames, const orc_task* tasks,
            int32_t* F_out, float* E_out, float* X_out, uint64_t* evals_out)
{
    orc_state st;
    memset(&st, 0, sizeof(st));
    st.cfg = cfg; st.T = T; st.H = H; st.W = W; st.tasks = tasks;
    st.lv = orc_level_count(H, W, cfg->patch_radius, cfg->levels);
    if (st.lv < 1) return -1;
    if (cfg->loss == ORC_PAIRWISE)  /* every task needs a counterpart with a source style */
        for (int t = 0; t < T; ++t)
            if (tasks[t].partner < 0 || tasks[t].partner >= T || tasks[t].src_style < 0 ||
                tasks[tasks[t].partner].src_style < 0)
                return -2;
    size_t npx0 = (size_t)H * W, pyr = orc_pyramid_pixels(H, W, st.lv);
    for (int k = 0; k < st.lv; ++k) { st.L[k].h = H >> k; st.L[k].w = W >> k; st.L[k].off = level_offset(H, W, k); }
    st.pyr_sg = (float**)calloc(T, sizeof(float*)); st.pyr_tg = (float**)calloc(T, sizeof(float*));
    st.pyr_ss = (float**)calloc(T, sizeof(float*)); st.pyr_ts = (float**)calloc(T, sizeof(float*));
    st.aux = (float**)calloc(T, sizeof(float*));
    st.F = (int32_t**)calloc(T, sizeof(int32_t*)); st.E = (float**)calloc(T, sizeof(float*));
    st.Fsnap = (int32_t**)calloc(T, sizeof(int32_t*));
    st.Fn = (int32_t**)calloc(T, sizeof(int32_t*)); st.En = (float**)calloc(T, sizeof(float*));
#pragma omp parallel for schedule(static)
    for (int t = 0; t < T; ++t) {
        const orc_task* tk = &tasks[t];
        st.pyr_sg[t] = (float*)malloc(sizeof(float) * 3 * pyr);
        st.pyr_tg[t] = (float*)malloc(sizeof(float) * 3 * pyr);
        orc_pyramid(frames + 3 * npx0 * tk->src_guide, H, W, st.lv, st.pyr_sg[t]);
        orc_pyramid(frames + 3 * npx0 * tk->tgt_guide, H, W, st.lv, st.pyr_tg[t]);
        if (tk->src_style >= 0) {
            st.pyr_ss[t] = (float*)malloc(sizeof(float) * 3 * pyr);
            orc_pyramid(frames + 3 * npx0 * tk->src_style, H, W, st.lv, st.pyr_ss[t]);
        }
        if (tk->tgt_style >= 0) {
            st.pyr_ts[t] = (float*)malloc(sizeof(float) * 3 * pyr);
            orc_pyramid(frames + 3 * npx0 * tk->tgt_style, H, W, st.lv, st.pyr_ts[t]);
        }
        st.aux[t] = (float*)malloc(sizeof(float) * 3 * npx0);
        st.F[t] = (int32_t*)malloc(sizeof(int32_t) * 2 * npx0); st.E[t] = (float*)malloc(sizeof(float) * npx0);
        st.Fn[t] = (int32_t*)malloc(sizeof(int32_t) * 2 * npx0); st.En[t] = (float*)malloc(sizeof(float) * npx0);
        st.Fsnap[t] = (int32_t*)malloc(sizeof(int32_t) * 2 * npx0);
    }
    uint64_t evals = 0;
    int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * 2 * npx0);
    for (int k = st.lv - 1; k >= 0; --k) {
        int h = st.L[k].h, w = st.L[k].w;
        for (int t = 0; t < T; ++t) {
            int32_t* F = st.F[t];
            if (k == st.lv - 1) {
                /* "Randomly initialize F" (D8), or identity (D33) */
                for (int r = 0; r < h; ++r)
                    for (int c = 0; c < w; ++c) {
                        size_t i = (size_t)r * w + c;
                        if (cfg->init == 1) { F[2 * i] = r; F[2 * i + 1] = c; continue; }
                        uint32_t u[4];
                        orc_draw(cfg->seed, (uint32_t)i, 0, (uint32_t)k, 0, 0, (uint32_t)tasks[t].src_id,
                                 (uint32_t)tasks[t].tag, (uint32_t)tasks[t].tgt_id, u);
                        F[2 * i] = (int32_t)mulhi32(u[0], (uint32_t)h);
                        F[2 * i + 1] = (int32_t)mulhi32(u[1], (uint32_t)w);
                    }
            } else {
                int hc = st.L[k + 1].h, wc = st.L[k + 1].w;
                memcpy(tmp, F, sizeof(int32_t) * 2 * (size_t)hc * wc);
                orc_upsample(tmp, hc, wc, F, h, w);
            }
        }
        for (int it = 0; it < cfg->iters_per_level; ++it) {
            refresh_aux(&st, k);
            uint64_t ev = 0;
            for (int t = 0; t < T; ++t) iterate_task(&st, t, k, it, &ev); /* rows run in parallel inside */
            evals += ev;
        }
    }
    for (int t = 0; t < T; ++t) {
        if (F_out) memcpy(F_out + 2 * npx0 * t, st.F[t], sizeof(int32_t) * 2 * npx0);
        if (E_out) memcpy(E_out + npx0 * t, st.E[t], sizeof(float) * npx0);
        if (X_out && st.pyr_ss[t]) orc_remap(st.pyr_ss[t], H, W, st.F[t], cfg->patch_radius, X_out + 3 * npx0 * t);
    }
    for (int t = 0; t < T; ++t) {
        free(st.pyr_sg[t]); free(st.pyr_tg[t]); free(st.pyr_ss[t]); free(st.pyr_ts[t]); free(st.aux[t]);
        free(st.F[t]); free(st.E[t]); free(st.Fn[t]); free(st.En[t]); free(st.Fsnap[t]);
    }
    free(st.pyr_sg); free(st.pyr_tg); free(st.pyr_ss); free(st.pyr_ts); free(st.aux);
    free(st.F); free(st.E); free(st.Fn); free(st.En); free(st.Fsnap); free(tmp);
    if (evals_out) *evals_out = evals;
    return 0;
}

/* ------------------------------------------------------------------------------------------------
 * Schedules.  Every function computes the outputs of the requested target frames only (with their
 * full dependency closure), so that full-size parity can be sampled.
 * ---------------------------------------------------------------------------------------------- */
static void u8_to_float(const uint8_t* src, size_t n, float* dst)
{
    for (size_t i = 0; i < n; ++i) dst[i] = (float)src[i];
}

/* Sliding-window blend, direct O(N*M) schedule: balanced (Eq. 2 + Eq. 3) or accurate
 * (Eq. 7/8).  W_i = [max(0,i-M), min(N-1,i+M)] (D3); X_{i->i} = S_i (D4);
 * out_i = (sum over j ascending of X_{j->i}) / |W_i|; X_{j->i} = remap of S_j with NNF(G_j, G_i). */
int orc_blend_direct(const orc_cfg* cfg, int N, int H, int W, int M, const uint8_t* guide,
                     const uint8_t* style, int n_targets, const int32_t* targets, float* out,
                     uint64_t* pairs_out, uint64_t* evals_out)
{
    size_t npx = (size_t)H * W;
    float* frames = (float*)malloc(sizeof(float) * 3 * npx * 2 * (size_t)N); /* [G_0..G_N-1, S_0..S_N-1] */
    u8_to_float(guide, 3 * npx * N, frames);
    u8_to_float(style, 3 * npx * N, frames + 3 * npx * N);
    /* Tracking in blending ("optional setting", reading D44): NNF(G_j, G_i) also tries the same source's
     * NNFs for the neighbouring targets, NNF(G_j, G_{i-1}) and NNF(G_j, G_{i+1}) when those pairs exist, frozen at
     * the start of each iteration (D42).  Every pair is then coupled to its neighbours, so all targets' pairs
     * are estimated together and the requested targets are read out of that run. */
    int nt = cfg->tracking ? N : n_targets;
    int32_t* tl = (int32_t*)malloc(sizeof(int32_t) * (nt > 0 ? nt : 1));
    for (int q = 0; q < nt; ++q) tl[q] = cfg->tracking ? q : targets[q];
    int maxT = 0;
    for (int q = 0; q < nt; ++q) maxT += 2 * M;
    orc_task* tasks = (orc_task*)malloc(sizeof(orc_task) * (maxT + 1));
    int* first = (int*)malloc(sizeof(int) * (nt + 1));
    int T = 0;
    for (int q = 0; q < nt; ++q) {
        int i = tl[q], lo = i - M < 0 ? 0 : i - M, hi = i + M > N - 1 ? N - 1 : i + M;
        first[q] = T;
        for (int j = lo; j <= hi; ++j) {
            if (j == i) continue;
            orc_task tk = { j, i, N + j, cfg->loss == ORC_MEAN_ALIGN ? N + i : -1, q, j, i, ORC_TAG_DIRECT, -1, -1, -1 };
            tasks[T++] = tk;
        }
    }
    if (cfg->tracking) /* tl = 0..N-1: the task (j, i') sits in target i''s list */
        for (int a = 0; a < T; ++a)
            for (int z = 0; z < 2; ++z) {
                int i2 = tasks[a].tgt_id + (z == 0 ? -1 : 1), j = tasks[a].src_id;
                if (i2 < 0 || i2 >= N || i2 == j) continue;
                for (int b = first[i2]; b < (i2 + 1 < nt ? first[i2 + 1] : T); ++b)
                    if (tasks[b].src_id == j) { if (z == 0) tasks[a].track_prev = b; else tasks[a].track_next = b; }
            }
    float* X = (float*)malloc(sizeof(float) * 3 * npx * (T > 0 ? T : 1));
    uint64_t evals = 0;
    if (T > 0 && orc_nnf(cfg, T, H, W, frames, tasks, NULL, NULL, X, &evals) != 0) {
        free(frames); free(tasks); free(X); free(tl); free(first); return -1;
    }
    for (int q = 0; q < n_targets; ++q) {
        int i = targets[q], lo = i - M < 0 ? 0 : i - M, hi = i + M > N - 1 ? N - 1 : i + M;
        int t0 = first[cfg->tracking ? i : q];
        float* o = out + 3 * npx * q;
        for (size_t e = 0; e < 3 * npx; ++e) {
            float a = 0.0f;
            int tt = t0;
            for (int j = lo; j <= hi; ++j) {
                if (j == i) a = a + frames[3 * npx * (N + i) + e];
                else a = a + X[3 * npx * (tt++) + e];
            }
            o[e] = a / (float)(hi - lo + 1);
        }
    }
    if (pairs_out) *pairs_out = (uint64_t)T;
    if (evals_out) *evals_out = evals;
    free(frames); free(tasks); free(X); free(tl); free(first);
    return 0;
}

/* ---- Fast mode: remapping table (Alg. 3), blending table (Alg. 4), query (Alg. 5), Eq. 6 ----
 * Tables are built in "orientation" coordinates: forward (v = orig) and the symmetric table on the
 * reversed order (v = N-1-orig) (reading D26).  Cells store means (D25):
 *   RT(j,L), L>=1: frames [j-2^L+1, j-2^(L-1)] remapped into j, summed ascending, / 2^(L-1);
 *   BT(j,0) = S_j, BT(j,L) = (BT(j,L-1) + RT(j,L)) * 0.5.
 * Only levels L <= floor(log2(M+1)) are built (D24); queried cells never need more. */

/* Alg. 5 with the decrement i <- i - 2^L (reading D23): the visited (node, level)
 * pairs of query(l, r), in visit order.  Returns the count. */
int orc_tree_query_nodes(int l, int r, int32_t* nodes, int32_t* levels)
{
    int n = 0, i = r;
    while (i >= l) {
        int L = 0;
        while ((i & (1 << L)) && i - (1 << (L + 1)) + 1 >= l) ++L;
        nodes[n] = i; levels[n] = L; ++n;
        i -= (1 << L);
    }
    return n;
}

/* Alg. 3 task enumeration with the level cap: for every i and every zero bit L of i
 * (L+1 <= lcap), j <- j | 2^L and, if j < N, task (i -> j) feeds RT(j, L+1).  Writes (i, j, L+1). */
int orc_tree_build_tasks(int N, int lcap, int32_t* src, int32_t* dst, int32_t* cell_level)
{
    int n = 0;
    for (int i = 0; i < N; ++i) {
        int j = i;
        for (int L = 0; L + 1 <= lcap; ++L) {
            if (i & (1 << L)) continue;
            j |= (1 << L);
            if (j < N) {
                if (src) { src[n] = i; dst[n] = j; cell_level[n] = L + 1; }
                ++n;
            }
        }
    }
    return n;
}

static int floor_log2(int x) { int l = 0; while ((2 << l) <= x) ++l; return l; }

typedef struct { int N, lcap; float** bt; } orc_table; /* bt[j*(lcap+1)+L], NULL if not built */

/* Builds the blending-table cells needed by the queries of the requested targets (orientation o).
 * frames layout as in orc_blend_direct; cells are float [H,W,3]. */
static int build_table_needed(const orc_cfg* cfg, int N, int H, int W, int M, int orient,
                              const float* frames, int n_targets, const int32_t* targets,
                              orc_table* tab, uint64_t* pairs, uint64_t* evals)
{
    size_t npx = (size_t)H * W;
    int lcap = floor_log2(M + 1);
    tab->N = N; tab->lcap = lcap;
    tab->bt = (float**)calloc((size_t)N * (lcap + 1), sizeof(float*));
    /* which cells (j, L) are needed: all (node, L) visited by the queries, plus their prefixes */
    char* need = (char*)calloc((size_t)N * (lcap + 1), 1);
    int32_t* nodes = (int32_t*)malloc(sizeof(int32_t) * 64);
    int32_t* lvls = (int32_t*)malloc(sizeof(int32_t) * 64);
    for (int q = 0; q < n_targets; ++q) {
        int v = orient == 0 ? targets[q] : N - 1 - targets[q];
        int l = v - M < 0 ? 0 : v - M;
        int nn = orc_tree_query_nodes(l, v, nodes, lvls);
        for (int a = 0; a < nn; ++a)
            for (int L = 1; L <= lvls[a]; ++L) need[(size_t)nodes[a] * (lcap + 1) + L] = 1;
    }
    /* Alg. 3 tasks restricted to the needed RT cells */
    int nb = orc_tree_build_tasks(N, lcap, NULL, NULL, NULL);
    int32_t* bs = (int32_t*)malloc(sizeof(int32_t) * (nb + 1));
    int32_t* bd = (int32_t*)malloc(sizeof(int32_t) * (nb + 1));
    int32_t* bl = (int32_t*)malloc(sizeof(int32_t) * (nb + 1));
    orc_tree_build_tasks(N, lcap, bs, bd, bl);
    orc_task* tasks = (orc_task*)malloc(sizeof(orc_task) * (nb + 1));
    int32_t* tcell = (int32_t*)malloc(sizeof(int32_t) * (nb + 1));
    int T = 0;
    for (int a = 0; a < nb; ++a) {
        if (!need[(size_t)bd[a] * (lcap + 1) + bl[a]]) continue;
        int oi = orient == 0 ? bs[a] : N - 1 - bs[a], oj = orient == 0 ? bd[a] : N - 1 - bd[a];
        orc_task tk = { oi, oj, N + oi, -1, 0, oi, oj, orient == 0 ? ORC_TAG_TREE_BUILD_F : ORC_TAG_TREE_BUILD_R, -1, -1, -1 };
        tasks[T] = tk; tcell[T] = a; ++T;
    }
    float* X = (float*)malloc(sizeof(float) * 3 * npx * (T > 0 ? T : 1));
    uint64_t ev = 0;
    if (T > 0) {
        orc_cfg c2 = *cfg; c2.loss = ORC_GUIDE_STYLE; /* D22: loss on the frame being remapped */
        if (orc_nnf(&c2, T, H, W, frames, tasks, NULL, NULL, X, &ev) != 0) return -1;
    }
    *pairs += (uint64_t)T; *evals += ev;
    /* RT(j,L) = (sum ascending i of X_{i->j}) / 2^(L-1); tasks were enumerated by ascending i, so
     * for a fixed cell the contributions appear in ascending i. */
    float** rt = (float**)calloc((size_t)N * (lcap + 1), sizeof(float*));
    for (int t = 0; t < T; ++t) {
        int a = tcell[t];
        size_t cid = (size_t)bd[a] * (lcap + 1) + bl[a];
        if (!rt[cid]) rt[cid] = (float*)calloc(3 * npx, sizeof(float));
        for (size_t e = 0; e < 3 * npx; ++e) rt[cid][e] = rt[cid][e] + X[3 * npx * t + e];
    }
    /* Alg. 4: BT(j,0) = S_j; BT(j,L) = (BT(j,L-1) + RT(j,L)) * 0.5 (means, D25) */
    for (int j = 0; j < N; ++j) {
        int oj = orient == 0 ? j : N - 1 - j;
        int top = 0;
        for (int L = 1; L <= lcap; ++L) if (need[(size_t)j * (lcap + 1) + L]) top = L;
        float* b0 = (float*)malloc(sizeof(float) * 3 * npx);
        memcpy(b0, frames + 3 * npx * (N + oj), sizeof(float) * 3 * npx);
        tab->bt[(size_t)j * (lcap + 1)] = b0;
        for (int L = 1; L <= top; ++L) {
            size_t cid = (size_t)j * (lcap + 1) + L;
            float scale = 1.0f / (float)(1 << (L - 1)); /* exact power of two */
            float* b = (float*)malloc(sizeof(float) * 3 * npx);
            const float* prev = tab->bt[cid - 1];
            for (size_t e = 0; e < 3 * npx; ++e) b[e] = (prev[e] + rt[cid][e] * scale) * 0.5f;
            tab->bt[cid] = b;
        }
    }
    for (size_t c = 0; c < (size_t)N * (lcap + 1); ++c) free(rt[c]);
    free(rt); free(need); free(nodes); free(lvls); free(bs); free(bd); free(bl); free(tasks); free(tcell); free(X);
    return 0;
}

/* Alg. 5 query for target v in orientation o, unnormalised: A = sum over visited nodes of
 * 2^L * (BT(i,L) -> S_r), with A = fma(2^L, X, A) (exact product, one rounding; D25). */
static int query_unnormalised(const orc_cfg* cfg, int N, int H, int W, int M, int orient, const float* frames,
                              const orc_table* tab, int target, float* A, uint64_t* pairs, uint64_t* evals)
{
    size_t npx = (size_t)H * W;
    int v = orient == 0 ? target : N - 1 - target;
    int l = v - M < 0 ? 0 : v - M;
    int32_t nodes[64], lvls[64];
    int nn = orc_tree_query_nodes(l, v, nodes, lvls);
    /* Build a frame stack holding the guides and the queried BT cells as source styles. */
    float* fr = (float*)malloc(sizeof(float) * 3 * npx * ((size_t)N + nn));
    memcpy(fr, frames, sizeof(float) * 3 * npx * N);
    orc_task tasks[64];
    int T = 0, slot_of[64];
    for (int a = 0; a < nn; ++a) {
        slot_of[a] = -1;
        if (nodes[a] == v) continue; /* self node: identity, no NNF (D23) */
        int oi = orient == 0 ? nodes[a] : N - 1 - nodes[a];
        memcpy(fr + 3 * npx * (N + T), tab->bt[(size_t)nodes[a] * (tab->lcap + 1) + lvls[a]], sizeof(float) * 3 * npx);
        orc_task tk = { oi, target, N + T, -1, 0, oi, target, orient == 0 ? ORC_TAG_TREE_QUERY_F : ORC_TAG_TREE_QUERY_R, -1, -1, -1 };
        tasks[T] = tk; slot_of[a] = T; ++T;
    }
    float* X = (float*)malloc(sizeof(float) * 3 * npx * (T > 0 ? T : 1));
    uint64_t ev = 0;
    if (T > 0) {
        orc_cfg c2 = *cfg; c2.loss = ORC_GUIDE_STYLE;
        if (orc_nnf(&c2, T, H, W, fr, tasks, NULL, NULL, X, &ev) != 0) { free(fr); free(X); return -1; }
    }
    *pairs += (uint64_t)T; *evals += ev;
    for (size_t e = 0; e < 3 * npx; ++e) A[e] = 0.0f;
    for (int a = 0; a < nn; ++a) {
        float wgt = (float)(1 << lvls[a]);
        const float* x = slot_of[a] < 0 ? tab->bt[(size_t)nodes[a] * (tab->lcap + 1) + lvls[a]]
                                        : X + 3 * npx * slot_of[a];
        for (size_t e = 0; e < 3 * npx; ++e) A[e] = fmaf(wgt, x[e], A[e]);
    }
    free(fr); free(X);
    return 0;
}

/* Fast blending: Eq. 6: out_i = ((A_fwd + A_rev) - S_i) / |W_i|. */
int orc_blend_tree(const orc_cfg* cfg, int N, int H, int W, int M, const uint8_t* guide, const uint8_t* style,
                   int n_targets, const int32_t* targets, float* out, uint64_t* pairs_out, uint64_t* evals_out)
{
    size_t npx = (size_t)H * W;
    float* frames = (float*)malloc(sizeof(float) * 3 * npx * 2 * (size_t)N);
    u8_to_float(guide, 3 * npx * N, frames);
    u8_to_float(style, 3 * npx * N, frames + 3 * npx * N);
    uint64_t pairs = 0, evals = 0;
    orc_table tab[2];
    for (int o = 0; o < 2; ++o)
        if (build_table_needed(cfg, N, H, W, M, o, frames, n_targets, targets, &tab[o], &pairs, &evals) != 0) return -1;
    float* Af = (float*)malloc(sizeof(float) * 3 * npx);
    float* Ar = (float*)malloc(sizeof(float) * 3 * npx);
    for (int q = 0; q < n_targets; ++q) {
        int i = targets[q];
        if (query_unnormalised(cfg, N, H, W, M, 0, frames, &tab[0], i, Af, &pairs, &evals) != 0) return -1;
        if (query_unnormalised(cfg, N, H, W, M, 1, frames, &tab[1], i, Ar, &pairs, &evals) != 0) return -1;
        int lo = i - M < 0 ? 0 : i - M, hi = i + M > N - 1 ? N - 1 : i + M;
        const float* S = frames + 3 * npx * (N + i);
        float* o = out + 3 * npx * q;
        for (size_t e = 0; e < 3 * npx; ++e) o[e] = ((Af[e] + Ar[e]) - S[e]) / (float)(hi - lo + 1);
    }
    for (int o = 0; o < 2; ++o) {
        for (size_t c = 0; c < (size_t)N * (tab[o].lcap + 1); ++c) free(tab[o].bt[c]);
        free(tab[o].bt);
    }
    free(Af); free(Ar); free(frames);
    if (pairs_out) *pairs_out = pairs;
    if (evals_out) *evals_out = evals;
    return 0;
}

/* Keyframe interpolation, Eq. 9 (reading D28): for l < m < r consecutive keys,
 * out_m = fma(X_l, w_l, X_r * w_r), w_l = (r-m)/(r-l), w_r = (m-l)/(r-l); outside the key span the
 * nearest key's remap; keys verbatim.  X_k = remap of key style with NNF(G_k, G_m).
 * cfg->loss == PAIRWISE selects the alignment of Eq. 10 (D38-D40): the two NNFs of a
 * frame between two keys are estimated jointly, each taking the other (frozen per iteration) in its
 * loss; single-key frames and every other cfg->loss use the guide+style loss of Eq. 3. */
int orc_interpolate(const orc_cfg* cfg, int N, int H, int W, const uint8_t* guide, int K,
                    const int32_t* key_index, const uint8_t* key_style, int n_targets, const int32_t* targets,
                    float* out, uint64_t* pairs_out, uint64_t* evals_out)
{
    size_t npx = (size_t)H * W;
    const int align = cfg->loss == ORC_PAIRWISE;
    float* frames = (float*)malloc(sizeof(float) * 3 * npx * ((size_t)N + K));
    u8_to_float(guide, 3 * npx * N, frames);
    u8_to_float(key_style, 3 * npx * K, frames + 3 * npx * N);
    /* with tracking (D42) every frame's estimation depends on its neighbours', so the closure of any
     * target is the whole video: estimate all frames and output the requested ones */
    int* all = NULL;
    const int n_req = n_targets;
    const int32_t* req = targets;
    if (cfg->tracking) {
        all = (int*)malloc(sizeof(int) * (N > 0 ? N : 1));
        for (int m = 0; m < N; ++m) all[m] = m;
        targets = all;
        n_targets = N;
    }
    /* two task lists: [0] single-key / unaligned (GUIDE_STYLE), [1] aligned pairs (PAIRWISE) */
    orc_task* tl[2];
    int nt[2] = { 0, 0 };
    tl[0] = (orc_task*)malloc(sizeof(orc_task) * (2 * (size_t)n_targets + 1));
    tl[1] = (orc_task*)malloc(sizeof(orc_task) * (2 * (size_t)n_targets + 1));
    int* ta = (int*)malloc(sizeof(int) * 4 * (n_targets + 1)); /* per target: (list, index) of left/right */
    for (int q = 0; q < n_targets; ++q) {
        int m = targets[q], a = -1;
        for (int z = 0; z < 4; ++z) ta[4 * q + z] = -1;
        for (int k = 0; k < K; ++k) if (key_index[k] == m) a = k;
        if (a >= 0) continue; /* key: verbatim */
        int left = -1, right = -1;
        for (int k = 0; k < K; ++k) {
            if (key_index[k] < m) left = k;
            if (key_index[k] > m && right < 0) right = k;
        }
        const int li = (align && left >= 0 && right >= 0) ? 1 : 0;
        if (left >= 0) {
            orc_task tk = { key_index[left], m, N + left, -1, 0, key_index[left], m, ORC_TAG_INTERP, -1, -1, -1 };
            ta[4 * q] = li; ta[4 * q + 1] = nt[li]; tl[li][nt[li]++] = tk;
        }
        if (right >= 0) {
            orc_task tk = { key_index[right], m, N + right, -1, 0, key_index[right], m, ORC_TAG_INTERP, -1, -1, -1 };
            ta[4 * q + 2] = li; ta[4 * q + 3] = nt[li]; tl[li][nt[li]++] = tk;
        }
        if (li == 1) { /* counterparts */
            tl[1][ta[4 * q + 1]].partner = ta[4 * q + 3];
            tl[1][ta[4 * q + 3]].partner = ta[4 * q + 1];
        }
    }
    if (cfg->tracking) /* D42: neighbours = tasks of the same key for targets m-1 and m+1 in the same list */
        for (int z = 0; z < 2; ++z)
            for (int a2 = 0; a2 < nt[z]; ++a2)
                for (int b2 = 0; b2 < nt[z]; ++b2) {
                    if (tl[z][b2].src_id != tl[z][a2].src_id) continue;
                    if (tl[z][b2].tgt_id == tl[z][a2].tgt_id - 1) tl[z][a2].track_prev = b2;
                    if (tl[z][b2].tgt_id == tl[z][a2].tgt_id + 1) tl[z][a2].track_next = b2;
                }
    float* X[2];
    uint64_t evals = 0;
    for (int z = 0; z < 2; ++z) {
        X[z] = (float*)malloc(sizeof(float) * 3 * npx * (nt[z] > 0 ? nt[z] : 1));
        if (nt[z] > 0) {
            orc_cfg c2 = *cfg;
            c2.loss = z == 1 ? ORC_PAIRWISE : ORC_GUIDE_STYLE;
            uint64_t ev = 0;
            if (orc_nnf(&c2, nt[z], H, W, frames, tl[z], NULL, NULL, X[z], &ev) != 0) return -1;
            evals += ev;
        }
    }
    for (int qr = 0; qr < n_req; ++qr) {
        int q = cfg->tracking ? req[qr] : qr;
        int m = targets[q];
        float* o = out + 3 * npx * qr;
        const int hl = ta[4 * q] >= 0, hr = ta[4 * q + 2] >= 0;
        const float* xl = hl ? X[ta[4 * q]] + 3 * npx * ta[4 * q + 1] : NULL;
        const float* xr = hr ? X[ta[4 * q + 2]] + 3 * npx * ta[4 * q + 3] : NULL;
        if (!hl && !hr) { /* key frame */
            int a = 0;
            for (int k = 0; k < K; ++k) if (key_index[k] == m) a = k;
            memcpy(o, frames + 3 * npx * (N + a), sizeof(float) * 3 * npx);
        } else if (!hl || !hr) {
            memcpy(o, hl ? xl : xr, sizeof(float) * 3 * npx);
        } else {
            int l = tl[ta[4 * q]][ta[4 * q + 1]].src_id, r = tl[ta[4 * q + 2]][ta[4 * q + 3]].src_id;
            float wl = (float)(r - m) / (float)(r - l), wr = (float)(m - l) / (float)(r - l);
            for (size_t e = 0; e < 3 * npx; ++e) o[e] = fmaf(xl[e], wl, xr[e] * wr);
        }
    }
    if (pairs_out) *pairs_out = (uint64_t)(nt[0] + nt[1]);
    if (evals_out) *evals_out = evals;
    free(frames); free(tl[0]); free(tl[1]); free(ta); free(X[0]); free(X[1]); free(all);
    return 0;
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
