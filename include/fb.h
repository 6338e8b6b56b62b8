/*
 * fb.h — C ABI of the B200-native FastBlend hot path (arXiv 2311.09265).
 *
 * The library (paper_2311_09265_b200/libfastblend.so) implements, as hand-written sm_100a CUDA
 * kernels, the data-parallel core of the paper: the pyramid PatchMatch NNF estimation of Alg. 1
 * (PAPER.md P:39-76), the memory-efficient remap of Alg. 2, the sliding-window blend of
 * Eq. 2 in its direct O(N*M) form (balanced Eq. 3 and accurate Eq. 7/8) and its
 * tree form (Alg. 3-5 + Eq. 6), and the keyframe interpolation of Eq. 9.
 * The readings of the paper that fix every silent or garbled detail are listed in DESIGN.md §3 and
 * are referred to below as D1..D34.
 *
 * Conventions (all entry points):
 *  - Pointers are DEVICE pointers on the context's device unless the argument says HOST.  The caller
 *    owns every buffer (inputs, outputs and the workspace); the library never allocates device memory
 *    on the hot path and never frees caller memory.
 *  - Every call enqueues work on the context's stream and returns; outputs are valid after the stream
 *    is synchronised.  Device faults surface as FB_ERR_CUDA at the next call.
 *  - Nothing is thrown across the ABI.  A non-OK status leaves a message in fb_last_error(ctx).
 *  - Images at the boundary are uint8 RGB [.., H, W, 3] (row-major, channel-last).  Float images are
 *    in 8-bit units (0..255, D5), [.., H, W, 3].  NNFs are int32 [.., H, W, 2] holding (row, col) of
 *    the matched source patch centre: F(i,j) = (x,y) means T[i,j] matches S[x,y].
 *  - Results are a pure function of (inputs, cfg, pair keys) (D21): batch size, batching, stream and
 *    device never change them.
 */
#ifndef FB_H
#define FB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fb_ctx_s* fb_ctx;

typedef enum {
    FB_OK = 0,
    FB_ERR_INVALID_ARG = 1, /* N<1, M<0, p<1, n<0 or n>1023, rs_steps>4095 (Philox counter fields, D21),
                             * alpha<0, bad enum, NULL required pointer, bad keys,
                             * BASE/PAIRWISE for a window blend, non-mutual PAIRWISE counterparts */
    FB_ERR_SHAPE = 2,       /* min(H,W) < 2p+1, or explicit levels whose coarsest side < 2p+1 (D32)  */
    FB_ERR_CUDA = 3,        /* a CUDA runtime error (message in fb_last_error)                         */
    FB_ERR_NCCL = 4,        /* reserved: the multi-GPU exchange runs on torch.distributed (D43) */
    FB_ERR_WORKSPACE = 5,   /* no workspace set, or smaller than fb_workspace_size() requires          */
    FB_ERR_UNSUPPORTED = 6  /* TREE + MEAN_ALIGN (accurate mode is O(N*M) by definition), p > 4 */
} fb_status;

/* Loss kinds: Eq. 1, Eq. 3, Eq. 8 (P:243-247 with reading D27), Eq. 10 (the
 * keyframe alignment loss, readings D38-D40: alpha*||G_k[F_k]-G_i||^2 + ||S_k[F_k]-S_o[F_o]||^2
 * with F_o the counterpart NNF frozen at the start of each iteration). */
typedef enum { FB_LOSS_BASE = 0, FB_LOSS_GUIDE_STYLE = 1, FB_LOSS_MEAN_ALIGN = 2, FB_LOSS_PAIRWISE = 3 } fb_loss;
/* Window schedules: DIRECT = balanced/accurate; TREE = fast (Alg. 3-5, Eq. 6). */
typedef enum { FB_SCHED_DIRECT = 0, FB_SCHED_TREE = 1 } fb_schedule;
/* NNF initialisation at the coarsest level: Philox-uniform or identity (D8/D33). */
typedef enum { FB_INIT_RANDOM = 0, FB_INIT_IDENTITY = 1 } fb_init;
/* Operation ids for fb_workspace_size. */
typedef enum { FB_OP_NNF = 0, FB_OP_BLEND_DIRECT = 1, FB_OP_BLEND_TREE = 2, FB_OP_INTERPOLATE = 3 } fb_op;

typedef struct {
    int32_t patch_radius;    /* p: a patch is (2p+1)^2 pixels; "patch 5" -> 2 (D1). 1..4   */
    int32_t levels;          /* pyramid levels; 0 = auto: 1+max{k: min(H,W)>>k >= 32}, cut to fit (D6, D32) */
    int32_t iters_per_level; /* n of Alg. 1                                                 */
    int32_t rs_radius0;      /* random-search start radius; 0 = max(h_k, w_k) per level (D13, D33)  */
    int32_t rs_steps;        /* random-search steps; 0 = halve until the radius is < 1 (D13, D33)  */
    float alpha;             /* guide weight alpha of Eq. 3 / Eq. 8 (D15)                          */
    int32_t loss;            /* fb_loss                                                             */
    int32_t init;            /* fb_init                                                             */
    uint64_t seed;           /* Philox4x32-10 key (D21)                                             */
    int32_t prop_scales;     /* propagation scales J (jump flood, D41): steps 2^(J-1)..1, each with the
                                four directions of P:72; 0 or 1 = the paper's unit-step propagation   */
    int32_t tracking;        /* add NNF(S,T_{i-1}), NNF(S,T_{i+1}) as candidate fields: interpolation
                                (D42) and the direct blend schedule ("optional setting in
                                blending", D44: NNF(G_j,G_{i+-1}) for NNF(G_j,G_i)); 0 = off   */
} fb_match_cfg;

typedef struct {
    uint64_t nnf_pairs;       /* NNF estimations performed (the unit of every complexity claim) */
    uint64_t candidate_evals; /* loss evaluations: sum over pairs of sum_k h_k w_k n (1 + 4 + K_k) */
    uint64_t remap_pixels;    /* output pixels of remap/vote operations (aux refreshes and final remaps)       */
} fb_stats;

/* The RNG key of one NNF task (D21): original frame ids and a task tag (0 direct, 1/2 tree build /
 * query forward, 3/4 reversed, 5 interpolation, 6 API). */
typedef struct { int32_t src_id, tgt_id, task_tag; } fb_pair_key;

/* ---- context -------------------------------------------------------------------------------- */

/* Creates a context on `device` that enqueues on `cuda_stream` (a cudaStream_t; NULL = legacy default
 * stream).  *out receives the handle.  Errors: FB_ERR_INVALID_ARG (out NULL), FB_ERR_CUDA. */
fb_status fb_ctx_create(int device, void* cuda_stream, fb_ctx* out);
void fb_ctx_destroy(fb_ctx ctx);
/* Message for the last non-OK status of this context (never NULL; "" if none). */
const char* fb_last_error(fb_ctx ctx);
/* Caller-owned device workspace (e.g. a torch.empty uint8 tensor).  The library sub-allocates from it;
 * it must stay alive and unused by others while calls that use it are in flight. */
fb_status fb_set_workspace(fb_ctx ctx, void* dev_ptr, size_t bytes);
/* Upper bound on the NNF pairs processed in lockstep by one batch (0 = automatic: as many as a
 * 64 GiB state budget allows).  Batching never changes results (D21). */
fb_status fb_set_max_batch_pairs(fb_ctx ctx, int64_t max_pairs);
/* Workspace bytes an operation needs.  op = fb_op; n = B pairs (FB_OP_NNF) or N frames; M = window
 * half-width (blend) or number of keyframes K (interpolate).  Returns 0 on invalid arguments. */
size_t fb_workspace_size(fb_ctx ctx, int op, const fb_match_cfg* cfg, int n, int H, int W, int M);
/* Workspace bytes of one fb_blend_window_range call (same arguments; 0 on invalid arguments). */
size_t fb_workspace_size_range(fb_ctx ctx, int schedule, const fb_match_cfg* cfg, int N_total, int f0, int N, int H,
                               int W, int M, int t0, int t1);
/* Number of kernels this context has launched so far (for launch accounting in bench.py). */
uint64_t fb_launch_count(fb_ctx ctx);

/* Kernel-schedule options of one context (A/B of equivalent kernel schedules; every setting gives
 * bit-identical results, which tests/test_gpu_parity.py checks).  Defaults are the measured optima:
 *   FB_OPT_FUSED_ITER   0  1 = a whole level-0 iteration per launch (k_iter_fast; measured slower)
 *   FB_OPT_FUSE13       1  0 = level-0 propagation fields 1-3 and the random search as separate launches
 *   FB_OPT_PHASE0_MID   1  0 = level-0 E init + field 0 with the register-target kernel
 *   FB_OPT_TGT_REG_ROWS 3  target patch rows held in registers by the fused level-0 kernel (0 = all, 1, 2,
 *                          3 = none: every row from the shared tile)
 *   FB_OPT_L1_FAST      0  level 1 (u8 sources, p = 2) through 16-byte TF10 targets and the level-0 kernels
 *                          instead of the general kernel: 1 = fields 1-3 fused, 2 = per-field shared-tile
 *                          launches (bit-identical, both measured slower)
 *   FB_OPT_SUM_BOUND    1  0 = no patch-sum lower bound in the random search (every candidate gathers its
 *                          patch rows; the bound only skips candidates that provably lose, DESIGN.md §6;
 *                          used at every level with exact packed sources and for float-style table cells)
 *   FB_OPT_P3_FUSED     1  0 = at p = 3, level-0 fields 1-3 and the random search as separate launches
 *   FB_OPT_TAIL_BOUND   0  1 = the level-0 fused random search adds the partial + remainder bound (p = 2, exact
 *                          u8 sources: the FP32 partial of the first rows plus Cauchy-Schwarz on the remaining
 *                          rows' sums; only skips candidates that provably lose; measured slower)
 * Errors: FB_ERR_INVALID_ARG (unknown option or value). */
typedef enum { FB_OPT_FUSED_ITER = 0, FB_OPT_FUSE13 = 1, FB_OPT_PHASE0_MID = 2, FB_OPT_TGT_REG_ROWS = 3,
               FB_OPT_L1_FAST = 4, FB_OPT_SUM_BOUND = 5, FB_OPT_P3_FUSED = 6,
               FB_OPT_TAIL_BOUND = 7 } fb_option;
fb_status fb_set_option(fb_ctx ctx, int option, int value);

/* ---- kernel timing (bench instrumentation) -----------------------------------------------------
 * When enabled, every kernel launch of this context is bracketed by two CUDA events recorded on the
 * context stream.  fb_profile_read synchronises those events and writes up to `cap` per-kernel-class
 * entries (returns how many classes exist).  `work` is the class's algorithmic unit count summed over
 * launches: candidate evaluations for the PatchMatch field kernels ("field<phase>.L<level>"), output pixels
 * for the remap / combine kernels, texels for the pyramid kernels.  fb_profile_reset clears totals. */
typedef struct {
    char name[32];
    uint64_t launches;
    double ms;
    uint64_t work;
} fb_profile_entry;
fb_status fb_profile_enable(fb_ctx ctx, int on);
int fb_profile_read(fb_ctx ctx, fb_profile_entry* out, int cap);
void fb_profile_reset(fb_ctx ctx);

/* ---- pyramid (Alg. 1 "Resize images"; D6) ----------------------------------------------
 * frames: uint8 [B,H,W,3].  out: float texels, per frame level-major: frame b, level k, pixel (r,c) is
 * out[4*(b*P + off_k + r*w_k + c) + ch], ch 0..2 = RGB in 8-bit units, ch 3 = 0, with
 * w_k = W>>k, h_k = H>>k, off_k = sum_{i<k} h_i w_i, P = fb_pyramid_elems(1,H,W,levels)/4.
 * Level k = ((a+b)+(d+e))*0.25 over the 2x2 block of level k-1 (exact in 8-bit units). */
size_t fb_pyramid_elems(int B, int H, int W, int levels); /* floats in `out` */
fb_status fb_build_pyramid(fb_ctx ctx, const uint8_t* frames, int B, int H, int W, int levels, float* out);

/* ---- NNF estimation (Alg. 1) on B independent or window-coupled pairs ----------------
 * src_guide, tgt_guide: uint8 [B,H,W,3] (required).  src_style: uint8 [B,H,W,3], required unless
 * loss = BASE.  tgt_style: uint8 [B,H,W,3], required for MEAN_ALIGN only.  group: HOST int32 [B]
 * (MEAN_ALIGN and PAIRWISE only, else NULL).  MEAN_ALIGN: pairs with equal group ids share one target
 * and one average remapped image T-bar = (sum over the window, ascending src_id, of the remaps, with the
 * target's own style at its tgt_id) / (count+1), refreshed at the start of every iteration (Eq. 7,
 * P:237-239, D27).  PAIRWISE: group[b] is the index of pair b's counterpart (mutual, distinct): the two
 * NNFs of one target from two keyframes, estimated jointly with Eq. 10.
 * pair_keys: HOST [B] (required).  Outputs (device, nullable except nnf_out): nnf_out int32 [B,H,W,2];
 * err_out float [B,H,W] = E after the last select (D30); remapped_out float [B,H,W,3] = Alg. 2 remap
 * of src_style with the final NNF. */
fb_status fb_nnf_estimate(fb_ctx ctx, const fb_match_cfg* cfg, int B, int H, int W, const uint8_t* src_guide,
                          const uint8_t* tgt_guide, const uint8_t* src_style, const uint8_t* tgt_style,
                          const int32_t* group, const fb_pair_key* pair_keys, int32_t* nnf_out, float* err_out,
                          float* remapped_out, fb_stats* stats /* HOST, nullable */);

/* ---- remap (Alg. 2, valid-tap average D19) ----------------------------------------------
 * src float [B,H,W,3], nnf int32 [B,H,W,2] -> out float [B,H,W,3]; out[b,r,c] = (sum over valid taps,
 * dr then dc ascending, of src[b, F(r+dr,c+dc) - (dr,dc)]) / n_valid. */
fb_status fb_remap(fb_ctx ctx, int B, int H, int W, int p, const float* src, const int32_t* nnf, float* out);

/* ---- sliding-window blend (Eq. 2) ------------------------------------------------------
 * guide, style: uint8 [N,H,W,3]; out float [N,H,W,3].  W_i = [max(0,i-M), min(N-1,i+M)] (D3), the
 * self term is S_i (D4).  schedule DIRECT: cfg.loss GUIDE_STYLE = balanced, MEAN_ALIGN = accurate;
 * out_i = (sum over j ascending of X_{j->i}) / |W_i|.  schedule TREE (fast; GUIDE_STYLE only):
 * Alg. 3 build (levels <= floor(log2(M+1)), D24) -> Alg. 4 -> Alg. 5 queries on the forward and the
 * reversed table (D26) -> out_i = ((A_f + A_r) - S_i) / |W_i| (Eq. 6).  M = 0 or N = 1 returns the
 * style exactly.  Sharded runs: only targets in [t0, t1) are written (rows t0..t1-1 of out);
 * fb_blend_window is the full range [0, N).  cfg.tracking = 1 (DIRECT only, "optional setting in
 * blending", D44) couples every pair of the schedule: one batch over all targets; FB_ERR_UNSUPPORTED for the
 * tree schedule, for a partial range, or beyond 65535 pairs. */
fb_status fb_blend_window(fb_ctx ctx, const fb_match_cfg* cfg, int schedule, int N, int H, int W, int M,
                          const uint8_t* guide, const uint8_t* style, float* out, fb_stats* stats);
/* Same, restricted to output targets [t0, t1) of a video whose frames [f0, f0+N) are given: guide/style
 * hold frames f0..f0+N-1 (a shard plus its halo), frame ids in RNG keys are original ids (f0 + local),
 * the window is clipped to [0, N_total), and out holds rows for targets t0..t1-1 (original ids). */
fb_status fb_blend_window_range(fb_ctx ctx, const fb_match_cfg* cfg, int schedule, int N_total, int f0, int N,
                                int H, int W, int M, const uint8_t* guide, const uint8_t* style, int t0, int t1,
                                float* out, fb_stats* stats);

/* ---- sharded tree schedule with blending-table cell exchange (Alg. 3-5) -------
 * A shard's Alg. 5 queries visit cells BT(node, L) of nodes up to M frames outside its targets; instead of
 * rebuilding those (fb_blend_window_range does), shards build the cells they own and exchange them.
 * A cell is three int32 {orient, j, L}: orient 0 = forward, 1 = reversed frame order (D26); j is the node
 * index in that order (frame j forward, frame N_total-1-j reversed); L >= 1 its table level.  Its value is
 * the mean BT(j, L) of the 2^L frames [j-2^L+1, j] (orientation order) remapped into frame j (D25), stored
 * as a float4 pyramid of fb_pyramid_elems(1, H, W, levels)/4 texels (the fb_build_pyramid layout, RGB + 0),
 * `levels` = the configuration's pyramid depth.  Results are identical to fb_blend_window_range whoever
 * builds a cell (pair-keyed RNG, D21).
 *
 * fb_tree_build_cells: builds the n_cells listed cells (HOST int32 [n_cells][3]) into cell_out (device,
 *   n_cells pyramids back to back).  Every frame a cell reads must lie in the local frames [f0, f0+N).
 * fb_tree_query: targets [t0, t1) from the local frames (which must cover [t0-M, t1+M) clipped) and the
 *   given cells (cell_ptrs: HOST array of n_cells device pointers, one pyramid each); every cell the queries
 *   visit must be listed (FB_ERR_INVALID_ARG otherwise).  out as in fb_blend_window_range.
 * fb_tree_cell_texels: float4 texels of one cell pyramid for (cfg, H, W).
 * ws_needed (nullable): when non-NULL, nothing runs; the workspace bytes the call needs are stored there. */
size_t fb_tree_cell_texels(const fb_match_cfg* cfg, int H, int W);
fb_status fb_tree_build_cells(fb_ctx ctx, const fb_match_cfg* cfg, int N_total, int f0, int N, int H, int W,
                              const uint8_t* guide, const uint8_t* style, int n_cells, const int32_t* cells,
                              float* cell_out, fb_stats* stats, size_t* ws_needed);
fb_status fb_tree_query(fb_ctx ctx, const fb_match_cfg* cfg, int N_total, int f0, int N, int H, int W, int M,
                        const uint8_t* guide, const uint8_t* style, int t0, int t1, int n_cells,
                        const int32_t* cells, const float* const* cell_ptrs, float* out, fb_stats* stats,
                        size_t* ws_needed);

/* ---- keyframe interpolation (Eq. 9; D28) ----------------------------------------------
 * guide uint8 [N,H,W,3]; key_index HOST int32 [K], strictly increasing in [0,N); key_style uint8
 * [K,H,W,3]; out float [N,H,W,3].  Keys are copied verbatim; a frame m between consecutive keys
 * l < m < r is fma(X_l, (r-m)/(r-l), X_r * ((m-l)/(r-l))) with X_k the remap of key k's style under
 * NNF(G_k, G_m); frames outside the key span take the nearest key's remap.  The NNFs use the GUIDE_STYLE
 * loss, except cfg.loss = PAIRWISE: then the two NNFs of every frame between two keys are estimated
 * jointly with the alignment loss of Eq. 10.  cfg.tracking = 1 adds the object tracking of
 * P:256-259 (D42): each NNF(S_k, G_m) also tries NNF(S_k, G_{m-1}) and NNF(S_k, G_{m+1}) (frozen at the
 * start of every iteration) as whole candidate fields; all frames of a key span advance in lockstep. */
fb_status fb_interpolate_keyframes(fb_ctx ctx, const fb_match_cfg* cfg, int N, int H, int W, const uint8_t* guide,
                                   int K, const int32_t* key_index, const uint8_t* key_style, float* out,
                                   fb_stats* stats);

/* Same, restricted to output frames [t0, t1) (sharded interpolation): guide holds frames
 * t0..t1-1 only, key_guide [K,H,W,3] the keyframes' guide frames (broadcast to every shard with the key
 * styles), out [t1-t0,H,W,3].  Frame ids in RNG keys are original ids, so the rows equal the full call's.
 * cfg.tracking couples all frames of a key span (D42): FB_ERR_UNSUPPORTED unless [t0,t1) = [0,N).
 * ws_needed (nullable): when non-NULL, nothing runs; the workspace bytes the call needs are stored there. */
fb_status fb_interpolate_keyframes_range(fb_ctx ctx, const fb_match_cfg* cfg, int N, int H, int W, int t0, int t1,
                                         const uint8_t* guide, int K, const int32_t* key_index,
                                         const uint8_t* key_guide, const uint8_t* key_style, float* out,
                                         fb_stats* stats, size_t* ws_needed);

#ifdef __cplusplus
}
#endif
#endif /* FB_H */
