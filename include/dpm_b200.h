/*
 * dpm_b200.h -- C ABI of the B200 DPM score path (libdpm_b200.so, sm_100a).
 *
 * Drop-in boundary for the reference package's scoring path
 * (/root/reference/pkg/src/cpdetect).  The reference is pure Python/numpy
 * and has no FFI of its own; each entry point below names the reference
 * function it replaces, and INTEGRATION.md shows the ctypes binding a
 * maintainer adds on the reference side.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Every array argument is DEVICE memory
 *    unless its name ends in `_host`.  Offsets inside descriptor structs are
 *    element offsets (floats / doubles / bytes as documented) from the base
 *    pointer passed to the call, so one descriptor table serves any buffer.
 *  - Every call takes a cudaStream_t as `void* stream` (NULL = legacy
 *    default stream) and is asynchronous on it; no call synchronises, none
 *    allocates device memory, none keeps global mutable state.  Results are
 *    deterministic (fixed reduction order, no atomics on score sums).
 *  - Return value: DPM_OK (0) or a negative dpm_status; dpm_last_error()
 *    returns a thread-local message naming the offending field.
 *
 * Layouts (HBM)
 *  - Feature level X: float32 [H][W][L] (channel fastest; reference
 *    check_feature_map order, validation.py:65-86).
 *  - Projected level P: float32 planar [R][H][pitch], pitch >= W, pitch % 4 == 0.
 *  - Core G of a filter group: float32 [h][w][R][nf_pad] (filter fastest).
 *  - Response maps S: float32 [nf][Ho][pitch] with Ho = H-h+1, Wo = W-w+1 and
 *    pitch = (Wo + 3) & ~3 (rows padded to 16 bytes; the padding is never
 *    read as data).  Map offsets (s_off) are multiples of 4 floats.  Every
 *    kernel that reads or writes S uses this pitch; descriptor fields named
 *    Wp / Wo hold the valid width.  (Since ABI version 2.)
 *
 * ABI version 3: dpm_place_range carries E2in (was a pad field); added the
 * rank-prefix K2 (dpm_correlate_prefix*, dpm_corr_job.mode = 1) and the HOG
 * pyramid builder (dpm_resample*, dpm_hog*).
 */
#ifndef DPM_B200_H
#define DPM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPM_ABI_VERSION 4
#define DPM_MAX_PARTS 16

typedef enum {
  DPM_OK = 0,
  DPM_ERR_ARG = -1,         /* invalid shape / descriptor -> ValidationError */
  DPM_ERR_UNSUPPORTED = -2, /* valid but not supported by this build        */
  DPM_ERR_CUDA = -3,        /* CUDA runtime failure -> DeviceError           */
  DPM_ERR_NUMERIC = -4      /* non-finite inputs where finiteness is required */
} dpm_status;

/* ------------------------------------------------------------------ misc */
int dpm_abi_version(void);
const char* dpm_last_error(void);
/* SM count and compute capability of `device` (sizing persistent grids). */
int dpm_device_query(int device, int* sm_count, int* cc_major, int* cc_minor);

/* ---------------------------------------------------------- K1: project
 * P[r][y][x] = sum_l X[y][x][l] * C[l][r]
 * Replaces the channel contraction of _term_stack (correlation.py:128) and,
 * with C = identity, the channel layout change feeding correlate3_full
 * (correlation.py:92-112).  One job per (image, level).
 * L = 32 with R <= 8 runs on mma.sync tensor-core tiles (3xTF32 split, FP32
 * accumulation; within 2e-6 of max |P| of the float64 product, as the FFMA
 * path is); every other shape on FP32 FFMA.  A prefix
 * of C's columns gives bit-identical planes on either path. */
typedef struct {
  int64_t x_off;  /* float offset of the level's X block [H][W][L]          */
  int64_t p_off;  /* float offset of the level's P block [R][H][pitch]      */
  int32_t H, W;
  int32_t pitch;  /* P row pitch in floats, >= W, multiple of 4             */
  int32_t block0; /* first CTA of this job; set by dpm_project_prepare      */
} dpm_proj_job;

/* Fills block0 of every job (host table) and returns the CTA count to pass
 * to dpm_project (negative dpm_status on error). */
int64_t dpm_project_prepare(dpm_proj_job* jobs_host, int njobs);
int dpm_project(const float* X, float* P, const float* C, int L, int R,
                const dpm_proj_job* jobs, int njobs, int64_t nblocks, void* stream);

/* ------------------------------------------- K2: shortened correlation
 * S_f[y][x] = sum_{i<h, j<w, r<R} G[i][j][r][f] * P[chan_off + r][y+i][x+j]
 * Implicit GEMM over (position x filter) with K = h*w*R, FP32 FFMA.
 * Replaces correlate3_cp (correlation.py:155-167; G[i][j][r] = w_r a_ir b_jr
 * over the filter's own c-projected channels), cp_partial_stack
 * (correlation.py:170-180; prefix k is a filter whose core keeps ranks <= k,
 * so prefixes are bit-identical to correlate3_cp(upto = k+1)) and
 * correlate3_full (correlation.py:92-112; C = identity, G = the filter). */
typedef struct {
  int64_t p_off;     /* float offset of the (image, level) P block           */
  int64_t s_off;     /* float offset of the output maps [nf][Ho][pitch(Wo)]  */
  int64_t g_off;     /* float offset of the group's core [h][w][R][nf_pad]   */
  int32_t H, W, pitch, chan_off;
  int32_t h, w, R, nf;
  int32_t nf_pad;    /* filter stride of the core: nf rounded up to 8        */
  int32_t mode;      /* 0: nf filters; 1: rank prefixes (dpm_correlate_prefix) */
  int32_t range_idx; /* >= 0: fold per-map max/min into ranges[range_idx+f]  */
  int32_t pad;
} dpm_corr_job;

/* One CTA work item: tile (ty, tx) of job `job`. */
typedef struct {
  int32_t job, ty, tx, pad;
} dpm_corr_tile;

/* Tile geometry the planner must use for a launch class (h, nf):
 * tile_w x tile_h output positions per tile; returns warps per CTA, or a
 * negative dpm_status if (h, nf) has no specialised kernel (then the
 * generic kernel is used: tile 32 x 8, 8 warps). */
int dpm_correlate_tile_shape(int h, int nf, int* tile_w, int* tile_h);

/* All tiles of one call must belong to jobs with the same (h, nf, R) class
 * and max filter width <= w_max.  `ranges` (uint32 pairs: ordered-key max,
 * ordered-key min; may be NULL) collects per-map extrema for r*. */
int dpm_correlate(const float* P, const float* G, float* S, const dpm_corr_job* jobs,
                  const dpm_corr_tile* tiles, int ntiles, int h, int nf, int R,
                  int w_max, uint32_t* ranges, void* stream);

/* K2 on tcgen05 (kind::tf32, 3xTF32 split) for one filter group:
 * M = 128 output positions of one row, N = nf filters (padded to 16),
 * K = 8 ranks per tap; A is the staged input row shifted per tap, B the
 * resident core.  Each work item is a 128-wide column strip
 * (dpm_corr_tile.tx = strip index) of one job, processed top to bottom.
 * `Gtc` is the core in the tensor layout [h*w][R/4][2N][4]: rows < N hold
 * the tf32-truncated filter values, rows >= N the exact remainders.
 * Requirements: R % 8 == 0, 1 <= nf <= 64, h + 2 <= 16 and the returned
 * shared-memory size <= 227 KB. */
size_t dpm_correlate_tc_smem(int h, int w, int R, int nf);
/* Floats of the `Gtc` block for (h, w, R, nf): the tf32 hi|lo layout above,
 * followed -- for the compile-time DPM shapes (R = 8, h = 6, w in {6, 11}),
 * whose kernel runs the correction MMA in bf16 over tap pairs -- by the bf16
 * block [h][ceil(w/2)][2][N][8] of the tf32-truncated values (tap 2p then
 * 2p+1; zeros past w).  When dpm_correlate_tc_stack() returns KS > 1 the
 * block is the stacked layout instead (KS output rows per accumulator group):
 * with NB = h + 2(KS-1) tap-row blocks, block b holding tap row
 * i = h-1+KS-1-b (zeros outside 0..h-1) as 16 N-rows [hi of filters 0..7 |
 * lo of filters 0..7], the tf32 part is [w][R/4][NB*16][4] and the bf16 part
 * [ceil(w/2)][2][NB*16][8] (hi values in rows 0..7 of each block, 0 in
 * rows 8..15). */
size_t dpm_correlate_tc_core_floats(int h, int w, int R, int nf);
/* Output rows per accumulator group of the tcgen05 kernel for this shape:
 * 6 for the compile-time DPM shapes with nf <= 8 (e.g. the DPM roots), else 1. */
int dpm_correlate_tc_stack(int h, int w, int R, int nf);
int dpm_correlate_tc(const float* P, const float* Gtc, float* S, const dpm_corr_job* jobs,
                     const dpm_corr_tile* strips, int nstrips, int h, int w, int R, int nf,
                     uint32_t* ranges, void* stream);
/* Several filter groups of one shape in one launch (the generic-shape
 * kernel: any (h, w, R) but the compile-time DPM shapes above): every group
 * has at most nf filters and its own core block in the tf32 hi|lo layout at
 * float offset tc_off[job] of Gtc (device array indexed by job id, 16-byte
 * aligned blocks).  Strips of different groups may interleave; a persistent
 * CTA reloads the core (one bulk copy) when a strip's group differs from
 * the resident one. */
int dpm_correlate_tc_groups(const float* P, const float* Gtc, const int64_t* tc_off, float* S,
                            const dpm_corr_job* jobs, const dpm_corr_tile* strips, int nstrips,
                            int h, int w, int R, int nf, uint32_t* ranges, void* stream);

/* K2 in rank-prefix mode (convolution shortening, paper Algorithm 1;
 * replaces the reference's _term_stack + cumsum, correlation.py:115-180,
 * behind cp_partial_stack / correlate3_cp and detect(pruning=True)).
 * Jobs have mode == 1: the job's nf output maps (s_off, [nf][Ho][pitch]) are
 * the cumulative rank prefixes 1..nf (nf <= R) of ONE filter whose core is
 * column 0 of the [h][w][R][nf_pad] block at g_off:
 *   T_r = sum_{j<w} sum_{i<h} G[i][j][r] P[chan_off + r][y+i][x+j],
 *   map k-1 = T_0 + ... + T_{k-1}   (FP32, rank order),
 * one pass over the ranks (the cost of one full correlation).  Tiles are
 * (job, ty, tx) of dpm_correlate_prefix_tile() output positions; all tiles
 * of one call have filter height h (1..16; width 1..16).  `ranges` as for
 * dpm_correlate (slot range_idx + k for map k). */
int dpm_correlate_prefix_tile(int* tile_w, int* tile_h);
int dpm_correlate_prefix_check(const dpm_corr_job* jobs, int njobs);
int dpm_correlate_prefix(const float* P, const float* G, float* S, const dpm_corr_job* jobs,
                         const dpm_corr_tile* tiles, int ntiles, int h, uint32_t* ranges,
                         void* stream);

/* ------------------------------- HOG feature pyramid
 * Generalises the reference's 9-bin demo extractor (features.py:16-68) to
 * the 32-channel DPM v5 layout on the pyramid geometry the planner uses
 * (oracle/hog_oracle.py states the algorithm).  Images are [H][W][C]
 * (C = 1..4, uint8 or float32 in [0, 255]).
 * dpm_resample: level image = box-filter resampling to Hs x Ws (Hs <= H,
 * Ws <= W), float32 [Hs][Ws][C] at out_off.  dpm_hog: 4 x 4-pixel cells of
 * a resampled image -> the level's X block [Hs/4][Ws/4][32] at x_off;
 * `hist` is scratch of 20 floats per cell at h_off. */
typedef struct {
  int64_t img_off;  /* element offset of the image                          */
  int64_t out_off;  /* float offset of the resampled level                  */
  int32_t H, W, C, Hs, Ws;
  int32_t block0;   /* set by dpm_resample_prepare                          */
} dpm_resample_job;
int64_t dpm_resample_prepare(dpm_resample_job* jobs_host, int njobs);
int dpm_resample(const void* img, int u8, float* out, const dpm_resample_job* jobs, int njobs,
                 int64_t nblocks, void* stream);

typedef struct {
  int64_t r_off;    /* float offset of the resampled level [Hs][Ws][C]      */
  int64_t x_off;    /* float offset of the level's X block [Hs/4][Ws/4][32] */
  int64_t h_off;    /* float offset of the histogram scratch (20 per cell)  */
  int32_t Hs, Ws, C;
  int32_t block0;   /* set by dpm_hog_prepare                               */
} dpm_hog_job;
int64_t dpm_hog_prepare(dpm_hog_job* jobs_host, int njobs);
int dpm_hog(const float* R, float* hist, float* X, const dpm_hog_job* jobs, int njobs,
            int64_t nblocks, void* stream);

/* Initialise `n` range slots to (-inf, +inf). */
int dpm_ranges_init(uint32_t* ranges, int n, void* stream);

/* ------------------------------- K3 + K4: part placement + assembly
 * For every root (ry, rx) of an assembly's rectangle:
 *   placed_i = max over a window around centre (scale*ry + ay_i, scale*rx + ax_i)
 *              of S_i - penalty, separable: x pass then y pass, strict '>'
 *              in ascending offset order (ties -> smallest (dy, dx)), the
 *              penalty subtracted in two stages exactly as _placement_grid
 *              (detection.py:320-373), in FP64 on the FP32 map;
 *   total    = S_root[ry][rx] + sum_i placed_i + bias
 *              (detection.py:449, 509-519; dense_detect 590-598).
 * radius >= 0: the reference's windowed semantics.  radius < 0: unbounded
 * generalised distance transform, realised as the window of radius r*
 * computed from the map's range (SURVEY.md App. A.2 lemma; requires
 * c_dxx, c_dyy > 0).  Every placed map needs a range slot (filled by
 * dpm_correlate): it bounds the FP32 screening error and gives r*. */
typedef struct {
  int64_t s_off;     /* float offset of the part response map [Hp][pitch(Wp)] */
  int64_t x_off;     /* GDT path: offset of the x-pass scratch (sv/dx)      */
  int32_t Hp, Wp;
  int32_t ay, ax;
  int32_t scale;
  int32_t radius;    /* >= 0 windowed, < 0 GDT via r*                        */
  int32_t rx0, wr;   /* root columns (centres scale*rx + ax) = the assembly's */
  int32_t range_idx; /* range slot of the map                                */
  int32_t block0;    /* reserved                                             */
  int32_t smap;      /* dpm_assemble: TMA tensor map (dpm_smap_encode) of the */
  int32_t smap_z;    /*   map's group, and the map's index in that group     */
  double cdx, cdy, cdxx, cdyy;
} dpm_place_job;

/* Validates the placement jobs (host table); returns 0 or a negative
 * dpm_status.  (block0 is reserved.) */
int64_t dpm_place_prepare(dpm_place_job* jobs_host, int njobs);

/* Optional outputs: totals (double), packed part positions (uint32
 * (int16 y) << 16 | (uint16)(int16 x)), per-part placed values (double), and
 * detections with total >= tau appended to `dets` (count in *det_count,
 * which the caller zeroes; records beyond max_dets are dropped but counted). */
typedef struct {
  int64_t root_off;   /* float offset of the root map, < 0: no root term      */
  int64_t total_off;  /* double offset of totals [hr][wr], < 0: not written   */
  int64_t pos_off;    /* uint32 offset of positions [nparts][hr][wr], < 0: no */
  int64_t placed_off; /* double offset of placed [nparts][hr][wr], < 0: no    */
  int32_t root_pitch; /* row pitch of the root map                            */
  int32_t ry0, ry1, rx0, rx1;
  int32_t part_job0;  /* first dpm_place_job of this assembly                 */
  int32_t nparts;
  int32_t image, level, component;
  int32_t block0;     /* first CTA of the specialised K3 kernel (its tiles)   */
  int32_t block1;     /* first CTA of the generic K3 kernel (the others);     */
                      /*   both set by dpm_assemble_prepare                   */
  double bias;
} dpm_asm_job;

typedef struct {
  int32_t image, level, component, ry, rx, nparts;
  double score;
  uint32_t parts[DPM_MAX_PARTS]; /* (int16 y) << 16 | (uint16)(int16 x) */
} dpm_detection;

/* Validates both tables (host memory), numbers the root tiles of the
 * assembly jobs (block0 / block1) and returns the total CTA count to pass to
 * dpm_assemble; *nfast (if not NULL) receives how many of them run on the
 * specialised kernel (tiles at least 17 roots wide of jobs whose parts are
 * all at scale 2 with radius < 0 or 7 <= radius <= 16; see place2.cu), the
 * rest run on the generic one.  One job's outputs (nparts x hr x wr) must
 * stay below 2^31 elements (32-bit offsets inside a job); larger rectangles
 * are split by the caller. */
int64_t dpm_assemble_prepare(dpm_asm_job* jobs_host, int njobs, const dpm_place_job* pjobs_host,
                             int npjobs, int64_t* nfast);

/* K3 prologue, once per run after K2: per placement job, the radius on each
 * axis (the job's radius, or r* from its map range when radius < 0), the
 * FP32 screening bound E2 = 2^-15 (max|S| + max |pen_x| + max |pen_y|) over
 * the whole window (see placement.cu) and E2in, the same over the inner
 * window |d| <= min(r, 6) that place2.cu screens. */
typedef struct {
  int32_t rx, ry;
  float E2;
  float E2in;
} dpm_place_range;
int dpm_place_ranges(const dpm_place_job* pjobs, int njobs, const uint32_t* ranges,
                     dpm_place_range* prep, void* stream);

/* TMA descriptors of S map groups.  One descriptor per group [nf][Ho][pitch]
 * (a 3-D tensor of floats, x = column < Wo, y = row < Ho, z = map < nf) at
 * S + s_off; dpm_assemble copies each part's band of the map into shared
 * memory with it (boxes of DPM_SMAP_BOX_W x DPM_SMAP_BOX_H, cells outside the
 * map read as NaN).  Host function (no GPU work): writes n descriptors of
 * DPM_SMAP_BYTES (64-byte aligned) to maps_host, which the caller copies to
 * device memory.  The descriptors embed the address of S. */
#define DPM_SMAP_BYTES 128
#define DPM_SMAP_BOX_W 100
#define DPM_SMAP_BOX_H 32
typedef struct {
  int64_t s_off;     /* float offset of the group (multiple of 4)            */
  int32_t Ho, Wo, nf;
  int32_t pad;
} dpm_smap_desc;
int dpm_smap_encode(const float* S, const dpm_smap_desc* descs_host, int n, void* maps_host);

/* Placement of every part (x pass + y pass) fused with the assembly; one
 * CTA per 32 x 64 tile of roots.  `prep` is dpm_place_ranges' output for the
 * same placement table; `smaps` the device copy of dpm_smap_encode's
 * descriptors for S (each placement job names its map by smap / smap_z).
 * Detections require the positions output. */
int dpm_assemble(const float* S, const void* smaps, const dpm_place_job* pjobs,
                 const dpm_asm_job* ajobs,
                 int najobs, int64_t nfast, int64_t nblocks, const dpm_place_range* prep,
                 double* total,
                 uint32_t* pos, double* placed, double tau, dpm_detection* dets, int max_dets,
                 int* det_count, void* stream);

/* ------------------------------- K3 as a lower-envelope GDT (+ K4 fused)
 * Unbounded placement (radius < 0, c_dxx, c_dyy > 0) on the GDT root domain
 * (every part centre scale*root + anchor inside its map): Felzenszwalb's
 * generalised distance transform, rows then columns, evaluated at the
 * centres.  Same values as dpm_assemble with radius < 0; argmaxes identical
 * except at exact ties.  Replaces _placement_grid (detection.py:320-373) at
 * an unbounded radius, and the assembly of detect (detection.py:449, 509-538).
 *
 * x pass: for every map row and centre column, the winning S value and dx
 * are written to sv / dx at the job's x_off ([Hp][wr], row-major; sv float,
 * dx int16).  block0 (in units of 32-row warps) is set by the prepare call,
 * which returns the CTA count. */
int64_t dpm_gdt_x_prepare(dpm_place_job* jobs_host, int njobs);
int dpm_gdt_x(const float* S, float* sv, int16_t* dx, const dpm_place_job* jobs, int njobs,
              int64_t nblocks, const uint32_t* ranges, void* stream);

/* y pass fused with the assembly: one warp per 32 root columns of an
 * assembly; parts are placed and summed into totals (required) in part
 * order, then bias and tau compaction as in dpm_assemble.  `pjobs` is the
 * full placement table the assemblies index (part_job0), with x_off set as
 * for dpm_gdt_x. */
int64_t dpm_gdt_y_prepare(dpm_asm_job* ajobs_host, int najobs, const dpm_place_job* pjobs_host,
                          int npjobs);
int dpm_gdt_y(const float* S, const float* sv, const int16_t* dx, const dpm_place_job* pjobs,
              const dpm_asm_job* ajobs, int najobs, int64_t nblocks, const uint32_t* ranges,
              double* total, uint32_t* pos, double* placed, double tau, dpm_detection* dets,
              int max_dets, int* det_count, void* stream);

/* ------------------------------------------ pruned detection (Algorithm 1)
 * First failing rank of every root hypothesis of a rectangle, from the
 * rank-prefix maps (cp_partial_stack order).  Replaces the per-rank root
 * checks (detection.py:452-460) and the per-rank part window-max checks
 * (detection.py:471-503) of detect(pruning=True).  Job = one (level, filter)
 * role: radius < 0 is the root (value at the root position); radius >= 0 a
 * part (max over the (2*radius+1)^2 window around scale*root + anchor, cells
 * outside the map ignored).  map_offs[offs0 + r] is the float offset in S of
 * prefix r (r < R), thr[thr0 + r] its threshold; out[out_off + iy*wr + ix]
 * receives r + 1 for the first r with value < thr[r], or 0. */
typedef struct {
  int64_t out_off;   /* byte offset of the job's [hr][wr] uint8 ranks       */
  int32_t offs0;     /* first entry in map_offs                             */
  int32_t thr0;      /* first entry in thr                                  */
  int32_t R;         /* ranks checked                                       */
  int32_t Hp, Wp;    /* prefix map extent                                   */
  int32_t ry0, ry1, rx0, rx1;
  int32_t ay, ax, scale;
  int32_t radius;    /* < 0: root job                                       */
  int32_t block0;    /* first CTA; set by dpm_prune_prepare                 */
} dpm_prune_job;
int64_t dpm_prune_prepare(dpm_prune_job* jobs_host, int njobs);
int dpm_prune_ranks(const float* S, const int64_t* map_offs, const double* thr,
                    const dpm_prune_job* jobs, int njobs, int64_t nblocks, uint8_t* out,
                    void* stream);

/* Pruned detection, composition (detection.py:433-542 after the per-rank
 * checks): per root of an assembly, in part order, the hypotheses alive when
 * each part is checked (kill: a part failure removes the root; lenient: it
 * only drops the part's term), the reference's counters as histograms, and
 * the detections (score >= tau among the alive roots: the assembled total in
 * kill mode; root + alive parts' placed values + bias, in part order, in
 * lenient mode; a lenient part that failed reports root + anchor).  Job =
 * one assembly of dpm_assemble.  Outputs per root: lim[i] = the rank bound
 * of part i's alive window (0: not alive when part i is checked; R_i: never
 * fails; else its failing rank), prank[i] = part i's failing rank or 0.
 * Histograms (uint32, 256 bins each, at hist + hist_off): row 0 the root
 * ranks (0 = never fails), row 1 + i part i's failing ranks among the roots
 * alive at part i (bin 0: how many roots are alive at part i).  Detections
 * are appended (count in *det_count). */
typedef struct {
  int64_t rank_off;   /* dpm_prune_ranks output: role k (0 root, 1+i part i) at rank_off + k hr wr */
  int64_t lim_off;    /* uint8 outputs: lim [nparts][hr][wr] at lim_off, prank right after      */
  int64_t total_off, pos_off, placed_off;  /* dpm_assemble outputs of the assembly (all required) */
  int64_t root_off;   /* float offset in S of the root map                                      */
  int32_t root_pitch;
  int32_t ry0, ry1, rx0, rx1;
  int32_t nparts;
  int32_t image, level;
  int32_t hist_off;   /* uint32 offset of the job's (1 + nparts) x 256 histogram               */
  int32_t block0;     /* first CTA; set by dpm_prune_compose_prepare                            */
  double bias;
  int32_t part_R[DPM_MAX_PARTS];
  int32_t ay[DPM_MAX_PARTS], ax[DPM_MAX_PARTS];
} dpm_prune_asm;
int64_t dpm_prune_compose_prepare(dpm_prune_asm* jobs_host, int njobs);
int dpm_prune_compose(const uint8_t* ranks, const float* S, const double* total,
                      const uint32_t* pos, const double* placed, const dpm_prune_asm* jobs,
                      int njobs, int64_t nblocks, int kill_mode, double tau, uint8_t* lim,
                      uint32_t* hist, dpm_detection* dets, int max_dets, int* det_count,
                      void* stream);

/* The multiplication counter of the pruned part stage (detection.py:474-486,
 * 545-567): per (assembly, part), every part-support cell of the union of the
 * roots' search windows gets M = max over the roots whose window holds it of
 * lim; hist[hist_off + M] counts the cells (so the work of rank r is the
 * number of cells with M > r).  Job = one (assembly, part). */
typedef struct {
  int64_t lim_off;    /* the part's lim map [hr][wr] (dpm_prune_compose)     */
  int32_t hr, wr;     /* root rectangle extent                               */
  int32_t y0, y1, x0, x1;  /* covered box in part-support coordinates        */
  int32_t oy, ox;     /* root index of box cell (y0, x0)'s window centre: iy = y - oy */
  int32_t radius;
  int32_t hist_off;   /* uint32 offset of the job's 256 bins                 */
  int32_t block0;     /* first CTA; set by dpm_prune_cover_prepare           */
  int32_t pad;
} dpm_cover_job;
int64_t dpm_prune_cover_prepare(dpm_cover_job* jobs_host, int njobs);
int dpm_prune_cover(const uint8_t* lim, const dpm_cover_job* jobs, int njobs, int64_t nblocks,
                    uint32_t* hist, void* stream);

/* ------------------------------------------------------- mixture max
 * SURVEY.md §8(f) row 3 (the reference has no combination rule; SPEC asks
 * for a max).  Job = one (image, root level): the union rectangle of its
 * component assemblies (listed as indices into `ajobs` at
 * members[member0 .. member0+nmembers)); for every root position, best =
 * max over the components whose rectangle holds it of their totals (ties to
 * the lowest component), comp = that component, or (-inf, -1). */
typedef struct {
  int64_t out_off;   /* offset of the job's [hu][wu] outputs                */
  int32_t ry0, ry1, rx0, rx1;
  int32_t member0, nmembers;
  int32_t block0;    /* set by dpm_mixture_prepare                          */
  int32_t pad;
} dpm_mix_job;
int64_t dpm_mixture_prepare(dpm_mix_job* jobs_host, int njobs);
int dpm_mixture_max(const double* total, const dpm_asm_job* ajobs, const int32_t* members,
                    const dpm_mix_job* jobs, int njobs, int64_t nblocks, double* best,
                    int32_t* comp, void* stream);

/* ----------------------------------------------------- micro-benchmark
 * FP32 FFMA peak probe used by bench.py for the K2 roofline denominator:
 * `iters` dependent-chain-free FFMA blocks on every SM; returns via
 * *flops the FLOPs the launch performs. */
int dpm_ffma_probe(float* sink, int iters, double* flops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DPM_B200_H */
