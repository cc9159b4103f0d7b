// Internal definitions shared by the blinkline_b200 kernels and the C-ABI host code.
//
// Exactness policy: every stage whose result the reference defines to the
// last bit -- resample, gradient/orientation, histogram, energy, features, the exact
// re-score, IoU, ERT traversal/accumulation -- lives in a translation unit compiled with
// --fmad=false and spells its double arithmetic with the _rn intrinsics in the reference's
// evaluation order.  Only the fp32 screening classifier (bl_classify.cu) is compiled with
// FMA contraction; its results never reach the output without an exact fp64 re-score.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/blinkline_b200.h"

#define BL_HD_INLINE __host__ __device__ __forceinline__

namespace blb {

#ifdef __CUDACC__
// mbarrier + bulk-copy (TMA engine, 1-D) helpers shared by the tcgen05 screen and the
// small-batch cascade
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
#endif

constexpr int kBins = 18;
constexpr int kFeat = 31;
constexpr int kFeatPad = 32;     // fp32 planar feature planes (31 real + 1 zero plane)
constexpr int kWin = 10;         // window cells (the reference's scorer is fixed at 10x10x31)
constexpr int kRowW = kWin * kFeat;  // 310 weights per window row
constexpr int kFilterW = kWin * kRowW;  // 3100
constexpr int kFilters = 5;
constexpr int kMaxLevels = 32;
// tcgen05 screen operands: fp16 chunk planes (8 features per 16-B chunk, 32 features incl. a
// zero pad), features scaled by 2^kTcFeatExp so values below 2^-14 keep precision
constexpr int kTcPlanesF16 = 4;
constexpr int kTcFeatExp = 8;

// Screening tile: a warp scores 128 anchors, 4 consecutive anchors along x per lane, all 5
// filters; per level the tile is 32x4, 16x8 or 8x16 anchors, whichever wastes least.
// Feature planes are padded so its float4 loads never go out of bounds.

// gradHist: a warp owns 31 cells of a cell-row strip over a segment of kGhSegRows cell rows.
constexpr int kGhCells = 31;
#ifndef BL_HOG_SEG
#define BL_HOG_SEG 64  // measured at 512 / 1024 frames: 24 -> 64 rows, gradHist 1.397 -> 1.363 / 2.653 -> 2.573 ms
#endif
constexpr int kGhSegRows = BL_HOG_SEG;

struct LevelDesc {
  int w, h;              // level pixel dims
  int cw, ch;            // cells (w/8, h/8)
  int sw, sh;            // anchors (cw-9, ch-9)
  int level;             // pyramid level index k
  int side;              // round_half_up(window_px / c)
  double c;              // (5/6)^k from the host's libm pow (detector.cpp:104)
  long long pix_off;     // level pixels: element offset of frame 0 in the level arena
  long long pix_fstride; // elements between frames
  int pix_pitch;         // elements between rows
  int pix_margin;        // readable elements left of x = 0 and right of x = w - 1 on every row
  long long cell_off;    // cells: offset of frame 0 in the cell arenas (bins/energy/feat64)
  long long f32_off;     // fp32 planar features: float offset of frame 0
  int cw_pad, ch_pad;    // fp32 planar plane dims
  long long f32_fstride; // floats between frames (= 32 * ch_pad * cw_pad)
  long long fld_off;     // gradient field (f64 magnitude / u8 bin planes): offset of frame 0
  // work decomposition (block ranges are global across levels)
  int gr_tiles_x, gr_tiles_y;  // gradient 32x32-pixel blocks per frame
  long long gr_begin;          // first gradient block id of this level
  int gh_tiles_x, gh_tiles_y;  // gradHist warp tiles per frame
  long long gh_begin;          // first gradHist warp-tile id of this level
  int sc_tiles_x, sc_tiles_y;  // screening warp tiles per frame
  int sc_lanes_x;              // lanes along x in a screening warp tile (8, 4 or 2): tile is
                               // (4 * sc_lanes_x) x (32 / sc_lanes_x) anchors
  long long sc_begin;          // first screening warp-tile id of this level
  long long cell_begin;        // first cell id (for per-cell kernels) of this level
  long long tc_off;            // tcgen05 screen features: 4-B word offset of frame 0 ([4 planes][tc_ncp][8 fp16])
  long long tc_ncp;            // cells per plane (linear index cy * cw + cx, zero-padded tail)
  long long anchor_base;       // per-frame anchor offset (for candidate records)
};

struct PlanDesc {
  int n_frames;
  int n_scored;                // scored levels (eligible and >= one window)
  LevelDesc lv[kMaxLevels];
  long long gr_total;          // total gradient blocks
  long long fld_total;         // gradient-field pixels over levels and frames
  long long gh_total;          // total gradHist warp tiles
  long long sc_total;          // total screening warp tiles
  long long cell_total;        // total cells over levels and frames
  long long cells_per_frame;
};

// Per-launch table of the first work-item id of each scored level, passed BY VALUE so the
// level search reads the kernel-parameter constant bank instead of global memory.
struct LevelBegins {
  int n;
  long long b[kMaxLevels + 1];  // b[s] = first id of level s; b[n] = total
};

BL_HD_INLINE int find_level(const LevelBegins& B, long long id) {
  int s = 0;
#pragma unroll 1
  while (s + 1 < B.n && id >= B.b[s + 1]) ++s;
  return s;
}

// Candidate from the screen: (frame, scored-level slot, filter mask, cx, cy).
struct Candidate {
  int frame;
  int slot_r;   // (slot << 8) | mask of the filters that passed the screen
  int cx, cy;
};

// One candidate per screened ANCHOR: slot_r = slot * 8 + r is replaced by (slot << 8) | mask,
// mask = the filters whose screen sum passed the cut, so the exact re-score stages the
// anchor's feature strips once for all of them.  Warp-aggregated append; all 32 lanes must
// call it (flags == 0: no candidate).
__device__ __forceinline__ void emit_candidates(unsigned flags, int frame, int slot, int cx, int cy,
                                                Candidate* __restrict__ cand, unsigned long long* __restrict__ n_cand,
                                                long long cap) {
  const int lane = threadIdx.x & 31;
  const bool mine = flags != 0;
  const unsigned ballot = __ballot_sync(0xffffffffu, mine);
  if (!ballot) return;
  const int leader = __ffs(ballot) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(n_cand, (unsigned long long)__popc(ballot));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (mine) {
    const long long pos = (long long)base + __popc(ballot & ((1u << lane) - 1u));
    if (pos < cap) {
      Candidate c;
      c.frame = frame;
      c.slot_r = (slot << 8) | (int)flags;
      c.cx = cx;
      c.cy = cy;
      cand[pos] = c;
    }
  }
}

// Raw detection record on the device (same layout as bl_detection).
struct DevDet {
  int x, y, w, h;
  double score;
  int scale_index, rotation_index;
};
static_assert(sizeof(DevDet) == sizeof(bl_detection), "layout");

// One split node, 48 B (three 16-B loads).  Stored node-major, [t][node][k], so the lanes of
// a warp (consecutive trees k) read consecutive records.
struct SplitRec {
  double oax, oay, obx, oby, thr;
  short2 anchors;
  int pad;
};
static_assert(sizeof(SplitRec) == 48, "split record layout");

struct ErtDev {
  int L, T, K, F, S, NL;
  double shrinkage;
  const double* mean_xy;      // L*2
  const double* mean_c;       // L*2: mean shape minus its centroid (ert.cpp:41-46 txp/typ)
  const SplitRec* split;      // 3 planes of 16-B entries [T][S][K]: (oax, oay), (obx, oby), (thr, anchors)
  long long split_plane;      // entries per plane
  const double* leaves;       // T*K*NL*L*2
  double mean_cx, mean_cy;    // centroid of the mean shape (host-computed, ert.cpp:33-43 order)
};

// ----------------------------------------------------------------- helpers ------
__host__ __device__ inline long long div_up(long long a, long long b) { return (a + b - 1) / b; }

#define BL_DEV __device__ __forceinline__

// Exact double ops, never contracted (these TUs are also compiled with --fmad=false).
BL_DEV double dadd(double a, double b) { return __dadd_rn(a, b); }
BL_DEV double dsub(double a, double b) { return __dsub_rn(a, b); }
BL_DEV double dmul(double a, double b) { return __dmul_rn(a, b); }
BL_DEV double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// ------------------------------------------------------------- host launchers ----
// Defined in the kernel TUs, called by bl_capi.cu.  All are asynchronous on `L.st`;
// `Pd` is the device copy of the host plan `Ph`.
struct Launch {
  cudaStream_t st;
  uint64_t* counter;  // incremented per kernel launch
};

// bl_pyramid.cu
void launch_resample(const Launch& L, const void* src, int src_u8, int sw, int sh, long long s_pitch,
                     long long s_fstride, double* dst, int dw, int dh, long long d_pitch, long long d_fstride, int n);
bool resample_pair_fits(int sw, int sh, int mw, int mh, int dw, int dh);
// The whole pyramid chain (levels 1 .. n_levels-1) in one cooperative launch (small batches).
struct PyrChain {
  int n_levels, n_frames;
  const void* src0;
  long long s0_pitch, s0_fstride;
  int lw[kMaxLevels], lh[kMaxLevels];
  double* lv[kMaxLevels];  // level k >= 1: frame 0, pixel (0, 0)
  long long lpitch[kMaxLevels], lfstride[kMaxLevels];
  double rx[kMaxLevels], ry[kMaxLevels];  // step k: double(w_{k-1}) / w_k (image.cpp:136-137)
  // the batch's detection counters, zeroed by the chain's first CTA (instead of three memset
  // nodes ahead of the next kernels; nullptr: not zeroed here)
  unsigned long long* zero_u64;
  int* zero_i32;  // [n_zero_i32]
  int n_zero_i32;
  int* zero_flag;
};
int launch_pyramid_chain(const Launch& L, const PyrChain& C, int src_u8);
void launch_resample_pair(const Launch& L, const void* src, int src_u8, int sw, int sh, long long s_pitch,
                          long long s_fstride, int mw, int mh, double* dst, int dw, int dh, long long d_pitch,
                          long long d_fstride, int n);
// bl_hog.cu
void set_direction_table(const double* ux, const double* uy);
// Dynamic shared-memory opt-in of one kernel on the current device: the largest dynamic
// allocation the device allows next to the kernel's static shared memory.
template <class Kernel>
inline void smem_optin(Kernel* k, int optin) {
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, (const void*)k) != cudaSuccess) return;
  cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)a.sharedSizeBytes);
}

// Per-device kernel configuration (dynamic shared-memory opt-in up to `optin` bytes), called by
// bl_ctx_create for the context's device.
void configure_screen_tc_kernels(int optin);
void configure_exact_kernels(int optin);
void configure_hog_kernels(int optin);
void configure_classify_kernels(int optin);
void configure_ert_kernels(int optin);
void configure_pyramid_kernels(int optin);
void launch_grad(const Launch& L, const PlanDesc& Ph, const PlanDesc* Pd, int s_lo, int s_hi, const void* base,
                 int src_kind /*0 u8, 1 f64*/, double* fmag, uint8_t* fori);
void launch_gradhist(const Launch& L, const PlanDesc& Ph, const PlanDesc* Pd, const double* fmag,
                     const uint8_t* fori, double* bins, double* energy);
void launch_hog(const Launch& L, const PlanDesc& Ph, const PlanDesc* Pd, int s_lo, int s_hi, const void* base,
                int src_kind /*0 u8, 1 f64*/, double* bins, double* energy);
void launch_orientation(const Launch& L, const double* gx, const double* gy, long long n, uint8_t* out);
void launch_sqrt_check(const Launch& L, const double* in, long long n, double* fast, double* ieee);
void launch_energy(const Launch& L, const double* bins, long long cells, double* energy);
void launch_features(const Launch& L, const PlanDesc& Ph, const PlanDesc* Pd, const double* bins,
                     const double* energy, double* feat64, float* feat32, float* feat_tc);
// bl_classify.cu
void launch_screen(const Launch& L, const PlanDesc& Ph, const PlanDesc* Pd, const float* feat32,
                   const float* w32, const float* cut, Candidate* cand, unsigned long long* n_cand,
                   long long cand_cap);
// bl_screen_tc.cu
size_t tc_feat_floats_per_frame(int cw, int ch, long long* ncp_out, int* tiles_out);
size_t tc_weight_floats();
void launch_screen_tc(const Launch& L, const PlanDesc& Ph, const PlanDesc* Pd, const float* feat_tc,
                      const float* w_tc, const float* cut, Candidate* cand, unsigned long long* n_cand,
                      long long cand_cap, float* dbg_scores);
// bl_exact.cu
void launch_rescore(const Launch& L, int n_frames, const PlanDesc* Pd, const double* feat64, const double* w64,
                    const double* w64t /* k_rescore_lat's [c][f][r][j] copy, or null */,
                    const double* bias, double thr, int cell_px, const Candidate* cand,
                    const unsigned long long* n_cand, long long cand_cap, DevDet* dets,
                    int* det_count, long long cap_pf, int* overflow);
void launch_score_dense(const Launch& L, const double* feat64, int cw, int ch, const double* w64, double bias,
                        double* scores);
void launch_score_exact_all(const Launch& L, const double* feat64, int cw, int ch, const double* w64,
                            double bias, double* scores);
size_t nms_key_bytes();
long long nms_gkeys_per_frame(long long cap_pf);
void launch_transpose_weights(const Launch& L, const double* w64, double* w64t);
void launch_nms(const Launch& L, const DevDet* dets, const int* det_count, long long cap_pf, int n_frames,
                double iou_thr, DevDet* kept_out, int* kept_count, void* gkeys, long long gkeys_pf);
void launch_flatten(const Launch& L, const DevDet* kept, const int* kept_count, long long cap_pf,
                    int n_frames, int* offsets, DevDet* flat, int* face_frame, int* meta,
                    long long flat_cap, const int* raw_overflow, DevDet* best = nullptr, int* best_frame = nullptr);
// bl_ert.cu
void launch_ert_init(const Launch& L, const ErtDev& M, const int* n_faces, int cap, double* cur);
void launch_ert_level(const Launch& L, const ErtDev& M, int t, const void* frames, int u8, int w, int h,
                      long long pitch, long long fstride, const int* face_frame, const int* boxes, int box_stride,
                      const int* n_faces, int cap, double* cur, double2* tf, uint8_t* leaf_idx,
                      long long leaf_stride, int* err);
bool ert_cascade_fits(const ErtDev& M);
bool ert_wide_fits(const ErtDev& M);
void launch_ert_wide(const Launch& L, const ErtDev& M, const void* frames, int u8, int w, int h, long long pitch,
                     long long fstride, const int* face_frame, const int* boxes, int box_stride, const int* n_faces,
                     int cap, double* out_xy, uint8_t* leaf_out, long long leaf_out_stride, int* err,
                     int cluster /* CTAs per face: 1, 2, 4 or 8 */);
void launch_ert_cascade(const Launch& L, const ErtDev& M, const void* frames, int u8, int w, int h, long long pitch,
                        long long fstride, const int* face_frame, const int* boxes, int box_stride,
                        const int* n_faces, int cap, double* out_xy, uint8_t* leaf_out, long long leaf_out_stride,
                        int* err);
void launch_ert_finish(const Launch& L, const ErtDev& M, const int* boxes, int box_stride,
                       const int* n_faces, int cap, const double* cur, double* out_xy);

}  // namespace blb
