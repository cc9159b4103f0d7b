// Classifier stage 2 (exact re-score), threshold + box mapping, and per-frame NMS.
//
// Compiled with --fmad=false.  The re-score evaluates a candidate window exactly as
// score_separable does (detector.cpp:66-100): for each window row j the 310-term dot
// product of the feature strip at (cx, cy+j) with filter row j, accumulated in order
// without FMA, then the 10 row sums in order, then + bias.  Detections therefore carry
// bit-identical scores, and threshold_detections' box mapping (detector.cpp:102-122) and
// NMS (detector.cpp:124-142, IoU detector.cpp:16-28) are replayed with the same double
// operations, so the kept list is bit-identical to the reference's.
#include <float.h>

#include <algorithm>

#include "bl_internal.cuh"

namespace blb {

// Exact separable window score.  A warp scores three windows at once: lanes 10g..10g+9 own
// the ten window rows of window g (g = 0, 1, 2; lanes 30-31 idle), each accumulating its
// 310-term row dot product in the reference's order; the row sums are then added in order
// by the group's first lane.  Result valid in lanes 0, 10, 20.
BL_DEV double exact_window_score3(const double* __restrict__ feat, int cw, int cx, int cy,
                                  const double* __restrict__ w, double bias, int lane, bool active) {
  const int g = lane / 10, j = lane - 10 * (lane / 10);
  double acc = 0.0;
  if (active && g < 3) {
    const double* strip = feat + ((long long)(cy + j) * cw + cx) * kFeat;
    const double* wr = w + j * kRowW;
#pragma unroll 10
    for (int k = 0; k < kRowW; ++k) acc = dadd(acc, dmul(__ldg(strip + k), __ldg(wr + k)));
  }
  double total = 0.0;
  const int base = (g < 3 ? g : 0) * 10;
#pragma unroll
  for (int jj = 0; jj < kWin; ++jj) total = dadd(total, __shfl_sync(0xffffffffu, acc, base + jj));
  return dadd(total, bias);
}

BL_DEV int round_half_up(double v) { return (int)floor(dadd(v, 0.5)); }  // detector.cpp:41

// The re-score proper.  A candidate is an anchor plus the mask of filters whose screen sum
// passed the cut.  Each CTA keeps all five filters' fp64 weights resident in shared memory
// (rows padded to 311 doubles so the ten window rows of a filter sit on distinct banks).  A
// warp scores three anchors; lanes 10g + j (g < 3) own window row j of anchor g.  The
// feature strips are staged one window cell (31 features) at a time into padded shared
// memory with coalesced loads (lane f fetches feature f of each of the 30 (anchor, row)
// strips), copied once into registers, and dotted with every masked filter's row: each
// filter's 310-term sum runs strictly in the reference's order (detector.cpp:77-88), and
// the strips cross L1 once per anchor rather than once per (anchor, filter).
constexpr int kRsPitch = 33;
constexpr int kRsWPitch = kRowW + 1;  // 311
#ifndef BL_RS_WARPS
#define BL_RS_WARPS 6
#endif
constexpr int kRsWarps = BL_RS_WARPS;
constexpr int kRsWarpDoubles = 30 * kRsPitch;
constexpr size_t kRsSmem =
    sizeof(double) * ((size_t)kRsWarps * kRsWarpDoubles + (size_t)kFilters * kWin * kRsWPitch);

__global__ void __launch_bounds__(32 * kRsWarps) k_rescore(const PlanDesc* __restrict__ P,
                                                 const double* __restrict__ feat64,
                                                 const double* __restrict__ w64,
                                                 const double* __restrict__ bias, double thr,
                                                 int cell_px, const Candidate* __restrict__ cand,
                                                 const unsigned long long* __restrict__ n_cand,
                                                 long long cand_cap, DevDet* __restrict__ dets,
                                                 int* __restrict__ det_count, long long cap_pf,
                                                 int* __restrict__ overflow) {
  extern __shared__ double rs_smem[];
  const long long n = min((long long)*n_cand, cand_cap);
  if (n == 0) return;
  double* Wsm = rs_smem + (size_t)kRsWarps * kRsWarpDoubles;  // [5][10][311]
  {  // stage the weights: 128-bit loads, 8 in flight per thread (a row of 310 is even, so a
     // pair never straddles two rows); one load at a time made this most of a small batch's time
    constexpr int kPairs = kFilters * kFilterW / 2, kU = 8;
    const double2* w2 = reinterpret_cast<const double2*>(w64);
    for (int e0 = threadIdx.x; e0 < kPairs; e0 += blockDim.x * kU) {
      double2 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = e0 + u * blockDim.x;
        v[u] = e < kPairs ? __ldg(w2 + e) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = 2 * (e0 + u * blockDim.x);
        if (e < kFilters * kFilterW) {
          const int rj = e / kRowW;  // r * 10 + j
          double* d = Wsm + rj * kRsWPitch + (e - rj * kRowW);
          d[0] = v[u].x;
          d[1] = v[u].y;
        }
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* Fs = rs_smem + warp * kRsWarpDoubles;
  const int g = lane / 10;
  const int jl = lane - 10 * g;  // this lane's window row (lanes < 30)
  const long long nw = (long long)gridDim.x * kRsWarps;
  for (long long i0 = ((long long)blockIdx.x * kRsWarps + warp) * 3; i0 < n; i0 += nw * 3) {
    const double* fst[3];
    int cwv[3];
    unsigned mask_any = 0, my_mask = 0;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const bool real = i0 + q < n;
      const Candidate c = cand[min(i0 + q, n - 1)];
      const LevelDesc& D = P->lv[c.slot_r >> 8];
      cwv[q] = D.cw;
      fst[q] = feat64 + (D.cell_off + (long long)c.frame * D.cw * D.ch + (long long)c.cy * D.cw + c.cx) * kFeat;
      const unsigned m = real ? (unsigned)(c.slot_r & 0x1f) : 0u;
      mask_any |= m;
      if (g == q) my_mask = m;
    }
    double acc[kFilters];
#pragma unroll
    for (int r = 0; r < kFilters; ++r) acc[r] = 0.0;
    const double* wrow = Wsm + (lane < 30 ? jl : 0) * kRsWPitch;
#pragma unroll 1
    for (int ci = 0; ci < kWin; ++ci) {
      if (lane < kFeat) {
#pragma unroll
        for (int q = 0; q < 3; ++q)
#pragma unroll
          for (int j = 0; j < kWin; ++j)
            Fs[(q * 10 + j) * kRsPitch + lane] = __ldg(fst[q] + ((long long)j * cwv[q] + ci) * kFeat + lane);
      }
      __syncwarp();
      if (lane < 30) {
        double fr[kFeat];
#pragma unroll
        for (int f = 0; f < kFeat; ++f) fr[f] = Fs[lane * kRsPitch + f];
        // all five filters' chains, branch-free and interleaved (five independent dependent-add
        // chains in flight instead of one); a filter outside the mask is computed and discarded
#pragma unroll
        for (int f = 0; f < kFeat; ++f)
#pragma unroll
          for (int r = 0; r < kFilters; ++r)
            acc[r] = dadd(acc[r], dmul(fr[f], wrow[r * kWin * kRsWPitch + ci * kFeat + f]));  // detector.cpp:84
      }
      __syncwarp();
    }
    // column pass (detector.cpp:91-95): the ten row sums in order, then + bias, per filter
    const int base = (g < 3 ? g : 0) * 10;
#pragma unroll
    for (int r = 0; r < kFilters; ++r) {
      if (!((mask_any >> r) & 1u)) continue;
      double total = 0.0;
#pragma unroll
      for (int jj = 0; jj < kWin; ++jj) total = dadd(total, __shfl_sync(0xffffffffu, acc[r], base + jj));
      const long long i = i0 + (g < 3 ? g : 0);
      if (!(g < 3 && i < n && lane == 10 * g && ((my_mask >> r) & 1u))) continue;
      const Candidate c = cand[i];
      const LevelDesc& D = P->lv[c.slot_r >> 8];
      const double sc = dadd(total, bias[r]);
      if (sc > thr) {  // detector.cpp:110 (strict)
        DevDet d;
        d.x = round_half_up(ddiv((double)(c.cx * cell_px), D.c));
        d.y = round_half_up(ddiv((double)(c.cy * cell_px), D.c));
        d.w = D.side;
        d.h = D.side;
        d.score = sc;
        d.scale_index = D.level;
        d.rotation_index = r;
        const int idx = atomicAdd(det_count + c.frame, 1);
        if (idx < cap_pf)
          dets[(long long)c.frame * cap_pf + idx] = d;
        else
          atomicExch(overflow, 1);
      }
    }
  }
}

// Small batches (a frame or a camera stream's 16): the re-score's time is latency -- a warp's
// three candidates x 10 window columns of 155 dependent fp64 multiply-adds per lane.  Here a
// CTA of 64 threads takes one candidate at a time: thread t = r * 10 + j (filter r, window row
// j) runs its own row chain scratch(r, j) = sum over c, f in the reference's order
// (detector.cpp:76-88, same as k_rescore), reading the candidate's 10 x 310 features from shared
// memory (staged with coalesced loads) and the weights from the transposed copy
// wT[c][f][r][j] (one coalesced 400-B line per step, L1-resident); then the column pass
// (detector.cpp:91-95).  Bit-identical to k_rescore.
constexpr int kRlPitch = kRowW + 1;  // 311: smem row pitch of the staged window
__global__ void __launch_bounds__(64) k_rescore_lat(const PlanDesc* __restrict__ P,
                                                    const double* __restrict__ feat64,
                                                    const double* __restrict__ wT,
                                                    const double* __restrict__ bias, double thr, int cell_px,
                                                    const Candidate* __restrict__ cand,
                                                    const unsigned long long* __restrict__ n_cand,
                                                    long long cand_cap, DevDet* __restrict__ dets,
                                                    int* __restrict__ det_count, long long cap_pf,
                                                    int* __restrict__ overflow) {
  __shared__ double Fs[kWin * kRlPitch];
  __shared__ double scr[kFilters * kWin];
  const long long n = min((long long)*n_cand, cand_cap);
  const int t = threadIdx.x;
  for (long long i = blockIdx.x; i < n; i += gridDim.x) {
    const Candidate c = cand[i];
    const LevelDesc& D = P->lv[c.slot_r >> 8];
    const double* src = feat64 + (D.cell_off + (long long)c.frame * D.cw * D.ch + (long long)c.cy * D.cw + c.cx) * kFeat;
    // the window's 10 rows of 10 cells x 31 features: each row is 310 contiguous doubles
    for (int e = t; e < kWin * kRowW; e += 64) {
      const int j = e / kRowW, k = e - j * kRowW;
      Fs[j * kRlPitch + k] = __ldg(src + (long long)j * D.cw * kFeat + k);
    }
    __syncthreads();
    if (t < kFilters * kWin) {
      const int r = t / kWin, j = t - r * kWin;
      const double* fr = Fs + j * kRlPitch;
      const double* wt = wT + t;  // + (c * 31 + f) * 50
      double acc = 0.0;
      // weights 31 steps ahead (one window column per batch): the chain waits on fp64 adds,
      // not on a load per step
      double wv[kFeat], wn[kFeat];
#pragma unroll
      for (int f = 0; f < kFeat; ++f) wv[f] = __ldg(wt + f * (kFilters * kWin));
#pragma unroll 1
      for (int c0 = 0; c0 < kRowW; c0 += kFeat) {
        const int cn = c0 + kFeat < kRowW ? c0 + kFeat : c0;  // next column's weights in flight
#pragma unroll
        for (int f = 0; f < kFeat; ++f) wn[f] = __ldg(wt + (cn + f) * (kFilters * kWin));
#pragma unroll
        for (int f = 0; f < kFeat; ++f) acc = dadd(acc, dmul(fr[c0 + f], wv[f]));
#pragma unroll
        for (int f = 0; f < kFeat; ++f) wv[f] = wn[f];
      }
      scr[r * kWin + j] = acc;
      (void)r;
    }
    __syncthreads();
    if (t < kFilters && ((c.slot_r >> t) & 1)) {
      double total = 0.0;
#pragma unroll
      for (int j = 0; j < kWin; ++j) total = dadd(total, scr[t * kWin + j]);
      const double sc = dadd(total, bias[t]);
      if (sc > thr) {  // detector.cpp:110 (strict)
        DevDet d;
        d.x = round_half_up(ddiv((double)(c.cx * cell_px), D.c));
        d.y = round_half_up(ddiv((double)(c.cy * cell_px), D.c));
        d.w = D.side;
        d.h = D.side;
        d.score = sc;
        d.scale_index = D.level;
        d.rotation_index = t;
        const int idx = atomicAdd(det_count + c.frame, 1);
        if (idx < cap_pf)
          dets[(long long)c.frame * cap_pf + idx] = d;
        else
          atomicExch(overflow, 1);
      }
    }
    __syncthreads();  // Fs / scr reused by the next candidate
  }
}

// wT[c][f][r][j] = w[r][j][c][f] (c = window column, f = feature, r = filter, j = window row)
__global__ void k_transpose_weights(const double* __restrict__ w, double* __restrict__ wT) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= kFilters * kFilterW) return;
  const int r = e / kFilterW, rem = e - r * kFilterW;
  const int j = rem / kRowW, cf = rem - j * kRowW;
  wT[(long long)cf * (kFilters * kWin) + r * kWin + j] = w[e];
}

void launch_transpose_weights(const Launch& L, const double* w64, double* w64t) {
  k_transpose_weights<<<(unsigned)div_up(kFilters * kFilterW, 256), 256, 0, L.st>>>(w64, w64t);
  ++*L.counter;
}

constexpr int kRsLatFrames = 16;
#ifndef BL_RS_LAT_GRID
#define BL_RS_LAT_GRID 4  // CTAs per SM of k_rescore_lat (C2: 25 -> 17 us vs 2)
#endif  // batches up to this many frames take k_rescore_lat
constexpr int kRsCtasPerFrame = 8;
void launch_rescore(const Launch& L, int n_frames, const PlanDesc* Pd, const double* feat64, const double* w64,
                    const double* w64t,
                    const double* bias, double thr, int cell_px, const Candidate* cand,
                    const unsigned long long* n_cand, long long cand_cap, DevDet* dets,
                    int* det_count, long long cap_pf, int* overflow) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // persistent: one CTA per SM (the weights fill most of its smem), but a small batch takes
  // fewer: every CTA stages all 124 KB of weights, and for a frame or two that staging, not the
  // few hundred candidates, is the kernel's time (C1: 27 us at 148 CTAs)
  if (w64t && n_frames <= kRsLatFrames) {
    k_rescore_lat<<<(unsigned)(sms * BL_RS_LAT_GRID), 64, 0, L.st>>>(Pd, feat64, w64t, bias, thr, cell_px, cand, n_cand, cand_cap,
                                                       dets, det_count, cap_pf, overflow);
    ++*L.counter;
    return;
  }
  const dim3 grid((unsigned)std::max(1, std::min(sms, n_frames * kRsCtasPerFrame)));
  k_rescore<<<grid, 32 * kRsWarps, kRsSmem, L.st>>>(Pd, feat64, w64, bias, thr, cell_px, cand, n_cand, cand_cap,
                                                    dets, det_count, cap_pf, overflow);
  ++*L.counter;
}

// Every anchor of one feature image, one filter: bl_score_window (score_separable).
__global__ void __launch_bounds__(256) k_score_all(const double* __restrict__ feat, int cw, int ch,
                                                   const double* __restrict__ w, double bias,
                                                   double* __restrict__ scores) {
  const int lane = threadIdx.x & 31;
  const int g = lane / 10;
  const int sw = cw - (kWin - 1), sh = ch - (kWin - 1);
  const long long n = (long long)sw * sh;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long i0 = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 3; i0 < n; i0 += nw * 3) {
    const long long i = i0 + (g < 3 ? g : 0);
    const bool active = g < 3 && i < n;
    const long long ii = active ? i : i0;
    const int cy = (int)(ii / sw), cx = (int)(ii - (long long)(ii / sw) * sw);
    const double sc = exact_window_score3(feat, cw, cx, cy, w, bias, lane, active);
    if (active && lane == 10 * g) scores[i] = sc;
  }
}

void launch_score_exact_all(const Launch& L, const double* feat64, int cw, int ch, const double* w64,
                            double bias, double* scores) {
  const long long n = (long long)(cw - 9) * (ch - 9);
  if (n <= 0) return;
  const int blocks = (int)min(div_up(n, 8), (long long)148 * 16);
  k_score_all<<<blocks, 256, 0, L.st>>>(feat64, cw, ch, w64, bias, scores);
  ++*L.counter;
}

// score_dense (detector.cpp:45-64), the definitional order: one accumulator from 0.0 over the
// window's 3100 terms, row j outer, feature k inner, + bias.  A thread per anchor (a stage
// API, not the detect path).
__global__ void __launch_bounds__(128) k_score_dense(const double* __restrict__ feat, int cw, int ch,
                                                     const double* __restrict__ w, double bias,
                                                     double* __restrict__ scores) {
  const int sw = cw - (kWin - 1), sh = ch - (kWin - 1);
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)sw * sh) return;
  const int cy = (int)(i / sw), cx = (int)(i - (long long)cy * sw);
  double acc = 0.0;
  for (int j = 0; j < kWin; ++j) {
    const double* strip = feat + ((long long)(cy + j) * cw + cx) * kFeat;  // 10 cells x 31, contiguous
    const double* wr = w + j * kRowW;
#pragma unroll 10
    for (int k = 0; k < kRowW; ++k) acc = dadd(acc, dmul(__ldg(strip + k), __ldg(wr + k)));
  }
  scores[i] = dadd(acc, bias);
}

void launch_score_dense(const Launch& L, const double* feat64, int cw, int ch, const double* w64, double bias,
                        double* scores) {
  const long long n = (long long)(cw - 9) * (ch - 9);
  if (n <= 0) return;
  k_score_dense<<<(unsigned)div_up(n, 128), 128, 0, L.st>>>(feat64, cw, ch, w64, bias, scores);
  ++*L.counter;
}

// ------------------------------------------------------------------------- NMS ----
// detector.cpp:16-28
BL_DEV double iou_exact(const DevDet& a, const DevDet& b) {
  const long long ix0 = max(a.x, b.x);
  const long long iy0 = max(a.y, b.y);
  const long long ix1 = min((long long)(a.x + a.w), (long long)(b.x + b.w));
  const long long iy1 = min((long long)(a.y + a.h), (long long)(b.y + b.h));
  const long long iw = ix1 - ix0;
  const long long ih = iy1 - iy0;
  if (iw <= 0 || ih <= 0) return 0.0;
  const double inter = dmul((double)iw, (double)ih);
  const double uni = dsub(dadd(dmul((double)a.w, (double)a.h), dmul((double)b.w, (double)b.h)), inter);
  if (uni <= 0.0) return 0.0;
  return ddiv(inter, uni);
}

// iou(a, b) > thr with the reference's rounding (detector.cpp:16-28, 134), deciding in fp32
// when the quotient is clearly away from thr (|fp32 quotient - exact| < 1e-6 for integer
// areas) and falling back to the exact fp64 quotient otherwise.
BL_DEV bool iou_exceeds(const DevDet& a, const DevDet& b, double thr) {
  const long long ix0 = max(a.x, b.x);
  const long long iy0 = max(a.y, b.y);
  const long long ix1 = min((long long)(a.x + a.w), (long long)(b.x + b.w));
  const long long iy1 = min((long long)(a.y + a.h), (long long)(b.y + b.h));
  const long long iw = ix1 - ix0;
  const long long ih = iy1 - iy0;
  if (iw <= 0 || ih <= 0) return 0.0 > thr;
  const long long uni = (long long)a.w * a.h + (long long)b.w * b.h - iw * ih;
  if (uni <= 0) return iou_exact(a, b) > thr;
  const float q = __fdividef((float)(iw * ih), (float)uni);
  const float t = (float)thr;
  if (q > t + 1e-5f) return true;
  if (q < t - 1e-5f) return false;
  return iou_exact(a, b) > thr;
}

struct NmsKey {
  double score;
  unsigned long long t1, t2;  // (y, x) and (scale, rotation), sign-flipped for unsigned order
  int idx;
  int pad;
};
static_assert(sizeof(NmsKey) == sizeof(DevDet), "sorted detections reuse the key slots");

// detector.cpp:125-129: score descending, then (y, x, scale_index, rotation_index) ascending.
// Branch-free (the sort's compare-exchanges are warp-wide: a data-dependent branch chain
// serialised the lanes); same result as the chain of "if different, compare" tests.
BL_DEV bool before(const NmsKey& a, const NmsKey& b) {
  const bool sg = a.score > b.score, se = a.score == b.score;
  const bool t1l = a.t1 < b.t1, t1e = a.t1 == b.t1;
  const bool t2l = a.t2 < b.t2, t2e = a.t2 == b.t2;
  return sg | (se & (t1l | (t1e & (t2l | (t2e & (a.idx < b.idx))))));
}

BL_DEV unsigned long long pack2(int hi, int lo) {
  return ((unsigned long long)((unsigned)hi ^ 0x80000000u) << 32) | (unsigned)(lo ^ 0x80000000);
}

constexpr int kNmsSmemKeys = 512;    // keys sorted in shared memory up to this count
constexpr int kNmsSmemKept = 256;    // kept boxes cached in shared memory
constexpr int kNmsSmallFrames = 32;  // batches up to this many frames use k_nms_small

// One CTA per frame: bitonic sort of the frame's detections, then the greedy scan by
// warp 0 (kept boxes checked 32 at a time with __any_sync).
// (the per-frame body, also run by k_nms_small for a frame above its shared-memory limit)
__device__ __forceinline__ void nms_frame(const DevDet* __restrict__ dets, long long cap_pf, double iou_thr,
                                          DevDet* __restrict__ kept_out, int* __restrict__ kept_count,
                                          NmsKey* __restrict__ gkeys, long long gkeys_pf, int f, int n) {
  extern __shared__ unsigned char nms_smem[];
  const DevDet* D = dets + (long long)f * cap_pf;
  if (n == 0) {
    if (threadIdx.x == 0) kept_count[f] = 0;
    return;
  }
  int Pn = 1;
  while (Pn < n) Pn <<= 1;
  NmsKey* keys = Pn <= kNmsSmemKeys ? reinterpret_cast<NmsKey*>(nms_smem) : gkeys + (long long)f * gkeys_pf;
  DevDet* kept_s = reinterpret_cast<DevDet*>(nms_smem + sizeof(NmsKey) * kNmsSmemKeys);
  for (int i = threadIdx.x; i < Pn; i += blockDim.x) {
    NmsKey k;
    if (i < n) {
      const DevDet d = D[i];
      k.score = d.score;
      k.t1 = pack2(d.y, d.x);
      k.t2 = pack2(d.scale_index, d.rotation_index);
      k.idx = i;
    } else {
      k.score = -DBL_MAX;
      k.t1 = k.t2 = ~0ull;
      k.idx = 0x7fffffff;
    }
    k.pad = 0;
    keys[i] = k;
  }
  __syncthreads();
  for (int k = 2; k <= Pn; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < Pn; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const NmsKey a = keys[i], b = keys[ixj];
          const bool up = (i & k) == 0;
          if (up ? before(b, a) : before(a, b)) {
            keys[i] = b;
            keys[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  // gather the detections in sorted order next to the SM (in place of their keys when those
  // live in shared memory: same 32-B size, each thread reads its own key before overwriting
  // it), so the serial greedy scan below reads shared memory, not scattered global lines
  const bool smem_sorted = Pn <= kNmsSmemKeys;
  DevDet* sorted = reinterpret_cast<DevDet*>(keys);
  if (smem_sorted) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int idx = keys[i].idx;
      sorted[i] = D[idx];
    }
    __syncthreads();
  }
  DevDet* out = kept_out + (long long)f * cap_pf;
  if (smem_sorted) {
    // Warp-batched form of the greedy scan (detector.cpp:130-140): 32 boxes of the order at a
    // time.  Each lane tests its box against every box kept so far and against the earlier
    // boxes of its batch; the batch is then resolved in order with bit operations (box j is
    // kept iff no kept box suppresses it and no earlier KEPT box of the batch overlaps it) --
    // exactly the sequential scan's decisions, in its order.
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    int kept = 0;
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const bool valid = i < n;
      const DevDet d = sorted[valid ? i : n - 1];
      bool sup = !valid;
      for (int k = 0; k < kept && !sup; ++k) {
        const DevDet kb = k < kNmsSmemKept ? kept_s[k] : out[k];
        if (iou_exceeds(d, kb, iou_thr)) sup = true;
      }
      uint32_t ovl = 0;  // bit j: earlier batch box j overlaps this box
#pragma unroll 4
      for (int jj = 0; jj < 31; ++jj) {
        DevDet o;
        o.x = __shfl_sync(0xffffffffu, d.x, jj);
        o.y = __shfl_sync(0xffffffffu, d.y, jj);
        o.w = __shfl_sync(0xffffffffu, d.w, jj);
        o.h = __shfl_sync(0xffffffffu, d.h, jj);
        if (jj < lane && iou_exceeds(d, o, iou_thr)) ovl |= 1u << jj;
      }
      const uint32_t alive = __ballot_sync(0xffffffffu, !sup);
      uint32_t keep = 0;
      for (int jj = 0; jj < 32; ++jj) {
        const uint32_t oj = __shfl_sync(0xffffffffu, ovl, jj);
        if (((alive >> jj) & 1u) && !(oj & keep)) keep |= 1u << jj;
      }
      if ((keep >> lane) & 1u) {
        const int pos = kept + __popc(keep & ((1u << lane) - 1u));
        out[pos] = d;
        if (pos < kNmsSmemKept) kept_s[pos] = d;
      }
      kept += __popc(keep);
      __syncwarp();
    }
    if (lane == 0) kept_count[f] = kept;
    return;
  }
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int kept = 0;
  for (int i = 0; i < n; ++i) {
    const DevDet d = smem_sorted ? sorted[i] : D[keys[i].idx];
    bool sup = false;
    for (int k = lane; k < kept; k += 32) {
      const DevDet kb = k < kNmsSmemKept ? kept_s[k] : out[k];
      if (iou_exceeds(d, kb, iou_thr)) sup = true;  // detector.cpp:134
    }
    if (!__any_sync(0xffffffffu, sup)) {
      if (lane == 0) {
        out[kept] = d;
        if (kept < kNmsSmemKept) kept_s[kept] = d;
      }
      ++kept;
      __syncwarp();
    }
  }
  if (lane == 0) kept_count[f] = kept;
}

__global__ void __launch_bounds__(256) k_nms(const DevDet* __restrict__ dets,
                                             const int* __restrict__ det_count, long long cap_pf,
                                             double iou_thr, DevDet* __restrict__ kept_out,
                                             int* __restrict__ kept_count, NmsKey* __restrict__ gkeys,
                                             long long gkeys_pf) {
  const int f = blockIdx.x;
  const int n = (int)min((long long)det_count[f], cap_pf);
  nms_frame(dets, cap_pf, iou_thr, kept_out, kept_count, gkeys, gkeys_pf, f, n);
}

// NMS for SMALL batches (one frame, a 16-frame camera stream): one 1024-thread CTA per frame
// with up to kNmsSmallMax detections sorted in shared memory, and the greedy scan
// (detector.cpp:130-140) in rounds over the whole CTA: the next <= 32 boxes of the order that
// no kept box suppresses so far are resolved among themselves in order (a 32 x 32 overlap
// matrix, one IoU per thread, then a 32-step bit scan), and every later box is tested against
// the round's newly kept boxes in parallel.  Rounds ~ kept / batch, not n, so a frame with
// a thousand raw detections and a handful of faces takes a few microseconds.
constexpr int kNmsSmallMax = 2048;
#ifndef BL_NMS_SMALL_THREADS
#define BL_NMS_SMALL_THREADS 256  // (1024: barriers over 32 warps dominated a 200-box frame)
#endif
constexpr int kNmsSmallThreads = BL_NMS_SMALL_THREADS;
#ifndef BL_NMS_RANK
#define BL_NMS_RANK 1  // k_nms_small: rank sort for n <= kNmsSmallThreads (0: always bitonic)
#endif

size_t nms_small_smem_bytes() {
  return sizeof(NmsKey) * kNmsSmallMax + sizeof(uint32_t) * (kNmsSmallMax / 32 + 32 + 32 + 8);
}

__global__ void __launch_bounds__(kNmsSmallThreads) k_nms_small(const DevDet* __restrict__ dets,
                                                                const int* __restrict__ det_count, long long cap_pf,
                                                                double iou_thr, DevDet* __restrict__ kept_out,
                                                                int* __restrict__ kept_count,
                                                                NmsKey* __restrict__ gkeys, long long gkeys_pf) {
  extern __shared__ __align__(16) unsigned char nsm[];
  NmsKey* keys = reinterpret_cast<NmsKey*>(nsm);
  DevDet* sorted = reinterpret_cast<DevDet*>(nsm);  // gathered in place of the keys
  uint32_t* supp = reinterpret_cast<uint32_t*>(nsm + sizeof(NmsKey) * kNmsSmallMax);  // processed / suppressed
  int* cand = reinterpret_cast<int*>(supp + kNmsSmallMax / 32);                         // [32]
  uint32_t* ovl = reinterpret_cast<uint32_t*>(cand + 32);                               // [32]
  int* ctl = reinterpret_cast<int*>(ovl + 32);  // [0] candidates, [1] kept so far, [2] keep mask, [3] next p
  const int f = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = (int)min((long long)det_count[f], cap_pf);
  if (n > kNmsSmallMax) {  // beyond the shared-memory sort: k_nms's body (keys in global memory)
    nms_frame(dets, cap_pf, iou_thr, kept_out, kept_count, gkeys, gkeys_pf, f, n);
    return;
  }
  if (n == 0) {
    if (tid == 0) kept_count[f] = 0;
    return;
  }
  const DevDet* D = dets + (long long)f * cap_pf;
  int Pn = 1;
  while (Pn < n) Pn <<= 1;
  for (int i = tid; i < Pn; i += blockDim.x) {
    NmsKey k;
    if (i < n) {
      const DevDet d = D[i];
      k.score = d.score;
      k.t1 = pack2(d.y, d.x);
      k.t2 = pack2(d.scale_index, d.rotation_index);
      k.idx = i;
    } else {
      k.score = -DBL_MAX;
      k.t1 = k.t2 = ~0ull;
      k.idx = 0x7fffffff;
    }
    k.pad = 0;
    keys[i] = k;
  }
  for (int i = tid; i < kNmsSmallMax / 32; i += blockDim.x) supp[i] = 0u;
  __syncthreads();
  if (BL_NMS_RANK && n <= kNmsSmallThreads) {
    // up to a block's worth of boxes (a frame's few hundred raw detections): rank sort -- box i
    // goes to the number of boxes ordered before it (the keys are distinct, so the ranks are a
    // permutation); every thread streams all keys (broadcast reads) with no barrier in between,
    // where the bitonic network's 36 dependent passes cost ~15 us for 256 keys
    int rank = 0;
    if (tid < n) {
      const NmsKey me = keys[tid];
      for (int j = 0; j < n; ++j) rank += before(keys[j], me) ? 1 : 0;
    }
    __syncthreads();  // every key read before the gather overwrites them
    if (tid < n) sorted[rank] = D[tid];
    if (tid == 0) {
      ctl[1] = 0;
      ctl[3] = 0;
    }
    __syncthreads();
  } else {
  for (int k = 2; k <= Pn; k <<= 1) {  // bitonic sort, detector.cpp:125-129 order
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < Pn; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const NmsKey a = keys[i], b = keys[ixj];
          const bool up = (i & k) == 0;
          if (up ? before(b, a) : before(a, b)) {
            keys[i] = b;
            keys[ixj] = a;
          }
        }
      }
      // a pass whose partner distance is below 32 stays inside each warp's 32-element slices,
      // so between two such passes a warp barrier suffices; a pass on either side of the
      // barrier that crosses warps needs the block barrier
      const int next_j = j > 1 ? j >> 1 : k;
      if (j < 32 && next_j < 32)
        __syncwarp();
      else
        __syncthreads();
    }
  }
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) {  // each thread reads its own key before overwriting it
    const int idx = keys[i].idx;
    sorted[i] = D[idx];
  }
  if (tid == 0) {
    ctl[1] = 0;
    ctl[3] = 0;
  }
  __syncthreads();
  }
  DevDet* out = kept_out + (long long)f * cap_pf;
  const int nwords = (n + 31) >> 5;
  while (true) {
    const int p = ctl[3];
    if (warp == 0) {  // the next <= 32 unprocessed boxes at or after p, in order
      const int w = (p >> 5) + lane;
      uint32_t free_bits = 0;
      if (w < nwords) {
        free_bits = ~supp[w];
        if (w == (p >> 5)) free_bits &= ~0u << (p & 31);
        if (w == nwords - 1 && (n & 31)) free_bits &= (1u << (n & 31)) - 1u;
      }
      const int cnt = __popc(free_bits);
      int pre = cnt;  // inclusive prefix over lanes
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += v;
      }
      int pos = pre - cnt;
      while (free_bits && pos < 32) {
        cand[pos++] = (w << 5) + __ffs(free_bits) - 1;
        free_bits &= free_bits - 1;
      }
      const int tot = __shfl_sync(0xffffffffu, pre, 31);
      if (lane == 0) ctl[0] = min(tot, 32);
    }
    __syncthreads();
    const int nc = ctl[0];
    if (nc == 0) break;
    for (int a = warp; a < 32; a += kNmsSmallThreads / 32) {  // overlap matrix of the candidates: row a, lane b < a
      const int b = lane;
      bool o = false;
      if (a < nc && b < a) o = iou_exceeds(sorted[cand[b]], sorted[cand[a]], iou_thr);
      const uint32_t m = __ballot_sync(0xffffffffu, o);
      if (lane == 0) ovl[a] = m;
    }
    __syncthreads();
    if (warp == 0) {  // resolve the batch in order (a register recurrence over the shuffled
                      // overlap rows), then every candidate lane marks itself processed and the
                      // kept ones store themselves at their rank
      const uint32_t my_ovl = lane < nc ? ovl[lane] : 0u;
      uint32_t keep = 0;
      for (int a = 0; a < nc; ++a) {
        const uint32_t oa = __shfl_sync(0xffffffffu, my_ovl, a);
        if (!(oa & keep)) keep |= 1u << a;
      }
      const int kept0 = ctl[1];
      if (lane < nc) {
        const int ci = cand[lane];
        atomicOr(&supp[ci >> 5], 1u << (ci & 31));
        if ((keep >> lane) & 1u) out[kept0 + __popc(keep & ((1u << lane) - 1u))] = sorted[ci];
      }
      __syncwarp();
      if (lane == 0) {
        ctl[1] = kept0 + __popc(keep);
        ctl[2] = (int)keep;
        ctl[3] = cand[nc - 1] + 1;
      }
    }
    __syncthreads();
    const uint32_t keep = (uint32_t)ctl[2];
    const int np = ctl[3];
    for (int j = np + tid; j < n; j += blockDim.x) {  // later boxes against the round's kept boxes
      if ((supp[j >> 5] >> (j & 31)) & 1u) continue;
      const DevDet dj = sorted[j];
      uint32_t kk = keep;
      while (kk) {
        const int a = __ffs(kk) - 1;
        kk &= kk - 1;
        if (iou_exceeds(sorted[cand[a]], dj, iou_thr)) {
          atomicOr(&supp[j >> 5], 1u << (j & 31));
          break;
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) kept_count[f] = ctl[1];
}

size_t nms_smem_bytes() { return sizeof(NmsKey) * kNmsSmemKeys + sizeof(DevDet) * kNmsSmemKept; }

long long nms_gkeys_per_frame(long long cap_pf) {
  long long p = 1;
  while (p < cap_pf) p <<= 1;
  return p > kNmsSmemKeys ? p : 0;
}

size_t nms_key_bytes() { return sizeof(NmsKey); }

void launch_nms(const Launch& L, const DevDet* dets, const int* det_count, long long cap_pf, int n_frames,
                double iou_thr, DevDet* kept_out, int* kept_count, void* gkeys, long long gkeys_pf) {
  if (n_frames <= 0) return;
  if (n_frames <= kNmsSmallFrames) {  // latency path (frames above its sort limit run k_nms's body)
    k_nms_small<<<n_frames, kNmsSmallThreads, nms_small_smem_bytes(), L.st>>>(dets, det_count, cap_pf, iou_thr,
                                                                               kept_out, kept_count, (NmsKey*)gkeys,
                                                                               gkeys_pf);
    ++*L.counter;
    return;
  }
  k_nms<<<n_frames, 256, nms_smem_bytes(), L.st>>>(dets, det_count, cap_pf, iou_thr, kept_out, kept_count,
                                                   (NmsKey*)gkeys, gkeys_pf);
  ++*L.counter;
}

// ------------------------------------------------- kept detections -> flat face list ----
// One CTA: prefix sum of kept counts (frame order), then every kept detection is copied to a
// flat array (the order a sequential per-frame loop produces) together with its frame index.
__global__ void __launch_bounds__(1024) k_flatten(const DevDet* __restrict__ kept,
                                                  const int* __restrict__ kept_count, long long cap_pf,
                                                  int n_frames, int* __restrict__ offsets,
                                                  DevDet* __restrict__ flat, int* __restrict__ face_frame,
                                                  int* __restrict__ meta, long long flat_cap,
                                                  const int* __restrict__ raw_overflow, DevDet* __restrict__ best,
                                                  int* __restrict__ best_frame) {
  // meta: [0, n) kept count per frame, [n] total kept, [n+1] raw-detection overflow flag
  __shared__ int s_part[1024];
  const int tid = threadIdx.x;
  // each thread scans a contiguous chunk of frames
  const int per = (n_frames + blockDim.x - 1) / blockDim.x;
  const int f0 = min(n_frames, tid * per), f1 = min(n_frames, f0 + per);
  int sum = 0;
  for (int f = f0; f < f1; ++f) sum += kept_count[f];
  s_part[tid] = sum;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {
    const int v = tid >= o ? s_part[tid - o] : 0;
    __syncthreads();
    s_part[tid] += v;
    __syncthreads();
  }
  int run = s_part[tid] - sum;
  for (int f = f0; f < f1; ++f) {
    offsets[f] = run;
    meta[f] = kept_count[f];
    run += kept_count[f];
  }
  if (tid == blockDim.x - 1) {
    offsets[n_frames] = s_part[tid];
    meta[n_frames] = s_part[tid];
    meta[n_frames + 1] = *raw_overflow;
    meta[n_frames + 2] = 0;  // the landmark cascade's error flag (the cascade runs after this kernel)
    meta[n_frames + 3] = n_frames;  // faces of the best-detection landmark list
  }
  if (best) {  // the face of every frame = its first kept detection (pipeline.cpp:167); a frame
               // without one gets a placeholder box whose landmarks nobody reads
    for (int f = tid; f < n_frames; f += blockDim.x) {
      DevDet d;
      if (kept_count[f] > 0) {
        d = kept[(long long)f * cap_pf];
      } else {
        d.x = d.y = 0;
        d.w = d.h = 1;
        d.score = 0.0;
        d.scale_index = d.rotation_index = 0;
      }
      best[f] = d;
      best_frame[f] = f;
    }
  }
  __syncthreads();
  // copy: warp per frame
  const int lane = tid & 31;
  for (int f = tid >> 5; f < n_frames; f += blockDim.x >> 5) {
    const int c = kept_count[f];
    const int o = offsets[f];
    for (int k = lane; k < c; k += 32) {
      if (o + k < flat_cap) {
        flat[o + k] = kept[(long long)f * cap_pf + k];
        face_frame[o + k] = f;
      }
    }
  }
}

void launch_flatten(const Launch& L, const DevDet* kept, const int* kept_count, long long cap_pf,
                    int n_frames, int* offsets, DevDet* flat, int* face_frame, int* meta,
                    long long flat_cap, const int* raw_overflow, DevDet* best, int* best_frame) {
  // block size by batch: the scan is log2(threads) barrier steps (one frame: 32 threads, one
  // warp-sized scan, instead of 1024 threads and ten barriers -- C1 flatten 4.6 us)
  const int threads = n_frames == 1 ? 32 : (n_frames <= 256 ? 256 : 1024);  // (C2's 16 frames: 32 -> 7.8 us)
  k_flatten<<<1, threads, 0, L.st>>>(kept, kept_count, cap_pf, n_frames, offsets, flat, face_frame, meta,
                                     flat_cap, raw_overflow, best, best_frame);
  ++*L.counter;
}

void configure_exact_kernels(int optin) {  // per device, see configure_screen_tc_kernels
  smem_optin(k_rescore, optin);
  smem_optin(k_nms, optin);
  smem_optin(k_nms_small, optin);
}

}  // namespace blb
