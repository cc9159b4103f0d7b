// Pyramid resample: one 5/6 bilinear step per launch, all frames of the batch at once
// (grid.z = frame -- the paper's multi-image batching).
//
// Follows downscale_bilinear (image.cpp:129-156) operation for operation; compiled with
// --fmad=false and written with _rn intrinsics, so every level is bit-identical to the
// reference's chain.  Level 0 may be u8 (integral frames) or fp64; levels >= 1 are fp64,
// which parity requires (an fp32 pyramid flips ~740 orientations/frame).
//
// Roofline: HBM-bound.  Algorithmic bytes per output pixel: 8 B written + the source
// level read once (1 B/px for u8 level 0, 8 B/px otherwise, 1.44 source px per output px).
#include <cooperative_groups.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "bl_internal.cuh"

namespace blb {

#ifndef BL_RS_ROWS
#define BL_RS_ROWS 4
#endif
constexpr int kRsRows = BL_RS_ROWS;  // output rows per thread (column terms computed once)
#ifndef BL_RS_PAIRS
#define BL_RS_PAIRS 1
#endif
constexpr bool kRsPairs = BL_RS_PAIRS;  // k_resample2 where the destination allows
#ifndef BL_RS_COLS
#define BL_RS_COLS 2
#endif
constexpr int kRsCols = BL_RS_COLS;  // output columns per k_resample2 thread (2 or 4)
#ifndef BL_RS_TALL
#define BL_RS_TALL 8  // output rows per k_resample2 thread for large levels
#endif

template <typename Tin>
__global__ void __launch_bounds__(256) k_resample(const Tin* __restrict__ src, int sw, int sh,
                                                  long long s_pitch, long long s_fstride,
                                                  double* __restrict__ dst, int dw, int dh, long long d_pitch,
                                                  long long d_fstride, double rx, double ry) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y_first = (blockIdx.y * blockDim.y + threadIdx.y) * kRsRows;
  if (x >= dw || y_first >= dh) return;
  const Tin* s = src + (long long)blockIdx.z * s_fstride;
  double* d = dst + (long long)blockIdx.z * d_fstride;
  // image.cpp:145-149 (rx = double(w)/dw is computed on the host, the same IEEE division)
  double sx = dsub(dmul(dadd((double)x, 0.5), rx), 0.5);
  const double xmax = (double)(sw - 1);
  sx = sx < 0.0 ? 0.0 : (xmax < sx ? xmax : sx);
  const int x0 = (int)sx;
  const int x1 = min(x0 + 1, sw - 1);
  const double fx = dsub(sx, (double)x0);
  const double gx = dsub(1.0, fx);
  const double ymax = (double)(sh - 1);
#pragma unroll
  for (int j = 0; j < kRsRows; ++j) {
    const int y = y_first + j;
    if (y >= dh) break;
    // image.cpp:139-143
    double sy = dsub(dmul(dadd((double)y, 0.5), ry), 0.5);
    sy = sy < 0.0 ? 0.0 : (ymax < sy ? ymax : sy);
    const int y0 = (int)sy;
    const int y1 = min(y0 + 1, sh - 1);
    const double fy = dsub(sy, (double)y0);
    // image.cpp:150-152
    const double a = (double)__ldg(s + y0 * s_pitch + x0);
    const double b = (double)__ldg(s + y0 * s_pitch + x1);
    const double c = (double)__ldg(s + y1 * s_pitch + x0);
    const double e = (double)__ldg(s + y1 * s_pitch + x1);
    const double top = dadd(dmul(a, gx), dmul(b, fx));
    const double bot = dadd(dmul(c, gx), dmul(e, fx));
    d[(long long)y * d_pitch + x] = dadd(dmul(top, dsub(1.0, fy)), dmul(bot, fy));
  }
}

// NC adjacent output columns per thread (16-B stores): the row terms computed once per NC
// columns.  Needs 16-B aligned destination rows (the plan's arena).
template <typename Tin, int NC, int ROWS = kRsRows>
__global__ void __launch_bounds__(256) k_resample2(const Tin* __restrict__ src, int sw, int sh,
                                                   long long s_pitch, long long s_fstride,
                                                   double* __restrict__ dst, int dw, int dh, long long d_pitch,
                                                   long long d_fstride, double rx, double ry) {
  const int x = NC * (blockIdx.x * blockDim.x + threadIdx.x);
  const int y_first = (blockIdx.y * blockDim.y + threadIdx.y) * ROWS;
  if (x >= dw || y_first >= dh) return;
  const Tin* s = src + (long long)blockIdx.z * s_fstride;
  double* d = dst + (long long)blockIdx.z * d_fstride;
  const double xmax = (double)(sw - 1);
  int x0[NC], x1[NC];
  double fx[NC], gx[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) {  // image.cpp:145-149
    double sx = dsub(dmul(dadd((double)(x + q), 0.5), rx), 0.5);
    sx = sx < 0.0 ? 0.0 : (xmax < sx ? xmax : sx);
    x0[q] = (int)sx;
    x1[q] = min(x0[q] + 1, sw - 1);
    fx[q] = dsub(sx, (double)x0[q]);
    gx[q] = dsub(1.0, fx[q]);
  }
  const double ymax = (double)(sh - 1);
#pragma unroll
  for (int j = 0; j < ROWS; ++j) {
    const int y = y_first + j;
    if (y >= dh) break;
    double sy = dsub(dmul(dadd((double)y, 0.5), ry), 0.5);  // image.cpp:139-143
    sy = sy < 0.0 ? 0.0 : (ymax < sy ? ymax : sy);
    const int y0 = (int)sy;
    const int y1 = min(y0 + 1, sh - 1);
    const double fy = dsub(sy, (double)y0);
    const double gy = dsub(1.0, fy);
    const Tin* r0 = s + y0 * s_pitch;
    const Tin* r1 = s + y1 * s_pitch;
    double o[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {  // image.cpp:150-152
      const double a = (double)__ldg(r0 + x0[q]), b = (double)__ldg(r0 + x1[q]);
      const double c = (double)__ldg(r1 + x0[q]), e = (double)__ldg(r1 + x1[q]);
      const double top = dadd(dmul(a, gx[q]), dmul(b, fx[q]));
      const double bot = dadd(dmul(c, gx[q]), dmul(e, fx[q]));
      o[q] = dadd(dmul(top, gy), dmul(bot, fy));
    }
    double* out = d + (long long)y * d_pitch + x;
#pragma unroll
    for (int q = 0; q < NC; q += 2) {
      if (x + q + 1 < dw)
        *reinterpret_cast<double2*>(out + q) = make_double2(o[q], o[q + 1]);
      else if (x + q < dw)
        out[q] = o[q];
    }
  }
}

// Two chained steps in one pass, for a level nobody but the next step reads (a level below
// the smallest eligible face size: C5 levels 1-5, C3 1-3): each CTA computes the
// region of the intermediate level m its output tile needs into shared memory (from level
// k-1, the same arithmetic as k_resample, so every value is bit-identical wherever it is
// computed -- ~14% of them twice at tile borders), then the tile of level k+1 from it.  Level
// m never reaches HBM: its write and re-read (the bulk of the pyramid's bytes at 1080p) go.
constexpr int kPrTX = 64, kPrTY = 32;  // output tile of level k+1

BL_DEV void resample_coord(int x, double r, int n_src, int& x0, int& x1, double& f) {  // image.cpp:139-149
  double sx = dsub(dmul(dadd((double)x, 0.5), r), 0.5);
  const double xmax = (double)(n_src - 1);
  sx = sx < 0.0 ? 0.0 : (xmax < sx ? xmax : sx);
  x0 = (int)sx;
  x1 = min(x0 + 1, n_src - 1);
  f = dsub(sx, (double)x0);
}

BL_DEV double bilerp(double a, double b, double c, double e, double fx, double fy) {  // image.cpp:150-152
  const double top = dadd(dmul(a, dsub(1.0, fx)), dmul(b, fx));
  const double bot = dadd(dmul(c, dsub(1.0, fx)), dmul(e, fx));
  return dadd(dmul(top, dsub(1.0, fy)), dmul(bot, fy));
}

template <typename Tin>
__global__ void __launch_bounds__(256) k_resample_pair(const Tin* __restrict__ src, int sw, int sh, long long s_pitch,
                                                       long long s_fstride, int mw, int mh, double rx1, double ry1,
                                                       double* __restrict__ dst, int dw, int dh, long long d_pitch,
                                                       long long d_fstride, double rx2, double ry2) {
  extern __shared__ double mid[];
  const int X0 = blockIdx.x * kPrTX, Y0 = blockIdx.y * kPrTY;
  const int X1 = min(X0 + kPrTX, dw) - 1, Y1 = min(Y0 + kPrTY, dh) - 1;
  const Tin* s = src + (long long)blockIdx.z * s_fstride;
  double* d = dst + (long long)blockIdx.z * d_fstride;
  // the intermediate region [mx_lo, mx_hi] x [my_lo, my_hi] the tile's taps touch (x0 and x1
  // are non-decreasing in the output coordinate)
  int mx_lo, mx_hi, my_lo, my_hi, t0;
  double tf;
  resample_coord(X0, rx2, mw, mx_lo, t0, tf);
  resample_coord(X1, rx2, mw, t0, mx_hi, tf);
  resample_coord(Y0, ry2, mh, my_lo, t0, tf);
  resample_coord(Y1, ry2, mh, t0, my_hi, tf);
  const int RW = mx_hi - mx_lo + 1, RH = my_hi - my_lo + 1;
  // 32 x 8 threads: a thread owns columns tx, tx + 32, ... and rows ty, ty + 8, ... of each
  // phase, so its column terms are computed once per column, its row terms once per row
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  constexpr int kCols1 = 4;  // region columns per thread (RW <= 128 for rx < 2)
  int cx0[kCols1], cx1[kCols1];
  double cfx[kCols1];
#pragma unroll
  for (int q = 0; q < kCols1; ++q) resample_coord(min(mx_lo + tx + 32 * q, mx_hi), rx1, sw, cx0[q], cx1[q], cfx[q]);
  for (int r = ty; r < RH; r += 8) {
    int y0, y1;
    double fy;
    resample_coord(my_lo + r, ry1, sh, y0, y1, fy);
    const Tin* r0 = s + y0 * s_pitch;
    const Tin* r1 = s + y1 * s_pitch;
#pragma unroll
    for (int q = 0; q < kCols1; ++q) {
      const int c = tx + 32 * q;
      if (c < RW)
        mid[r * RW + c] = bilerp((double)__ldg(r0 + cx0[q]), (double)__ldg(r0 + cx1[q]), (double)__ldg(r1 + cx0[q]),
                                 (double)__ldg(r1 + cx1[q]), cfx[q], fy);
    }
  }
  __syncthreads();
  const int TW = X1 - X0 + 1, TH = Y1 - Y0 + 1;
  constexpr int kCols2 = kPrTX / 32;
  int ox0[kCols2], ox1[kCols2];
  double ofx[kCols2];
#pragma unroll
  for (int q = 0; q < kCols2; ++q) {
    resample_coord(X0 + min(tx + 32 * q, TW - 1), rx2, mw, ox0[q], ox1[q], ofx[q]);
    ox0[q] -= mx_lo;
    ox1[q] -= mx_lo;
  }
  for (int r = ty; r < TH; r += 8) {
    int y0, y1;
    double fy;
    resample_coord(Y0 + r, ry2, mh, y0, y1, fy);
    const double* m0 = mid + (y0 - my_lo) * RW;
    const double* m1 = mid + (y1 - my_lo) * RW;
    double* out = d + (long long)(Y0 + r) * d_pitch + X0;
#pragma unroll
    for (int q = 0; q < kCols2; ++q) {
      const int c = tx + 32 * q;
      if (c < TW) out[c] = bilerp(m0[ox0[q]], m0[ox1[q]], m1[ox0[q]], m1[ox1[q]], ofx[q], fy);
    }
  }
}

bool resample_pair_fits(int sw, int sh, int mw, int mh, int dw, int dh) {
  // ratios < 1.9: a tile's region stays within 4 x 32 columns (floor(63 * r) + 4 <= 123)
  return 10LL * sw < 19LL * mw && 10LL * sh < 19LL * mh && 10LL * mw < 19LL * dw && 10LL * mh < 19LL * dh;
}

void launch_resample_pair(const Launch& L, const void* src, int src_u8, int sw, int sh, long long s_pitch,
                          long long s_fstride, int mw, int mh, double* dst, int dw, int dh, long long d_pitch,
                          long long d_fstride, int n) {
  const double rx1 = double(sw) / mw, ry1 = double(sh) / mh;  // image.cpp:136-137, each step
  const double rx2 = double(mw) / dw, ry2 = double(mh) / dh;
  const dim3 grid((unsigned)div_up(dw, kPrTX), (unsigned)div_up(dh, kPrTY), (unsigned)n);
  // region bound: floor((T - 1) * r) + 3 taps, +1 for the rounding of the computed coordinate
  const int rw = (int)((kPrTX - 1) * rx2) + 4, rh = (int)((kPrTY - 1) * ry2) + 4;
  const size_t smem = sizeof(double) * rw * rh;
  if (src_u8)
    k_resample_pair<uint8_t><<<grid, 256, smem, L.st>>>((const uint8_t*)src, sw, sh, s_pitch, s_fstride, mw, mh, rx1,
                                                        ry1, dst, dw, dh, d_pitch, d_fstride, rx2, ry2);
  else
    k_resample_pair<double><<<grid, 256, smem, L.st>>>((const double*)src, sw, sh, s_pitch, s_fstride, mw, mh, rx1,
                                                       ry1, dst, dw, dh, d_pitch, d_fstride, rx2, ry2);
  ++*L.counter;
}

void launch_resample(const Launch& L, const void* src, int src_u8, int sw, int sh, long long s_pitch,
                     long long s_fstride, double* dst, int dw, int dh, long long d_pitch, long long d_fstride,
                     int n) {
  const double rx = double(sw) / dw, ry = double(sh) / dh;  // image.cpp:136-137
  const dim3 block(32, 8);
  const bool vec = ((uintptr_t)dst & 15) == 0 && d_pitch % 2 == 0 && d_fstride % 2 == 0;
  if (vec && kRsPairs) {
    // large levels (the bench's 512 frames): 8 output rows per thread (pyramid 1.27 -> 1.24 ms
    // per step); small ones keep 4 for more threads (C2's 16 frames: 0.040 vs 0.049 ms)
    const bool tall = (long long)n * dw * dh >= (8LL << 20);
    const int rows = tall ? BL_RS_TALL : kRsRows;
    const dim3 grid2((unsigned)div_up(dw, 32 * kRsCols), (unsigned)div_up(dh, 8 * rows), (unsigned)n);
    if (src_u8) {
      if (tall)
        k_resample2<uint8_t, kRsCols, BL_RS_TALL><<<grid2, block, 0, L.st>>>((const uint8_t*)src, sw, sh, s_pitch, s_fstride,
                                                                    dst, dw, dh, d_pitch, d_fstride, rx, ry);
      else
        k_resample2<uint8_t, kRsCols><<<grid2, block, 0, L.st>>>((const uint8_t*)src, sw, sh, s_pitch, s_fstride, dst,
                                                                 dw, dh, d_pitch, d_fstride, rx, ry);
    } else {
      if (tall)
        k_resample2<double, kRsCols, BL_RS_TALL><<<grid2, block, 0, L.st>>>((const double*)src, sw, sh, s_pitch, s_fstride,
                                                                   dst, dw, dh, d_pitch, d_fstride, rx, ry);
      else
        k_resample2<double, kRsCols><<<grid2, block, 0, L.st>>>((const double*)src, sw, sh, s_pitch, s_fstride, dst,
                                                                dw, dh, d_pitch, d_fstride, rx, ry);
    }
    ++*L.counter;
    return;
  }
  const dim3 grid((unsigned)div_up(dw, 32), (unsigned)div_up(dh, 8 * kRsRows), (unsigned)n);
  if (src_u8)
    k_resample<uint8_t><<<grid, block, 0, L.st>>>((const uint8_t*)src, sw, sh, s_pitch, s_fstride, dst, dw, dh,
                                                   d_pitch, d_fstride, rx, ry);
  else
    k_resample<double><<<grid, block, 0, L.st>>>((const double*)src, sw, sh, s_pitch, s_fstride, dst, dw, dh,
                                                  d_pitch, d_fstride, rx, ry);
  ++*L.counter;
}

// The whole chain for SMALL batches (one frame, a 16-frame camera stream): each step is too
// small to fill the GPU and its cost is launch + drain latency, so every level is produced
// by ONE cooperative launch, a grid-stride pass per level with a grid barrier between levels
// (level k reads level k-1).  Per pixel the same arithmetic as k_resample (bit-identical).
namespace cg = cooperative_groups;
#ifndef BL_PYR_CHAIN_CTAS_DEFAULT
#define BL_PYR_CHAIN_CTAS_DEFAULT 2  // C1 chain 25.0 (1) -> 22.1 (2) -> 25.7 us (4)
#endif

template <typename T0>
__global__ void __launch_bounds__(256) k_pyramid_chain(const PyrChain C) {
  cg::grid_group grid = cg::this_grid();
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (blockIdx.x == 0 && C.zero_i32) {  // read by kernels after this one in the stream
    for (int i = threadIdx.x; i < C.n_zero_i32; i += blockDim.x) C.zero_i32[i] = 0;
    if (threadIdx.x == 0) {
      *C.zero_u64 = 0ull;
      *C.zero_flag = 0;
    }
  }
  for (int k = 1; k < C.n_levels; ++k) {
    const int sw = C.lw[k - 1], sh = C.lh[k - 1], dw = C.lw[k], dh = C.lh[k];
    const double rx = C.rx[k], ry = C.ry[k];
    const double xmax = (double)(sw - 1), ymax = (double)(sh - 1);
    // 32-bit index math (a one-frame pyramid is < 2^31 pixels per level; kChainMaxPx): the
    // 64-bit division per pixel was a software routine
    const unsigned plane = (unsigned)dh * (unsigned)dw, total = (unsigned)C.n_frames * plane;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (unsigned)stride) {
      const unsigned f = C.n_frames == 1 ? 0u : i / plane;
      const unsigned rem = i - f * plane;
      const int y = (int)(rem / (unsigned)dw), x = (int)(rem - (unsigned)y * (unsigned)dw);
      double sx = dsub(dmul(dadd((double)x, 0.5), rx), 0.5);  // image.cpp:139-149
      sx = sx < 0.0 ? 0.0 : (xmax < sx ? xmax : sx);
      const int x0 = (int)sx, x1 = min(x0 + 1, sw - 1);
      const double fx = dsub(sx, (double)x0), gx = dsub(1.0, fx);
      double sy = dsub(dmul(dadd((double)y, 0.5), ry), 0.5);
      sy = sy < 0.0 ? 0.0 : (ymax < sy ? ymax : sy);
      const int y0 = (int)sy, y1 = min(y0 + 1, sh - 1);
      const double fy = dsub(sy, (double)y0), gy = dsub(1.0, fy);
      double a, b, c, e;
      if (k == 1) {
        const T0* s = reinterpret_cast<const T0*>(C.src0) + (long long)f * C.s0_fstride;
        a = (double)__ldg(s + y0 * C.s0_pitch + x0);
        b = (double)__ldg(s + y0 * C.s0_pitch + x1);
        c = (double)__ldg(s + y1 * C.s0_pitch + x0);
        e = (double)__ldg(s + y1 * C.s0_pitch + x1);
      } else {  // written by this launch: plain loads (not the read-only path)
        const double* s = C.lv[k - 1] + (long long)f * C.lfstride[k - 1];
        const long long p = C.lpitch[k - 1];
        a = s[y0 * p + x0];
        b = s[y0 * p + x1];
        c = s[y1 * p + x0];
        e = s[y1 * p + x1];
      }
      const double top = dadd(dmul(a, gx), dmul(b, fx));  // image.cpp:150-152
      const double bot = dadd(dmul(c, gx), dmul(e, fx));
      C.lv[k][(long long)f * C.lfstride[k] + (long long)y * C.lpitch[k] + x] = dadd(dmul(top, gy), dmul(bot, fy));
    }
    if (k + 1 < C.n_levels) grid.sync();
  }
}

int launch_pyramid_chain(const Launch& L, const PyrChain& C, int src_u8) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const void* fn = src_u8 ? (const void*)k_pyramid_chain<uint8_t> : (const void*)k_pyramid_chain<double>;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0);
  long long most = 0;  // the largest level's pixels: no more CTAs than it needs
  for (int k = 1; k < C.n_levels; ++k) most = std::max(most, (long long)C.n_frames * C.lw[k] * C.lh[k]);
  static const int cap_per_sm = [] {  // BL_PYR_CHAIN_CTAS: co-resident CTAs per SM (A/B)
    const char* e = std::getenv("BL_PYR_CHAIN_CTAS");
    return e ? std::max(1, std::atoi(e)) : BL_PYR_CHAIN_CTAS_DEFAULT;
  }();
  const unsigned grid = (unsigned)std::max<long long>(
      1, std::min<long long>((long long)sms * std::min(per_sm, cap_per_sm), div_up(most, 256)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = L.st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = src_u8 ? cudaLaunchKernelEx(&cfg, k_pyramid_chain<uint8_t>, C)
                               : cudaLaunchKernelEx(&cfg, k_pyramid_chain<double>, C);
  ++*L.counter;
  return e == cudaSuccess ? 0 : (int)e;
}

void configure_pyramid_kernels(int optin) {  // per device, see configure_screen_tc_kernels
  smem_optin(k_resample_pair<uint8_t>, optin);
  smem_optin(k_resample_pair<double>, optin);
}

}  // namespace blb
