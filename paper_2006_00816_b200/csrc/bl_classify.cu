// Sliding-window linear classifier, stage 1: the fp32 SCREEN (PAPER.md:559-579 recast).
//
// score(anchor, r) = sum over the 10x10x31 window of feature * W_r + bias_r is an implicit
// GEMM with K = 3100 and N = 5 filters.  This kernel evaluates it on the CUDA-core FMA pipe
// in fp32 with register tiling (each lane: 4 horizontally adjacent anchors x 5 filters, so
// every feature load feeds 50 FMAs and the sliding-window overlap is reused in registers)
// and emits as CANDIDATES every (anchor, filter) whose fp32 sum exceeds
//     cut_r = threshold - bias_r - delta_r,
// where delta_r is a rigorous bound on |fp32 sum - exact sum| (0 <= features
// <= 0.8486 by construction, per-window-row blocked accumulation -> error <= 324 u S with
// S <= 0.8486 ||W_r||_1).  Every candidate is re-scored exactly in fp64 by bl_exact.cu in
// the reference's separable order, so the detections that survive are bit-identical to the
// reference; nothing scored here reaches the output directly.
//
// This is the only translation unit compiled with FMA contraction.
//
// Roofline: FP32 FMA pipe (5 x 3100 FMA per anchor); features are read from L1/L2 as
// fp32 planes (algorithmic bytes: 124 B per cell read once + 16 B per candidate written).
#include "bl_internal.cuh"

namespace blb {

constexpr int kWBlock = 52;  // per (window row j, feature f): 10 cells x 5 filters, padded to 13 float4
constexpr int kScreenSmem = kWin * kFeat * kWBlock * (int)sizeof(float);  // 64,480 B

constexpr int kScreenWarps = 8;  // warps per CTA sharing one smem copy of the weights

__global__ void __launch_bounds__(kScreenWarps * 32, 2) k_screen(const PlanDesc* __restrict__ P, const LevelBegins B,
                                                const float* __restrict__ feat32,
                                                const float* __restrict__ w32,
                                                const float* __restrict__ cut,
                                                Candidate* __restrict__ cand,
                                                unsigned long long* __restrict__ n_cand,
                                                long long cap, long long total) {
  extern __shared__ float4 sW4[];
  {
    const float4* src = reinterpret_cast<const float4*>(w32);
    for (int i = threadIdx.x; i < kScreenSmem / 16; i += blockDim.x) sW4[i] = __ldg(src + i);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long wid = (long long)blockIdx.x * kScreenWarps + warp;
  if (wid >= total) return;
  const int s = find_level(B, wid);
  const LevelDesc& D = P->lv[s];
  const long long local = wid - D.sc_begin;
  const int tiles = D.sc_tiles_x * D.sc_tiles_y;
  const int f = (int)(local / tiles);
  const int t = (int)(local - (long long)f * tiles);
  const int x = (t % D.sc_tiles_x) * kTileAX + (lane & 7) * 4;
  const int y = (t / D.sc_tiles_x) * kTileAY + (lane >> 3);
  const int cw_pad = D.cw_pad;
  const long long plane = (long long)D.ch_pad * cw_pad;
  const float* fb = feat32 + D.f32_off + (long long)f * D.f32_fstride + x;

  float acc[4][kFilters];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int r = 0; r < kFilters; ++r) acc[q][r] = 0.f;

  // software pipeline: the next (j, f) feature vectors are in flight while the current
  // ones feed 200 FMAs
  const float* rowp0 = fb + (long long)y * cw_pad;
  float4 n0 = __ldg(reinterpret_cast<const float4*>(rowp0)), n1 = __ldg(reinterpret_cast<const float4*>(rowp0) + 1),
         n2 = __ldg(reinterpret_cast<const float4*>(rowp0) + 2), n3 = __ldg(reinterpret_cast<const float4*>(rowp0) + 3);
#pragma unroll 1
  for (int j = 0; j < kWin; ++j) {
    float aj[4][kFilters];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int r = 0; r < kFilters; ++r) aj[q][r] = 0.f;
    const float4* wj = sW4 + j * kFeat * (kWBlock / 4);
#pragma unroll 1
    for (int ff = 0; ff < kFeat; ++ff) {
      const float v[16] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w,
                           n2.x, n2.y, n2.z, n2.w, n3.x, n3.y, n3.z, n3.w};
      {  // prefetch (j, ff+1), or (j+1, 0); the last prefetch re-reads row y+9, harmlessly
        const int nf = ff + 1 < kFeat ? ff + 1 : 0;
        const int nj = ff + 1 < kFeat ? j : min(j + 1, kWin - 1);
        const float4* p = reinterpret_cast<const float4*>(fb + (long long)(y + nj) * cw_pad + nf * plane);
        n0 = __ldg(p);
        n1 = __ldg(p + 1);
        n2 = __ldg(p + 2);
        n3 = __ldg(p + 3);
      }
      const float4* wp = wj + ff * (kWBlock / 4);
      float wv[kWBlock];
#pragma unroll
      for (int k = 0; k < kWBlock / 4; ++k) {
        const float4 t4 = wp[k];
        wv[4 * k] = t4.x;
        wv[4 * k + 1] = t4.y;
        wv[4 * k + 2] = t4.z;
        wv[4 * k + 3] = t4.w;
      }
#pragma unroll
      for (int i = 0; i < kWin; ++i)
#pragma unroll
        for (int r = 0; r < kFilters; ++r)
#pragma unroll
          for (int q = 0; q < 4; ++q) aj[q][r] = fmaf(v[q + i], wv[i * kFilters + r], aj[q][r]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int r = 0; r < kFilters; ++r) acc[q][r] += aj[q][r];
  }

  // epilogue: threshold with the rigorous cut, warp-aggregated compaction
  unsigned flags = 0;
  int cnt = 0;
  const bool row_ok = y < D.sh;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool ok = row_ok && (x + q) < D.sw;
#pragma unroll
    for (int r = 0; r < kFilters; ++r) {
      if (ok && acc[q][r] > __ldg(cut + r)) {
        flags |= 1u << (q * kFilters + r);
        ++cnt;
      }
    }
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int warp_total = __shfl_sync(0xffffffffu, incl, 31);
  if (warp_total == 0) return;
  unsigned long long base = 0;
  if (lane == 31) base = atomicAdd(n_cand, (unsigned long long)warp_total);
  base = __shfl_sync(0xffffffffu, base, 31);
  long long pos = (long long)base + incl - cnt;
  while (flags) {
    const int bit = __ffs(flags) - 1;
    flags &= flags - 1;
    if (pos < cap) {
      Candidate c;
      c.frame = f;
      c.slot_r = s * 8 + bit % kFilters;
      c.cx = x + bit / kFilters;
      c.cy = y;
      cand[pos] = c;
    }
    ++pos;
  }
}

void launch_screen(const Launch& L, const PlanDesc& Ph, const PlanDesc* Pd, const float* feat32,
                   const float* w32, const float* cut, Candidate* cand, unsigned long long* n_cand,
                   long long cand_cap) {
  if (Ph.sc_total <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_screen, cudaFuncAttributeMaxDynamicSharedMemorySize, kScreenSmem);
    attr = true;
  }
  LevelBegins B{};
  B.n = Ph.n_scored;
  for (int s = 0; s < Ph.n_scored; ++s) B.b[s] = Ph.lv[s].sc_begin;
  B.b[B.n] = Ph.sc_total;
  k_screen<<<(unsigned)div_up(Ph.sc_total, kScreenWarps), kScreenWarps * 32, kScreenSmem, L.st>>>(Pd, B, feat32, w32, cut, cand,
                                                                        n_cand, cand_cap, Ph.sc_total);
  ++*L.counter;
}

}  // namespace blb
