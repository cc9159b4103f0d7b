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
  const int lx = D.sc_lanes_x;
  const int x = (t % D.sc_tiles_x) * (4 * lx) + (lane % lx) * 4;
  const int y = (t / D.sc_tiles_x) * (32 / lx) + lane / lx;
  const int cw_pad = D.cw_pad;
  const long long plane = (long long)D.ch_pad * cw_pad;
  const float* fb = feat32 + D.f32_off + (long long)f * D.f32_fstride + x;

  float acc[4][kFilters];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int r = 0; r < kFilters; ++r) acc[q][r] = 0.f;

  // software pipeline: feature vectors of step (j, f+1) are in flight while step (j, f) feeds
  // 200 FMAs; the f loop is unrolled by two so the two prefetch buffers alternate by name.
  auto load4 = [&](int j, int ff, float4& a0, float4& a1, float4& a2, float4& a3) {
    const float4* p = reinterpret_cast<const float4*>(fb + (long long)(y + j) * cw_pad + ff * plane);
    a0 = __ldg(p);
    a1 = __ldg(p + 1);
    a2 = __ldg(p + 2);
    a3 = __ldg(p + 3);
  };
  auto step = [&](float (&aj)[4][kFilters], const float4& a0, const float4& a1, const float4& a2, const float4& a3,
                  const float4* wp) {
    const float v[16] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w,
                         a2.x, a2.y, a2.z, a2.w, a3.x, a3.y, a3.z, a3.w};
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
  };
  float4 p0, p1, p2, p3, q0, q1, q2, q3;
  load4(0, 0, p0, p1, p2, p3);
#pragma unroll 1
  for (int j = 0; j < kWin; ++j) {
    float aj[4][kFilters];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int r = 0; r < kFilters; ++r) aj[q][r] = 0.f;
    const float4* wj = sW4 + j * kFeat * (kWBlock / 4);
    // kFeat = 31 = 15 pairs + 1
#pragma unroll 1
    for (int ff = 0; ff < kFeat - 1; ff += 2) {
      load4(j, ff + 1, q0, q1, q2, q3);
      step(aj, p0, p1, p2, p3, wj + ff * (kWBlock / 4));
      const int nf = ff + 2;  // < kFeat
      load4(j, nf, p0, p1, p2, p3);
      step(aj, q0, q1, q2, q3, wj + (ff + 1) * (kWBlock / 4));
    }
    {  // f = 30, prefetch (j+1, 0); the last prefetch re-reads row y+9, harmlessly
      load4(min(j + 1, kWin - 1), 0, q0, q1, q2, q3);
      step(aj, p0, p1, p2, p3, wj + (kFeat - 1) * (kWBlock / 4));
      p0 = q0;
      p1 = q1;
      p2 = q2;
      p3 = q3;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int r = 0; r < kFilters; ++r) acc[q][r] += aj[q][r];
  }

  // epilogue: threshold with the rigorous cut, warp-aggregated append per filter list
  const bool row_ok = y < D.sh;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool ok = row_ok && (x + q) < D.sw;
    unsigned flags = 0;
#pragma unroll
    for (int r = 0; r < kFilters; ++r)
      if (ok && acc[q][r] > __ldg(cut + r)) flags |= 1u << r;
    emit_candidates(flags, f, s, x + q, y, cand, n_cand, cap);
  }
}

void launch_screen(const Launch& L, const PlanDesc& Ph, const PlanDesc* Pd, const float* feat32,
                   const float* w32, const float* cut, Candidate* cand, unsigned long long* n_cand,
                   long long cand_cap) {
  if (Ph.sc_total <= 0) return;
  LevelBegins B{};
  B.n = Ph.n_scored;
  for (int s = 0; s < Ph.n_scored; ++s) B.b[s] = Ph.lv[s].sc_begin;
  B.b[B.n] = Ph.sc_total;
  k_screen<<<(unsigned)div_up(Ph.sc_total, kScreenWarps), kScreenWarps * 32, kScreenSmem, L.st>>>(Pd, B, feat32, w32, cut, cand,
                                                                        n_cand, cand_cap, Ph.sc_total);
  ++*L.counter;
}

void configure_classify_kernels(int optin) {  // per device, see configure_screen_tc_kernels
  smem_optin(k_screen, optin);
}

}  // namespace blb
