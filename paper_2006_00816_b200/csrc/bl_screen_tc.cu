// Sliding-window linear classifier, stage 1 on the 5th-generation tensor cores (tcgen05).
//
// The screen score(anchor, r) = sum_{j, dx, f} F[cy + j][cx + dx][f] * W_r[j][dx][f] is an
// implicit GEMM.  Linearise each (level, frame) feature image row-major with pitch cw:
// anchor (cx, cy) -> L = cy * cw + cx, window cell (dx, j) -> L + j * cw + dx.  Per window
// row j one MMA chain computes, for 128 consecutive cells L' of row offset j,
//
//     Q_j[L'][dx, r] = sum_f F[L' + j*cw][f] * W[j][dx][f][r]        (N = 10 dx x 5 r -> 64)
//
// accumulated over j in TMEM, and the epilogue finishes the correlation along x:
// score[L][r] = sum_dx Q[L + dx][dx, r] (cells L .. L+9 of the same 128-cell tile, so a tile
// yields 119 anchors).  Putting dx into N instead of shifting A keeps every MMA at
// M = 128, N = 64, K = 16 with a 4 KB A tile (an N = 16 per-dx formulation re-reads A from
// shared memory ten times and is smem-bandwidth-bound).  Anchors whose cx lands in the last
// 9 columns wrap into the next image row; they are discarded by the epilogue's
// (cx < sw, cy < sh) test.
//
// Per CTA (persistent, one per SM): the fp16 weights of all 10 window rows (40 KB) stay in
// shared memory; warp 0 streams, per unit, the 4 feature planes (8 fp16 features each) of the
// cell band all 10 window rows read (rows overlap by all but cw cells, so the band is
// copied once; levels wider than 80 cells take several row groups) into a 2-stage ring with
// cp.async.bulk; one thread of warp 1 issues 2 k-steps of tcgen05.mma.kind::f16 per row and
// m-tile into TMEM; warps 2-5 read the accumulators back with tcgen05.ld (one cell per TMEM lane), do the dx-correlation through
// shared memory, apply the rigorous cut and append candidates.  Two TMEM accumulator sets
// let the epilogue of unit u overlap the MMAs of unit u + 1.
//
// Precision: features (scaled by 2^8) and weights (scaled per filter by a power of two to
// [2^14, 2^15)) are rounded to fp16 (round-to-nearest-even) and the MMA accumulates in fp32;
// the power-of-two scales are exact and folded into the cut, so |screen - exact| <= delta_tc
// (bl_capi.cu: rigorous bound with 2^-10 relative operand rounding, the fp16 subnormal floor
// and accumulation); every candidate is re-scored exactly in fp64 by bl_exact.cu, so output
// bits never depend on this kernel's rounding.  (fp16 vs tf32: the same 11-bit significand,
// half the feature bytes and twice the MMA K per instruction.)
#include "bl_internal.cuh"

namespace blb {

namespace {

constexpr int kTcM = 128;             // cells per m-tile (TMEM lanes)
constexpr int kTcV = kTcM - (kWin - 1);   // anchors per m-tile (119)
constexpr int kTcN = 64;              // 10 dx x 5 filters = 50 columns, padded
constexpr int kTcNM = 2;              // m-tiles per work unit
constexpr int kTcNA = 248;            // cells staged per plane: kTcV * (kTcNM - 1) + kTcM, rounded to 8
constexpr int kTcPlanes = kTcPlanesF16;  // 32 features / 8 fp16 per 16-B chunk
constexpr int kTcKSteps = kTcPlanes / 2;  // MMAs (K = 16 = two chunks) per window row
#ifndef BL_TC_J
#define BL_TC_J 10
#endif
constexpr int kTcJ = BL_TC_J;        // window rows per stage: their cell ranges overlap by cw
constexpr int kTcCwMax = 80;          // a stage holds kTcJ rows of levels up to this wide
constexpr int kTcNAS = kTcNA + (kTcJ - 1) * kTcCwMax;      // cells per plane per stage
#ifndef BL_TC_STAGES
#define BL_TC_STAGES 2
#endif
constexpr int kTcStages = BL_TC_STAGES;
constexpr int kTcABytes = kTcPlanes * kTcNAS * 16;          // 61,952 per stage (J = 10)
constexpr int kTcWRowBytes = kTcPlanes * kTcN * 16;         // 4,096 per window row j
constexpr int kTcWBytes = kWin * kTcWRowBytes;              // 40,960 resident
constexpr int kTcEpiBytes = 50 * kTcM * 4;                  // 25,600: Q tile for the dx-correlation
constexpr int kTcAccCols = kTcNM * kTcN;                    // 128 columns per accumulator set
constexpr int kTcTmemCols = 256;                            // two sets
constexpr int kTcThreads = 6 * 32;
constexpr size_t kTcSmem = (size_t)kTcWBytes + kTcStages * kTcABytes + kTcEpiBytes + 1024;
static_assert(kTcNA >= kTcV * (kTcNM - 1) + kTcM && kTcNA % 8 == 0, "stage width");
static_assert(kTcSmem <= 227 * 1024, "shared memory");

// window rows staged together for a level cw cells wide: as many as the stage holds
__device__ __forceinline__ int rows_per_stage(int cw) {
  return min(kTcJ, 1 + (kTcNAS - kTcNA) / max(cw, 1));
}

// K-major, no-swizzle canonical smem descriptor: core matrix = 8 rows x 16 B contiguous;
// lbo = byte distance between the two 16-B K chunks, sbo = between 8-row groups.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// kind::f16 instruction descriptor: D f32 (bits 4-5 = 1), A/B f16 (format 0), both K-major,
// N = 64, M = 128.
constexpr uint32_t kTcIdesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(kTcN >> 3) << 17) |
                              ((uint32_t)(kTcM >> 4) << 24);

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kTcIdesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

}  // namespace

// Work unit u -> (scored slot s, frame f, first anchor L0).  TcUnits is passed by value.
struct TcUnits {
  int n;                       // scored levels
  long long b[kMaxLevels + 1]; // first unit of each level; b[n] = total units
  int tiles[kMaxLevels];       // units per (level, frame)
};

__global__ void __launch_bounds__(kTcThreads, 1) k_screen_tc(const PlanDesc* __restrict__ P, const TcUnits U,
                                                            const float* __restrict__ feat_tc,
                                                            const float* __restrict__ w_tc,
                                                            const float* __restrict__ cut,
                                                            Candidate* __restrict__ cand,
                                                            unsigned long long* __restrict__ n_cand, long long cap,
                                                            float* __restrict__ dbg_scores) {
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  __shared__ uint64_t full_bar[kTcStages], empty_bar[kTcStages], tfull_bar[2], tempty_bar[2], w_bar;
  __shared__ uint32_t tmem_base_sh;
  uint8_t* sW = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_smem) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sW + kTcWBytes;
  float* sQ = reinterpret_cast<float*>(sA + kTcStages * kTcABytes);  // [50][128]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long total = U.b[U.n];

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);  // one arrive per epilogue warp
    }
    mbar_init(&w_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "n"(kTcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  auto unit_info = [&](long long u, int& s, int& f, long long& L0) {
    s = 0;
    while (s + 1 < U.n && u >= U.b[s + 1]) ++s;
    const long long local = u - U.b[s];
    f = (int)(local / U.tiles[s]);
    L0 = (local - (long long)f * U.tiles[s]) * (kTcV * kTcNM);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer (bulk copies)
    if (lane == 0) {
      mbar_expect_tx(&w_bar, kTcWBytes);  // all 10 weight rows, once per CTA
      for (int j = 0; j < kWin; ++j) bulk_g2s(sW + j * kTcWRowBytes, w_tc + j * (kTcWRowBytes / 4), kTcWRowBytes, &w_bar);
      int stage = 0;
      uint32_t phase = 0;
      for (long long u = blockIdx.x; u < total; u += gridDim.x) {
        int s, f;
        long long L0;
        unit_info(u, s, f, L0);
        const LevelDesc& D = P->lv[s];
        const long long ncp = D.tc_ncp;
        const float* fbase = feat_tc + D.tc_off + (long long)f * kTcPlanes * ncp * 4;
        const int jpl = rows_per_stage(D.cw);
        for (int j0 = 0; j0 < kWin; j0 += jpl) {
          // window rows j0 .. j0+J-1 read cells [L0 + j0*cw, L0 + (j0+J-1)*cw + NA): one copy
          const int J = min(jpl, kWin - j0);
          const int nc = kTcNA + (J - 1) * D.cw;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = sA + stage * kTcABytes;
          mbar_expect_tx(&full_bar[stage], (uint32_t)(kTcPlanes * nc * 16));
          const long long c0 = L0 + (long long)j0 * D.cw;
#pragma unroll 1
          for (int kc = 0; kc < kTcPlanes; ++kc)
            bulk_g2s(sa + kc * kTcNAS * 16, fbase + ((long long)kc * ncp + c0) * 4, (uint32_t)nc * 16,
                     &full_bar[stage]);
          if (++stage == kTcStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    mbar_wait(&w_bar, 0);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t sw0 = smem_u32(sW);
    for (long long u = blockIdx.x; u < total; u += gridDim.x) {
      int us, uf;
      long long uL0;
      unit_info(u, us, uf, uL0);
      const int cw = P->lv[us].cw;
      const int jpl = rows_per_stage(cw);
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem_base + acc * kTcAccCols;
      for (int j0 = 0; j0 < kWin; j0 += jpl) {
        const int J = min(jpl, kWin - j0);
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(sA + stage * kTcABytes);
#pragma unroll 1
          for (int jj = 0; jj < J; ++jj) {
            const int j = j0 + jj;
#pragma unroll
            for (int kk = 0; kk < kTcKSteps; ++kk) {
              // B (weights of row j): [kc][64 n][16 B]: K chunk step 1024 B, 8-row group step 128 B
              const uint64_t db = umma_desc(sw0 + j * kTcWRowBytes + (2 * kk) * (kTcN * 16), kTcN * 16, 128);
#pragma unroll
              for (int m = 0; m < kTcNM; ++m) {
                // A (cells of row j): [kc][NAS cells][16 B], row j starts jj*cw cells into the stage
                const uint64_t da = umma_desc(sa + (uint32_t)(((2 * kk) * kTcNAS + jj * cw + m * kTcV) * 16),
                                              kTcNAS * 16, 128);
                mma_f16(d0 + m * kTcN, da, db, (j | kk) != 0);
              }
            }
          }
          mma_commit(&empty_bar[stage]);  // frees the smem stage once these MMAs have read it
          if (j0 + J == kWin) mma_commit(&tfull_bar[acc]);
        }
        __syncwarp();
        if (++stage == kTcStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;     // TMEM lane quarter this warp may access
    const int t = 32 * q + lane;  // cell (TMEM lane) within the m-tile
    int acc = 0;
    uint32_t acc_phase = 0;
    float cutv[kFilters], unscale[kFilters];  // cut in the scaled domain; 2^-(scale exponents)
#pragma unroll
    for (int r = 0; r < kFilters; ++r) {
      cutv[r] = __ldg(cut + r);
      unscale[r] = __ldg(cut + kFilters + r);
    }
    for (long long u = blockIdx.x; u < total; u += gridDim.x) {
      int s, f;
      long long L0;
      unit_info(u, s, f, L0);
      const LevelDesc& D = P->lv[s];
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int m = 0; m < kTcNM; ++m) {
        {  // Q[t][0..49] of this m-tile -> smem [col][cell]
          uint32_t r0[32], r1[32];
          const uint32_t ta = tmem_base + ((uint32_t)(32 * q) << 16) + acc * kTcAccCols + m * kTcN;
          tmem_ld32(ta, r0);
          tmem_ld32(ta + 32, r1);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 32; ++c) sQ[c * kTcM + t] = __uint_as_float(r0[c]);
#pragma unroll
          for (int c = 0; c < 50 - 32; ++c) sQ[(32 + c) * kTcM + t] = __uint_as_float(r1[c]);
        }
        epi_bar();
        // score[t][r] = sum_dx Q[t + dx][dx * 5 + r]
        float v[kFilters];
#pragma unroll
        for (int r = 0; r < kFilters; ++r) v[r] = 0.f;
        if (t < kTcV) {
#pragma unroll
          for (int dx = 0; dx < kWin; ++dx)
#pragma unroll
            for (int r = 0; r < kFilters; ++r) v[r] += sQ[(dx * kFilters + r) * kTcM + t + dx];
        }
        epi_bar();  // sQ is rewritten by the next m-tile
        const long long L = L0 + (long long)m * kTcV + t;
        const int cy = (int)(L / D.cw), cx = (int)(L - (long long)cy * D.cw);
        const bool ok = t < kTcV && cx < D.sw && cy < D.sh;
        if (dbg_scores && ok) {
#pragma unroll
          for (int r = 0; r < kFilters; ++r) dbg_scores[((long long)r * D.sh + cy) * D.sw + cx] = v[r] * unscale[r];
        }
        unsigned flags = 0;
#pragma unroll
        for (int r = 0; r < kFilters; ++r)
          if (ok && v[r] > cutv[r]) flags |= 1u << r;
        emit_candidates(flags, f, s, cx, cy, cand, n_cand, cap);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTcTmemCols));
}

size_t tc_feat_floats_per_frame(int cw, int ch, long long* ncp_out, int* tiles_out) {
  const int sw = cw - (kWin - 1), sh = ch - (kWin - 1);
  const long long lmax = (long long)(sh - 1) * cw + sw;  // anchors live in [0, lmax)
  const int tiles = (int)div_up(lmax, kTcV * kTcNM);
  const long long ncp = div_up((long long)tiles * kTcV * kTcNM + (long long)(kWin - 1) * cw + kTcNA, 8) * 8;
  if (ncp_out) *ncp_out = ncp;
  if (tiles_out) *tiles_out = tiles;
  return (size_t)kTcPlanes * ncp * 4;
}

size_t tc_weight_floats() { return (size_t)kTcWBytes / 4; }

void launch_screen_tc(const Launch& L, const PlanDesc& Ph, const PlanDesc* Pd, const float* feat_tc,
                      const float* w_tc, const float* cut, Candidate* cand, unsigned long long* n_cand,
                      long long cand_cap, float* dbg_scores) {
  TcUnits U{};
  U.n = Ph.n_scored;
  long long units = 0;
  for (int s = 0; s < Ph.n_scored; ++s) {
    int tiles = 0;
    tc_feat_floats_per_frame(Ph.lv[s].cw, Ph.lv[s].ch, nullptr, &tiles);
    U.tiles[s] = tiles;
    U.b[s] = units;
    units += (long long)tiles * Ph.n_frames;
  }
  U.b[U.n] = units;
  if (units <= 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)(units < sms ? units : sms);
  k_screen_tc<<<grid, kTcThreads, kTcSmem, L.st>>>(Pd, U, feat_tc, w_tc, cut, cand, n_cand, cand_cap, dbg_scores);
  ++*L.counter;
}

// Dynamic shared-memory opt-in of this file's kernels, for the CURRENT device (the attribute is
// per device: bl_ctx_create calls this after cudaSetDevice, so contexts on several GPUs work).
void configure_screen_tc_kernels(int optin) {
  smem_optin(k_screen_tc, optin);
}

}  // namespace blb
