// Ensemble-of-regression-trees 68-landmark cascade (ert.cpp:15-136) on the device.
//
// The cascade levels are strictly sequential (ert.cpp:108); within a level every face and
// every tree is independent.  Per level three fully parallel kernels:
//   1. k_ert_xform    thread per face: similarity transform current -> mean (ert.cpp:26-69),
//                     fp64 sums in a fixed order, the linear part (a, b) taken directly
//                     (the reference's hypot/atan2/cos/sin round trip returns it up to a few
//                     ulp: face_transform_warp);
//   2. k_ert_traverse thread per (face, tree): walks the F splits in level order, left iff
//                     Ia - Ib > thr (ert.cpp:87-97), sampling the ORIGINAL frame through
//                     apply_linear + box map + llround + clamp (ert.cpp:20-24, 71-85);
//   3. k_ert_accum    thread per (face, coordinate): sums the K selected leaf rows IN TREE
//                     ORDER in fp64 (ert.cpp:118-121), cur += shrinkage * delta (:123-126).
// Compiled with --fmad=false; all arithmetic mirrors the reference operation for operation.
//
// Level-synchronous launches keep one level's trees (K * 2^F * L * 16 B = 8.7 MB at 500
// trees, depth 4, L = 68) resident in L2 for every face of the batch: HBM reads the model
// once per batch; L2 serves the 1088-B leaf row each (face, tree) selects.
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <cstdlib>

#include "bl_internal.cuh"

namespace blb {

__global__ void k_ert_init(ErtDev M, const int* __restrict__ n_faces, int cap, double* __restrict__ cur) {
  const int n = min(*n_faces, cap);
  const int L2 = 2 * M.L;
  const long long total = (long long)n * L2;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    cur[i] = M.mean_xy[i % L2];
}

void launch_ert_init(const Launch& L, const ErtDev& M, const int* n_faces, int cap, double* cur) {
  k_ert_init<<<148 * 4, 256, 0, L.st>>>(M, n_faces, cap, cur);
  ++*L.counter;
}

#ifndef BL_ERT_EVICT_LAST
#define BL_ERT_EVICT_LAST 0  // leaf rows loaded with an L2 evict_last policy (experiment)
#endif
BL_DEV double2 ld_leaf(const double2* p, uint64_t pol) {
  if (!BL_ERT_EVICT_LAST) return __ldg(p);
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}

template <bool U8>
BL_DEV double sample_px(const void* fr, int w, int h, long long pitch, int bx, int by, int bw, int bh,
                        const double* cur, double A, double B, int anchor, double ox, double oy) {
  const double offx = dsub(dmul(A, ox), dmul(B, oy));  // apply_linear, ert.cpp:22
  const double offy = dadd(dmul(B, ox), dmul(A, oy));
  const double nx = dadd(cur[2 * anchor], offx);       // ert.cpp:75-76
  const double ny = dadd(cur[2 * anchor + 1], offy);
  const double px = dadd((double)bx, dmul(nx, (double)bw));  // ert.cpp:77-78
  const double py = dadd((double)by, dmul(ny, (double)bh));
  int ix = (int)llround(px);
  int iy = (int)llround(py);
  ix = ix < 0 ? 0 : (w - 1 < ix ? w - 1 : ix);
  iy = iy < 0 ? 0 : (h - 1 < iy ? h - 1 : iy);
  if (U8) return (double)__ldg((const uint8_t*)fr + (long long)iy * pitch + ix);
  return __ldg((const double*)fr + (long long)iy * pitch + ix);
}

__device__ int face_transform_warp(const ErtDev& M, const double* c, const double* mc, int lane, double& A,
                                   double& B);

// (1) similarity_transform(current, mean) per face, ert.cpp:26-69.  A warp per face stages
// the current shape in shared memory and runs face_transform_warp.  Stores the linear part
// (scale*cos, scale*sin) that apply_linear recomputes for every sample (ert.cpp:21-22).
constexpr int kXfFaces = 4;
constexpr int kMaxL2 = 512;  // 2L <= 512 (L <= 256) for the staged kernels

__global__ void __launch_bounds__(32 * kXfFaces) k_ert_xform(ErtDev M, const int* __restrict__ n_faces, int cap,
                                                             const double* __restrict__ cur_g,
                                                             double2* __restrict__ tf, int* __restrict__ err) {
  __shared__ double sc[kXfFaces][kMaxL2];
  const int n = min(*n_faces, cap);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int face = blockIdx.x * kXfFaces + warp;
  if (face >= n) return;
  const int L = M.L, L2 = 2 * L;
  const double* cur = cur_g + (long long)face * L2;
  for (int i = lane; i < L2; i += 32) sc[warp][i] = cur[i];
  __syncwarp();
  double A = 0.0, B = 0.0;
  const int e = face_transform_warp(M, sc[warp], M.mean_c, lane, A, B);
  if (lane != 0) return;
  if (e) atomicExch(err, e);
  tf[face] = make_double2(A, B);
}

// Canonical device summation order of the cascade (every kernel uses it, so the kernels are
// bit-identical to each other; against the reference's sequential sums the landmarks move by
// ~1e-16 relative, far inside the 1e-3 px contract, and no leaf decision flips -- SURVEY.md
// §0.6 measured 0 mismatches in 7.5 M decisions for arbitrary fp64 summation orders, and the
// C4 test checks all 10k boxes against the reference):
//  * shape sums of the similarity transform: lane l of a warp adds points l, l + 32, ... in
//    order, then an xor butterfly over the 32 lanes (every lane ends with the same bits);
//  * leaf sums: partial sums over chunks of kLeafChunk consecutive trees (each in tree order,
//    from 0.0), then the partials in chunk order.
#ifndef BL_LEAF_CHUNK
#define BL_LEAF_CHUNK 64
#endif
constexpr int kLeafChunk = BL_LEAF_CHUNK;
static_assert(kLeafChunk % 16 == 0, "16 leaf indices per 16-B load");

BL_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = dadd(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// similarity_transform(current -> mean) of one face (ert.cpp:26-69), computed by a whole warp
// (c, mc: the current shape and the centred mean shape, shared or global).  Returns 0 or the
// reference's error (1: source shape has no spread, 2: target shape has no spread) and the
// linear part (scale*cos, scale*sin) in A, B; identical in every lane.
__device__ int face_transform_warp(const ErtDev& M, const double* c, const double* mc, int lane, double& A,
                                   double& B) {
  const int L = M.L;
  double sx = 0.0, sy = 0.0;
  for (int i = lane; i < L; i += 32) {  // ert.cpp:33-43 centroid
    sx = dadd(sx, c[2 * i]);
    sy = dadd(sy, c[2 * i + 1]);
  }
  const double mfx = ddiv(warp_sum(sx), (double)L), mfy = ddiv(warp_sum(sy), (double)L);
  double sff = 0.0, sre = 0.0, sim = 0.0;
  for (int i = lane; i < L; i += 32) {  // ert.cpp:44-55
    const double fx = dsub(c[2 * i], mfx);
    const double fy = dsub(c[2 * i + 1], mfy);
    const double txp = mc[2 * i], typ = mc[2 * i + 1];  // to.x - mt.x, host-computed with the same op
    sff = dadd(sff, dadd(dmul(fx, fx), dmul(fy, fy)));
    sre = dadd(sre, dadd(dmul(fx, txp), dmul(fy, typ)));
    sim = dadd(sim, dsub(dmul(fx, typ), dmul(fy, txp)));
  }
  sff = warp_sum(sff);
  sre = warp_sum(sre);
  sim = warp_sum(sim);
  A = 0.0;
  B = 0.0;
  if (!(sff > 0.0)) return 1;  // "source shape has no spread" (ert.cpp:56-57)
  // ert.cpp:58-67 stores scale = hypot(a, b) and rotation = atan2(b, a), and apply_linear
  // (ert.cpp:21-22) multiplies back scale * cos(rotation), scale * sin(rotation): in real
  // arithmetic exactly a and b.  The round trip through libm only adds a few ulp of noise (and
  // costs a dependent hypot / atan2 / sin / cos chain per face and level), so the linear part
  // is taken directly; the reference's "no spread" test scale <= 0 is a == b == 0.
  A = ddiv(sre, sff);
  B = ddiv(sim, sff);
  if (A == 0.0 && B == 0.0) return 2;  // "target shape has no spread" (ert.cpp:62-63)
  return 0;
}

// (2) one CTA per face, one thread per tree: traverse_tree (ert.cpp:87-97) with
// sample_intensity (ert.cpp:71-85) on the ORIGINAL frame; the face's current shape is staged
// in shared memory; split records are node-major so a warp's loads are contiguous.
template <bool U8>
__global__ void __launch_bounds__(256) k_ert_traverse(ErtDev M, int t, const void* __restrict__ frames, int w,
                                                      int h, long long pitch, long long fstride,
                                                      const int* __restrict__ face_frame,
                                                      const int* __restrict__ boxes, int box_stride,
                                                      const int* __restrict__ n_faces, int cap,
                                                      const double* __restrict__ cur_g,
                                                      const double2* __restrict__ tf,
                                                      uint8_t* __restrict__ leaf_idx, long long leaf_stride) {
  __shared__ double sc[kMaxL2];
  const int n = min(*n_faces, cap);
  const int face = blockIdx.x;
  if (face >= n) return;
  const int K = M.K, S = M.S, L2 = 2 * M.L;
  const double* cur = cur_g + (long long)face * L2;
  for (int i = threadIdx.x; i < L2; i += blockDim.x) sc[i] = cur[i];
  __syncthreads();
  const double2 ab = tf[face];
  const int* bx = boxes + (long long)face * box_stride;
  const int X = bx[0], Y = bx[1], W = bx[2], H = bx[3];
  const void* fr = (const char*)frames + (long long)face_frame[face] * fstride * (U8 ? 1 : 8);
  const int4* lvl = reinterpret_cast<const int4*>(M.split) + (long long)t * S * K;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    int node = 0;
    while (node < S) {
      const int4* r = lvl + (long long)node * K + k;
      const double2 oa = __ldg(reinterpret_cast<const double2*>(r));                  // offset_a
      const double2 ob = __ldg(reinterpret_cast<const double2*>(r + M.split_plane));  // offset_b
      const int4 tail = __ldg(r + 2 * M.split_plane);                                 // thr, anchors
      const double thr = __hiloint2double(tail.y, tail.x);
      const int an_a = (short)(tail.z & 0xffff), an_b = (short)(tail.z >> 16);
      const double ia = sample_px<U8>(fr, w, h, pitch, X, Y, W, H, sc, ab.x, ab.y, an_a, oa.x, oa.y);
      const double ib = sample_px<U8>(fr, w, h, pitch, X, Y, W, H, sc, ab.x, ab.y, an_b, ob.x, ob.y);
      node = dsub(ia, ib) > thr ? 2 * node + 1 : 2 * node + 2;
    }
    leaf_idx[(long long)face * leaf_stride + k] = (uint8_t)(node - S);
  }
}

// (3) one thread per (face, landmark): sums the K selected leaf rows IN TREE ORDER in fp64
// (ert.cpp:118-121) for the landmark's (x, y) pair, then cur += shrinkage * delta
// (ert.cpp:123-126).  Consecutive threads read consecutive 16-B pairs of one leaf row
// (coalesced, L2-resident for the level); 16 leaf indices arrive per 128-bit load and the
// 16 trees' loads are issued ahead of their adds.
__global__ void __launch_bounds__(256) k_ert_accum(ErtDev M, int t, const int* __restrict__ n_faces, int cap,
                                                   double* __restrict__ cur_g,
                                                   const uint8_t* __restrict__ leaf_idx, long long leaf_stride) {
  const int n = min(*n_faces, cap);
  const int L = M.L, K = M.K, NL = M.NL;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (long long)n * L) return;
  const int face = (int)(g / L), p = (int)(g - (long long)face * L);
  const uint8_t* li = leaf_idx + (long long)face * leaf_stride;
  const double2* lv = reinterpret_cast<const double2*>(M.leaves + (long long)t * K * NL * 2 * L) + p;
  const int row = NL * L;  // double2 per tree
  double ax = 0.0, ay = 0.0;  // the canonical chunked order (face_transform_warp's note)
  const bool vec = ((reinterpret_cast<uintptr_t>(li) & 15) == 0);
  for (int c0 = 0; c0 < K; c0 += kLeafChunk) {
    const int c1 = min(K, c0 + kLeafChunk);
    double px = 0.0, py = 0.0;
    int k = c0;
    for (; vec && k + 16 <= c1; k += 16) {
      const uint4 q = *reinterpret_cast<const uint4*>(li + k);
      const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
      double2 v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int idx = (wv[u >> 2] >> ((u & 3) * 8)) & 0xff;
        v[u] = __ldg(lv + (k + u) * row + idx * L);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        px = dadd(px, v[u].x);
        py = dadd(py, v[u].y);
      }
    }
    for (; k < c1; ++k) {
      const double2 v = __ldg(lv + k * row + li[k] * L);
      px = dadd(px, v.x);
      py = dadd(py, v.y);
    }
    ax = dadd(ax, px);
    ay = dadd(ay, py);
  }
  double2* cur = reinterpret_cast<double2*>(cur_g + (long long)face * 2 * L) + p;
  double2 cv = *cur;
  cv.x = dadd(cv.x, dmul(M.shrinkage, ax));
  cv.y = dadd(cv.y, dmul(M.shrinkage, ay));
  *cur = cv;
}

void launch_ert_level(const Launch& L, const ErtDev& M, int t, const void* frames, int u8, int w, int h,
                      long long pitch, long long fstride, const int* face_frame, const int* boxes, int box_stride,
                      const int* n_faces, int cap, double* cur, double2* tf, uint8_t* leaf_idx,
                      long long leaf_stride, int* err) {
  k_ert_xform<<<(unsigned)div_up(cap, kXfFaces), 32 * kXfFaces, 0, L.st>>>(M, n_faces, cap, cur, tf, err);
  const int tb = M.K >= 256 ? 256 : (int)div_up(M.K, 32) * 32;
  if (u8)
    k_ert_traverse<true><<<(unsigned)cap, tb, 0, L.st>>>(M, t, frames, w, h, pitch, fstride, face_frame, boxes,
                                                        box_stride, n_faces, cap, cur, tf, leaf_idx, leaf_stride);
  else
    k_ert_traverse<false><<<(unsigned)cap, tb, 0, L.st>>>(M, t, frames, w, h, pitch, fstride, face_frame, boxes,
                                                         box_stride, n_faces, cap, cur, tf, leaf_idx, leaf_stride);
  k_ert_accum<<<(unsigned)div_up((long long)cap * M.L, 256), 256, 0, L.st>>>(M, t, n_faces, cap, cur, leaf_idx,
                                                                           leaf_stride);
  *L.counter += 3;
}

// The whole cascade for a group of faces in ONE launch (ert.cpp:99-136).  Faces are
// independent, so a CTA owns kFcFaces faces and runs every level itself, with block barriers
// between the level's three phases -- the same arithmetic as k_ert_xform / k_ert_traverse /
// k_ert_accum (bit-identical), without 3 x T launches and the inter-kernel gaps:
//   xform    warp per face: similarity transform of the staged current shape;
//   traverse thread per (face, tree): level-order descent, leaf index -> smem;
//   accum    thread per (face, landmark pair): the K selected leaf rows in tree order.
// Current shapes, transforms and the level's leaf indices live in shared memory.
struct TravItem {  // one (face, tree) traversal in flight
  const void* fr;
  double2 ab;
  int X, Y, W, H, k, fi, node;
};

#ifndef BL_ERT_FACES
#define BL_ERT_FACES 4
#endif
constexpr int kFcFaces = BL_ERT_FACES;
constexpr int kFcThreads = ((kFcFaces * 68 + 31) / 32) * 32;  // one thread per (face, pair) at L = 68
#ifndef BL_FC_LEAN
#define BL_FC_LEAN 1  // k_ert_cascade leaf sums: 16 leaf indices per 16-B shared load (not 16 LDS.U8)
#endif
BL_HD_INLINE int fc_sli_stride(int K) { return (K + 15) & ~15; }  // per-face leaf indices, 16-B rows

template <bool U8>
__global__ void __launch_bounds__(kFcThreads) k_ert_cascade(ErtDev M, const void* __restrict__ frames, int w, int h,
                                                     long long pitch, long long fstride,
                                                     const int* __restrict__ face_frame,
                                                     const int* __restrict__ boxes, int box_stride,
                                                     const int* __restrict__ n_faces, int cap,
                                                     double* __restrict__ out_xy, uint8_t* __restrict__ leaf_out,
                                                     long long leaf_out_stride, int* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char fc_smem[];
  const int L = M.L, L2 = 2 * L, K = M.K, S = M.S, NL = M.NL;
  double* sc = reinterpret_cast<double*>(fc_smem);                    // [kFcFaces][2L]
  double2* stf = reinterpret_cast<double2*>(sc + kFcFaces * L2);      // [kFcFaces]
  uint8_t* sli = reinterpret_cast<uint8_t*>(stf + kFcFaces);          // [kFcFaces][Kp]
  const int Kp = fc_sli_stride(K);
  const int n = min(*n_faces, cap);
  const int f0 = blockIdx.x * kFcFaces;
  if (f0 >= n) return;
  const int nf = min(kFcFaces, n - f0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < nf * L2; e += blockDim.x) sc[e] = M.mean_xy[e % L2];  // ert.cpp:106
  __syncthreads();
  for (int t = 0; t < M.T; ++t) {
    // (1) transforms, a warp per face
    if (warp < nf) {
      double A, B;
      const int e = face_transform_warp(M, sc + warp * L2, M.mean_c, lane, A, B);
      if (lane == 0) {
        if (e) atomicExch(err, e);
        stf[warp] = make_double2(A, B);
      }
    }
    __syncthreads();
    // (2) traversals: two (face, tree) items per thread walk their trees in lock-step (all
    // trees have depth F), so each level's record and pixel loads of both are in flight together
    const int4* lvl = reinterpret_cast<const int4*>(M.split) + (long long)t * S * K;
    const int items = nf * K;
    for (int e0 = tid; e0 < items; e0 += 2 * blockDim.x) {
      const int e1 = min(e0 + (int)blockDim.x, items - 1);  // a duplicate of e0's last item when odd
      TravItem it[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int e = q == 0 ? e0 : e1;
        const int fi = e / K;
        it[q].k = e - fi * K;
        it[q].fi = fi;
        const int face = f0 + fi;
        it[q].ab = stf[fi];
        const int* bx = boxes + (long long)face * box_stride;
        it[q].X = bx[0];
        it[q].Y = bx[1];
        it[q].W = bx[2];
        it[q].H = bx[3];
        it[q].fr = (const char*)frames + (long long)face_frame[face] * fstride * (U8 ? 1 : 8);
        it[q].node = 0;
      }
      for (int d = 0; d < M.F; ++d) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int4* r = lvl + (long long)it[q].node * K + it[q].k;
          const double2 oa = __ldg(reinterpret_cast<const double2*>(r));
          const double2 ob = __ldg(reinterpret_cast<const double2*>(r + M.split_plane));
          const int4 tail = __ldg(r + 2 * M.split_plane);
          const double thr = __hiloint2double(tail.y, tail.x);
          const int an_a = (short)(tail.z & 0xffff), an_b = (short)(tail.z >> 16);
          const double* cur = sc + it[q].fi * L2;
          const double ia = sample_px<U8>(it[q].fr, w, h, pitch, it[q].X, it[q].Y, it[q].W, it[q].H, cur,
                                          it[q].ab.x, it[q].ab.y, an_a, oa.x, oa.y);
          const double ib = sample_px<U8>(it[q].fr, w, h, pitch, it[q].X, it[q].Y, it[q].W, it[q].H, cur,
                                          it[q].ab.x, it[q].ab.y, an_b, ob.x, ob.y);
          it[q].node = dsub(ia, ib) > thr ? 2 * it[q].node + 1 : 2 * it[q].node + 2;  // ert.cpp:87-97
        }
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int leaf = it[q].node - S;
        sli[it[q].fi * Kp + it[q].k] = (uint8_t)leaf;
        if (leaf_out)
          leaf_out[(long long)(f0 + it[q].fi) * leaf_out_stride + (long long)t * K + it[q].k] = (uint8_t)leaf;
      }
    }
    __syncthreads();
    // (3) leaf sums in tree order, cur += shrinkage * delta (ert.cpp:118-126)
    uint64_t pol = 0;
    if (BL_ERT_EVICT_LAST) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    if (tid < nf * L) {
      const int fi = tid / L, p = tid - fi * L;
      const uint8_t* li = sli + fi * Kp;
      const double2* lv = reinterpret_cast<const double2*>(M.leaves + (long long)t * K * NL * 2 * L) + p;
      const int row = NL * L;
      double ax = 0.0, ay = 0.0;  // the canonical chunked order
      for (int c0 = 0; c0 < K; c0 += kLeafChunk) {
        const int c1 = min(K, c0 + kLeafChunk);
        double px = 0.0, py = 0.0;
        int k = c0;
        for (; k + 16 <= c1; k += 16) {
          double2 v[16];
#if BL_FC_LEAN
          const uint4 li4 = *reinterpret_cast<const uint4*>(li + k);
          const uint32_t lw[4] = {li4.x, li4.y, li4.z, li4.w};
#pragma unroll
          for (int u = 0; u < 16; ++u)
            v[u] = ld_leaf(lv + (k + u) * row + (int)((lw[u >> 2] >> (8 * (u & 3))) & 0xffu) * L, pol);
#else
#pragma unroll
          for (int u = 0; u < 16; ++u) v[u] = ld_leaf(lv + (k + u) * row + li[k + u] * L, pol);
#endif
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            px = dadd(px, v[u].x);
            py = dadd(py, v[u].y);
          }
        }
        for (; k < c1; ++k) {
          const double2 v = ld_leaf(lv + k * row + li[k] * L, pol);
          px = dadd(px, v.x);
          py = dadd(py, v.y);
        }
        ax = dadd(ax, px);
        ay = dadd(ay, py);
      }
      double* c = sc + fi * L2 + 2 * p;
      c[0] = dadd(c[0], dmul(M.shrinkage, ax));
      c[1] = dadd(c[1], dmul(M.shrinkage, ay));
    }
    __syncthreads();
  }
  // ert.cpp:132-133: box.x + p.x * box.w, box.y + p.y * box.h
  for (int e = tid; e < nf * L2; e += blockDim.x) {
    const int fi = e / L2, c = e - fi * L2;
    const int* b = boxes + (long long)(f0 + fi) * box_stride;
    out_xy[(long long)(f0 + fi) * L2 + c] = (c & 1) ? dadd((double)b[1], dmul(sc[e], (double)b[3]))
                                                    : dadd((double)b[0], dmul(sc[e], (double)b[2]));
  }
}

// The cascade for SMALL batches (a camera stream's 16 frames, one frame): latency-bound, a
// face's 15 levels are one dependent chain, so each level is spread over a whole CTA:
//   xform    warp 0: face_transform_warp (shuffle reductions);
//   traverse thread per tree: level-order descent with the root's split record prefetched
//            before the transform, leaf index -> smem;
//   accum    thread per (landmark pair, chunk of kLeafChunk trees): the chunk's selected leaf
//            pairs in tree order, 16 loads in flight, partial -> smem; then thread per pair:
//            the partials in chunk order, cur += shrinkage * delta.
// The leaf sum of a level is then ~kLeafChunk dependent adds and loads deep instead of K.
// Same canonical order as k_ert_cascade / k_ert_accum (bit-identical to both).
#ifndef BL_WD_CLOCK
#define BL_WD_CLOCK 0  // per-phase clock64 totals of face 0, printed (experiments)
#endif
#ifndef BL_WD_LEAN
#define BL_WD_LEAN 1  // k_ert_wide: 16-B leaf-index loads and 32-bit row offsets in the leaf sums
#endif
#ifndef BL_WD_MINB
#define BL_WD_MINB 1  // k_ert_wide CTAs per SM the register budget must allow (experiment)
#endif
constexpr int kWdMaxThreads = 640;  // 96 registers per thread
constexpr int kWdInFlight = 16;  // leaf loads in flight per (pair, chunk) thread

struct SplitPlanes {  // one split record as its three 16-B planes
  double2 oa, ob;
  int4 tail;  // thr (lo, hi), anchors (a | b << 16)
};

int ert_wide_threads(const ErtDev& M) {
  const int items = M.L * (int)div_up(M.K, kLeafChunk);
  return (int)std::min<long long>(kWdMaxThreads, div_up(std::max(std::max(M.K, items), 32), 32) * 32);
}

template <bool U8>
__global__ void __launch_bounds__(kWdMaxThreads, BL_WD_MINB) k_ert_wide(ErtDev M, const void* __restrict__ frames, int w, int h,
                                                     long long pitch, long long fstride,
                                                     const int* __restrict__ face_frame,
                                                     const int* __restrict__ boxes, int box_stride,
                                                     const int* __restrict__ n_faces, int cap,
                                                     double* __restrict__ out_xy, uint8_t* __restrict__ leaf_out,
                                                     long long leaf_out_stride, int* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char wd_smem[];
  const int L = M.L, L2 = 2 * L, K = M.K, S = M.S, NL = M.NL;
  const int nchunk = (K + kLeafChunk - 1) / kLeafChunk;
  double* sc = reinterpret_cast<double*>(wd_smem);             // [2L] current shape
  double* smc = sc + L2;                                       // [2L] centred mean shape
  double2* stf = reinterpret_cast<double2*>(smc + L2);         // [1] transform
  double2* spart = stf + 1;                                    // [nchunk][L] partial leaf sums
  uint8_t* sli = reinterpret_cast<uint8_t*>(spart + nchunk * L);  // [K]
  const int bd = blockDim.x;
  const int n = min(*n_faces, cap);
  const int face = blockIdx.x;
  if (face >= n) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < L2; e += bd) {
    sc[e] = M.mean_xy[e];  // ert.cpp:106
    smc[e] = M.mean_c[e];
  }
  const int* bx = boxes + (long long)face * box_stride;
  const int X = bx[0], Y = bx[1], W = bx[2], H = bx[3];
  const void* fr = (const char*)frames + (long long)face_frame[face] * fstride * (U8 ? 1 : 8);
  __syncthreads();
#if BL_WD_CLOCK
  long long clk[3] = {0, 0, 0};
#endif
  for (int t = 0; t < M.T; ++t) {
    const int4* lvl = reinterpret_cast<const int4*>(M.split) + (long long)t * S * K;
    auto rec = [&](int node, int k, SplitPlanes& r) {
      const int4* q = lvl + (long long)node * K + k;
      r.oa = __ldg(reinterpret_cast<const double2*>(q));
      r.ob = __ldg(reinterpret_cast<const double2*>(q + M.split_plane));
      r.tail = __ldg(q + 2 * M.split_plane);
    };
    SplitPlanes root;  // this thread's first tree's root record: independent of the transform
    if (tid < K && S > 0) rec(0, tid, root);
#if BL_WD_CLOCK
    long long c0 = clock64();
#endif
    if (warp == 0) {  // (1) transform
      double A, B;
      const int e = face_transform_warp(M, sc, smc, lane, A, B);
      if (lane == 0) {
        if (e) atomicExch(err, e);
        stf[0] = make_double2(A, B);
      }
    }
    __syncthreads();
#if BL_WD_CLOCK
    long long c1 = clock64();
#endif
    // (2) traversals, ert.cpp:87-97
    const double2 ab = stf[0];
    for (int k = tid; k < K; k += bd) {
      // both children's records are loaded while a node's pixels are sampled, so a descent
      // step waits on its pixel loads only
      int node = 0;
      SplitPlanes r;
      if (k == tid)
        r = root;
      else
        rec(0, k, r);
      for (int d = 0; d < M.F; ++d) {
        SplitPlanes c1, c2;
        const bool more = d + 1 < M.F;
        if (more) {
          rec(2 * node + 1, k, c1);
          rec(2 * node + 2, k, c2);
        }
        const double thr = __hiloint2double(r.tail.y, r.tail.x);
        const int an_a = (short)(r.tail.z & 0xffff), an_b = (short)(r.tail.z >> 16);
        const double ia = sample_px<U8>(fr, w, h, pitch, X, Y, W, H, sc, ab.x, ab.y, an_a, r.oa.x, r.oa.y);
        const double ib = sample_px<U8>(fr, w, h, pitch, X, Y, W, H, sc, ab.x, ab.y, an_b, r.ob.x, r.ob.y);
        const bool right = dsub(ia, ib) > thr;
        node = right ? 2 * node + 1 : 2 * node + 2;
        if (more) r = right ? c1 : c2;
      }
      sli[k] = (uint8_t)(node - S);
      if (leaf_out) leaf_out[(long long)face * leaf_out_stride + (long long)t * K + k] = (uint8_t)(node - S);
    }
    __syncthreads();
#if BL_WD_CLOCK
    long long c2 = clock64();
#endif
    // (3a) partial leaf sums: item = (chunk, pair), consecutive threads read consecutive pairs
    // of one leaf row
    const double2* lv = reinterpret_cast<const double2*>(M.leaves + (long long)t * K * NL * L2);
    const int row = NL * L;  // double2 per tree
    for (int it = tid; it < nchunk * L; it += bd) {
      const int ch = it / L, p = it - ch * L;
      const int k0 = ch * kLeafChunk, k1 = min(K, k0 + kLeafChunk);
      double px = 0.0, py = 0.0;
      int k = k0;
#if BL_WD_LEAN
      // 16 leaf indices per 16-B shared load, 32-bit row offsets from the chunk's base
      const double2* src = lv + (long long)k0 * row + p;
      for (int qrow = 0; k + kWdInFlight <= k1; k += kWdInFlight, qrow += kWdInFlight * row) {
        const uint4 li4 = *reinterpret_cast<const uint4*>(sli + k);
        const uint32_t lw[4] = {li4.x, li4.y, li4.z, li4.w};
        double2 v[kWdInFlight];
#pragma unroll
        for (int u = 0; u < kWdInFlight; ++u)
          v[u] = __ldg(src + (qrow + u * row + (int)((lw[u >> 2] >> (8 * (u & 3))) & 0xffu) * L));
#pragma unroll
        for (int u = 0; u < kWdInFlight; ++u) {
          px = dadd(px, v[u].x);
          py = dadd(py, v[u].y);
        }
      }
#endif
      for (; k + kWdInFlight <= k1; k += kWdInFlight) {
        double2 v[kWdInFlight];
#pragma unroll
        for (int u = 0; u < kWdInFlight; ++u) v[u] = __ldg(lv + (long long)(k + u) * row + sli[k + u] * L + p);
#pragma unroll
        for (int u = 0; u < kWdInFlight; ++u) {
          px = dadd(px, v[u].x);
          py = dadd(py, v[u].y);
        }
      }
      for (; k < k1; ++k) {
        const double2 v = __ldg(lv + (long long)k * row + sli[k] * L + p);
        px = dadd(px, v.x);
        py = dadd(py, v.y);
      }
      spart[it] = make_double2(px, py);
    }
    __syncthreads();
    // (3b) partials in chunk order, cur += shrinkage * delta (ert.cpp:118-126)
    if (tid < L) {
      double ax = 0.0, ay = 0.0;
      for (int ch = 0; ch < nchunk; ++ch) {
        const double2 q = spart[ch * L + tid];
        ax = dadd(ax, q.x);
        ay = dadd(ay, q.y);
      }
      sc[2 * tid] = dadd(sc[2 * tid], dmul(M.shrinkage, ax));
      sc[2 * tid + 1] = dadd(sc[2 * tid + 1], dmul(M.shrinkage, ay));
    }
    __syncthreads();
#if BL_WD_CLOCK
    long long c3 = clock64();
    if (tid == 0) { clk[0] += c1 - c0; clk[1] += c2 - c1; clk[2] += c3 - c2; }
#endif
  }
#if BL_WD_CLOCK
  if (tid == 0 && face == 0) printf("k_ert_wide face 0 cycles: xform %lld traverse %lld accum %lld\n", clk[0], clk[1], clk[2]);
#endif
  // ert.cpp:132-133: box.x + p.x * box.w, box.y + p.y * box.h
  for (int c = tid; c < L2; c += bd)
    out_xy[(long long)face * L2 + c] = (c & 1) ? dadd((double)Y, dmul(sc[c], (double)H))
                                               : dadd((double)X, dmul(sc[c], (double)W));
}

// The small-batch cascade spread over a CLUSTER of CL CTAs per face.  Per level a face reads
// K selected leaf rows (544 KB at 500 trees, L = 68): through one SM's L2 port that is ~9k
// cycles, the largest part of k_ert_wide's level.  Here CTA rank r of the face's cluster
// traverses the trees of chunks c = r, r + CL, ... and sums their leaf rows (same per-chunk
// canonical order as k_ert_wide / k_ert_cascade), broadcasts the chunk partials into every
// CTA's shared memory (DSMEM), and after one cluster barrier every CTA applies the identical
// update (partials in chunk order, ert.cpp:118-126) to its own copy of the shape; the
// transform (warp 0) is computed redundantly and identically in each CTA.  Bit-identical to
// k_ert_wide.
#ifndef BL_ERT_SPEC2
#define BL_ERT_SPEC2 1  // k_ert_wcl traversal: two depths per pixel round trip (speculative children;
                        // all 15 nodes at once measured slower: C1 0.289 vs 0.216 ms, stack use)
#endif
#ifndef BL_ERT_SREC
#define BL_ERT_SREC 1  // split records of my trees staged in shared memory one level ahead
#endif

// shared-memory plan of k_ert_wcl (host and device compute the same offsets)
struct WclSmem {
  int my_chunks_max, items_max;
  bool staged, srec;
  size_t stage_off, srec_off, total;
};
BL_HD_INLINE WclSmem wcl_smem(int L, int K, int S, int CL, int threads) {
  WclSmem m;
  const int nchunk = (K + kLeafChunk - 1) / kLeafChunk;
  m.my_chunks_max = (nchunk + CL - 1) / CL;
  m.items_max = m.my_chunks_max * L;
  m.staged = m.items_max <= threads;
  m.srec = BL_ERT_SREC && m.staged && S > 0;
  size_t off = sizeof(double) * 4 * (size_t)L + sizeof(double2) * (1 + 2 * (size_t)nchunk * L) + (size_t)((K + kLeafChunk - 1) / kLeafChunk * kLeafChunk);
  m.stage_off = off;
  if (m.staged) off += sizeof(double2) * kLeafChunk * (size_t)m.items_max;
  m.srec_off = off;
  const size_t recs = sizeof(int4) * 3 * (size_t)S * kLeafChunk * m.my_chunks_max;
  if (off + recs > 227u * 1024u) m.srec = false;  // the per-CTA shared-memory opt-in limit
  if (m.srec) off += recs;
  m.total = off;
  return m;
}

template <bool U8, int CL>
__global__ void __launch_bounds__(256) k_ert_wcl(ErtDev M, const void* __restrict__ frames, int w, int h,
                                                 long long pitch, long long fstride,
                                                 const int* __restrict__ face_frame,
                                                 const int* __restrict__ boxes, int box_stride,
                                                 const int* __restrict__ n_faces, int cap,
                                                 double* __restrict__ out_xy, uint8_t* __restrict__ leaf_out,
                                                 long long leaf_out_stride, int* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char wd_smem[];
  const int L = M.L, L2 = 2 * L, K = M.K, S = M.S, NL = M.NL;
  const int nchunk = (K + kLeafChunk - 1) / kLeafChunk;
  double* sc = reinterpret_cast<double*>(wd_smem);             // [2L] current shape
  double* smc = sc + L2;                                       // [2L] centred mean shape
  double2* stf = reinterpret_cast<double2*>(smc + L2);         // [1] transform
  double2* spart = stf + 1;                                    // [2][nchunk][L] partial leaf sums (by level parity)
  uint8_t* sli = reinterpret_cast<uint8_t*>(spart + 2 * nchunk * L);  // [K]
  const int bd = blockDim.x;
  const WclSmem plan = wcl_smem(L, K, S, CL, bd);
  // [kLeafChunk][items] leaf pairs of this CTA's items, landed by cp.async (16-B aligned)
  double2* stage = reinterpret_cast<double2*>(wd_smem + plan.stage_off);
  // the next level's split records of my trees, [3 planes][S][my trees] (cp.async, landed
  // during this level's accumulation, cluster barrier and transform)
  int4* srecs = reinterpret_cast<int4*>(wd_smem + plan.srec_off);
  const int n = min(*n_faces, cap);
  const int face = blockIdx.x / CL;
  const unsigned rank = blockIdx.x % CL;  // == %cluster_ctarank for cluster dims (CL, 1, 1)
  if (face >= n) return;                  // the whole cluster leaves together
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < L2; e += bd) {
    sc[e] = M.mean_xy[e];  // ert.cpp:106
    smc[e] = M.mean_c[e];
  }
  const int* bx = boxes + (long long)face * box_stride;
  const int X = bx[0], Y = bx[1], W = bx[2], H = bx[3];
  const void* fr = (const char*)frames + (long long)face_frame[face] * fstride * (U8 ? 1 : 8);
  // my chunks: rank, rank + CL, ...; my trees: kLeafChunk per chunk
  const int my_chunks = nchunk > (int)rank ? (nchunk - 1 - (int)rank) / CL + 1 : 0;
  const int my_trees = my_chunks * kLeafChunk;
  const bool srec = plan.srec;
  auto tree_of = [&](int lt) { return (int)(rank + CL * (lt / kLeafChunk)) * kLeafChunk + lt % kLeafChunk; };
  // DSMEM base addresses of spart in every CTA of the cluster
  uint32_t rpart[CL];
  {
    const uint32_t local = (uint32_t)__cvta_generic_to_shared(spart);
#pragma unroll
    for (int q = 0; q < CL; ++q)
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rpart[q]) : "r"(local), "r"(q));
  }
  // level t's split records of my trees -> srecs (cp.async, one commit group), issued by
  // threads [t0, bd) while warp 0 computes the level's transform: they land before the
  // traversal needs them, off the level's critical path
  auto copy_recs = [&](int t, int t0) {
    const int4* src = reinterpret_cast<const int4*>(M.split) + (long long)t * S * K;
    for (int lt = tid - t0; lt < my_trees; lt += bd - t0) {
      const int k = tree_of(lt);
      if (k >= K) continue;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(srecs + lt);
      for (int pl = 0; pl < 3; ++pl)
        for (int nd = 0; nd < S; ++nd)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + (uint32_t)((pl * S + nd) * my_trees * 16)),
                       "l"(src + (long long)pl * M.split_plane + (long long)nd * K + k)
                       : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  __syncthreads();
#if BL_WD_CLOCK
  long long clk[7] = {0, 0, 0, 0, 0, 0, 0};
#endif
  for (int t = 0; t < M.T; ++t) {
#if BL_WD_CLOCK
    const long long c0 = clock64();
#endif
    const int4* lvl = reinterpret_cast<const int4*>(M.split) + (long long)t * S * K;
    auto rec = [&](int node, int k, SplitPlanes& r) {
      const int4* q = lvl + (long long)node * K + k;
      r.oa = __ldg(reinterpret_cast<const double2*>(q));
      r.ob = __ldg(reinterpret_cast<const double2*>(q + M.split_plane));
      r.tail = __ldg(q + 2 * M.split_plane);
    };
    auto rec_s = [&](int node, int lt, SplitPlanes& r) {  // lt: my local tree index
      const int4* q = srecs + node * my_trees + lt;
      const int4 a = q[0], b = q[S * my_trees], c = q[2 * S * my_trees];
      r.oa = make_double2(__hiloint2double(a.y, a.x), __hiloint2double(a.w, a.z));
      r.ob = make_double2(__hiloint2double(b.y, b.x), __hiloint2double(b.w, b.z));
      r.tail = c;
    };
    SplitPlanes root;
    const int k_first = tid < my_trees ? tree_of(tid) : K;
    if (!srec && k_first < K && S > 0) rec(0, k_first, root);
    if (srec && (bd == 32 || warp > 0)) copy_recs(t, bd == 32 ? 0 : 32);
    if (warp == 0) {  // (1) transform (identical in every CTA of the cluster)
      double A, B;
      const int e = face_transform_warp(M, sc, smc, lane, A, B);
      if (lane == 0) {
        if (e && rank == 0) atomicExch(err, e);
        stf[0] = make_double2(A, B);
      }
    }
    if (srec) asm volatile("cp.async.wait_group 0;" ::: "memory");  // this level's records landed
    __syncthreads();
#if BL_WD_CLOCK
    const long long c1 = clock64();
#endif
    // (2) traversals of my trees, ert.cpp:87-97
    const double2 ab = stf[0];
    for (int lt = tid; lt < my_trees; lt += bd) {
      const int k = tree_of(lt);
      if (k >= K) continue;
      int node = 0;
      SplitPlanes r;
      const int jl = lt;
      if (srec) {  // records in shared memory: no prefetch of the children needed
        // two depths per step: the node's and both children's pixels are sampled together
        // (6 loads in flight), then both decisions are taken -- one pixel round trip per two
        // depths; the same decisions as the one-node walk (ert.cpp:87-97)
        auto px_of = [&](const SplitPlanes& q, bool second) {
          const int an = second ? (short)(q.tail.z >> 16) : (short)(q.tail.z & 0xffff);
          const double2 o = second ? q.ob : q.oa;
          return sample_px<U8>(fr, w, h, pitch, X, Y, W, H, sc, ab.x, ab.y, an, o.x, o.y);
        };
        int d = 0;
        for (; BL_ERT_SPEC2 && d + 2 <= M.F; d += 2) {
          SplitPlanes r0, r1, r2;
          rec_s(node, jl, r0);
          rec_s(2 * node + 1, jl, r1);
          rec_s(2 * node + 2, jl, r2);
          const double i0a = px_of(r0, false), i0b = px_of(r0, true);
          const double i1a = px_of(r1, false), i1b = px_of(r1, true);
          const double i2a = px_of(r2, false), i2b = px_of(r2, true);
          const bool right0 = dsub(i0a, i0b) > __hiloint2double(r0.tail.y, r0.tail.x);
          const int c = right0 ? 2 * node + 1 : 2 * node + 2;
          const SplitPlanes& rc = right0 ? r1 : r2;
          const bool right1 = dsub(right0 ? i1a : i2a, right0 ? i1b : i2b) > __hiloint2double(rc.tail.y, rc.tail.x);
          node = right1 ? 2 * c + 1 : 2 * c + 2;
        }
        for (; d < M.F; ++d) {
          rec_s(node, jl, r);
          const double thr = __hiloint2double(r.tail.y, r.tail.x);
          const int an_a = (short)(r.tail.z & 0xffff), an_b = (short)(r.tail.z >> 16);
          const double ia = sample_px<U8>(fr, w, h, pitch, X, Y, W, H, sc, ab.x, ab.y, an_a, r.oa.x, r.oa.y);
          const double ib = sample_px<U8>(fr, w, h, pitch, X, Y, W, H, sc, ab.x, ab.y, an_b, r.ob.x, r.ob.y);
          node = dsub(ia, ib) > thr ? 2 * node + 1 : 2 * node + 2;
        }
        sli[k] = (uint8_t)(node - S);
        if (leaf_out) leaf_out[(long long)face * leaf_out_stride + (long long)t * K + k] = (uint8_t)(node - S);
        continue;
      }
      if (lt == tid)
        r = root;
      else
        rec(0, k, r);
      for (int d = 0; d < M.F; ++d) {
        SplitPlanes c1, c2;
        const bool more = d + 1 < M.F;
        if (more) {
          rec(2 * node + 1, k, c1);
          rec(2 * node + 2, k, c2);
        }
        const double thr = __hiloint2double(r.tail.y, r.tail.x);
        const int an_a = (short)(r.tail.z & 0xffff), an_b = (short)(r.tail.z >> 16);
        const double ia = sample_px<U8>(fr, w, h, pitch, X, Y, W, H, sc, ab.x, ab.y, an_a, r.oa.x, r.oa.y);
        const double ib = sample_px<U8>(fr, w, h, pitch, X, Y, W, H, sc, ab.x, ab.y, an_b, r.ob.x, r.ob.y);
        const bool right = dsub(ia, ib) > thr;
        node = right ? 2 * node + 1 : 2 * node + 2;
        if (more) r = right ? c1 : c2;
      }
      sli[k] = (uint8_t)(node - S);
      if (leaf_out) leaf_out[(long long)face * leaf_out_stride + (long long)t * K + k] = (uint8_t)(node - S);
    }
    __syncthreads();
#if BL_WD_CLOCK
    const long long c2 = clock64();
#endif
    // (3a) partial leaf sums of my chunks, broadcast to every CTA's spart[t & 1]
    const double2* lv = reinterpret_cast<const double2*>(M.leaves + (long long)t * K * NL * L2);
    const int row = NL * L;
    const uint32_t boff = (uint32_t)((t & 1) * nchunk * L) * (uint32_t)sizeof(double2);
    const int items = my_chunks * L;
    for (int it = tid; it < items; it += bd) {
      const int ci = it / L, p = it - ci * L;
      const int ch = (int)rank + CL * ci;
      const int k0 = ch * kLeafChunk, k1 = min(K, k0 + kLeafChunk);
      double px = 0.0, py = 0.0;
      if (items <= bd) {
        // every selected leaf pair of the chunk in flight at once: cp.async into this item's
        // column of the staging buffer ([tree][item]: conflict-free), one wait, then the
        // tree-ordered sum from shared memory -- one L2 round trip instead of K/16
        // (lean: 32-bit offsets, running pointers, no per-tree predicates -- the kernel runs
        // 3 warps per SM, so its level time is mostly instruction issue)
        const uint32_t istride = (uint32_t)items * 16u;
        const uint32_t st0 = (uint32_t)__cvta_generic_to_shared(stage + it);
        const int nk = k1 - k0;
        {
          // the chunk's leaf indices into registers first: an LDS after an LDGSTS waits for
          // it (possible aliasing), which serialised the issue loop at ~60 cycles per tree
          uint32_t lw[kLeafChunk / 4];
#pragma unroll
          for (int q = 0; q < kLeafChunk / 16; ++q) {
            const uint4 v = *reinterpret_cast<const uint4*>(sli + k0 + 16 * q);
            lw[4 * q] = v.x;
            lw[4 * q + 1] = v.y;
            lw[4 * q + 2] = v.z;
            lw[4 * q + 3] = v.w;
          }
          const double2* src = lv + (long long)k0 * row + p;
          uint32_t dst = st0;
          int roff = 0;
#pragma unroll
          for (int j = 0; j < kLeafChunk; ++j) {
            if (j < nk)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                           "l"(src + (roff + (int)((lw[j >> 2] >> (8 * (j & 3))) & 0xffu) * L)));
            dst += istride;
            roff += row;
          }
#if BL_WD_CLOCK
          const long long ca = clock64();
#endif
          asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
#if BL_WD_CLOCK
          const long long cb = clock64();
          if (tid == 0) { clk[4] += ca - c2; clk[5] += cb - ca; }
#endif
        }
        const double2* sp = stage + it;
#pragma unroll 16
        for (int j = 0; j < nk; ++j) {
          const double2 v = *sp;
          px = dadd(px, v.x);
          py = dadd(py, v.y);
          sp += items;
        }
#if BL_WD_CLOCK
        if (tid == 0) clk[6] -= clock64();
#endif
      } else {
        int k = k0;
        for (; k + kWdInFlight <= k1; k += kWdInFlight) {
          double2 v[kWdInFlight];
#pragma unroll
          for (int u = 0; u < kWdInFlight; ++u) v[u] = __ldg(lv + (long long)(k + u) * row + sli[k + u] * L + p);
#pragma unroll
          for (int u = 0; u < kWdInFlight; ++u) {
            px = dadd(px, v[u].x);
            py = dadd(py, v[u].y);
          }
        }
        for (; k < k1; ++k) {
          const double2 v = __ldg(lv + (long long)k * row + sli[k] * L + p);
          px = dadd(px, v.x);
          py = dadd(py, v.y);
        }
      }
      const uint32_t off = boff + (uint32_t)(ch * L + p) * (uint32_t)sizeof(double2);
#pragma unroll
      for (int q = 0; q < CL; ++q)
        asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(rpart[q] + off), "d"(px), "d"(py) : "memory");
#if BL_WD_CLOCK
      if (tid == 0) clk[6] += clock64();
#endif
    }
    // every chunk's partial is in every CTA (release / acquire across the cluster)
#if BL_WD_CLOCK
    const long long c3 = clock64();
#endif
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
#if BL_WD_CLOCK
    const long long c4 = clock64();
    if (tid == 0) {
      clk[0] += c1 - c0;
      clk[1] += c2 - c1;
      clk[2] += c3 - c2;
      clk[3] += c4 - c3;
    }
#endif
    // (3b) partials in chunk order, cur += shrinkage * delta (ert.cpp:118-126), same in every CTA
    if (tid < L) {
      const double2* pp = spart + (t & 1) * nchunk * L;
      double ax = 0.0, ay = 0.0;
      for (int ch = 0; ch < nchunk; ++ch) {
        const double2 q = pp[ch * L + tid];
        ax = dadd(ax, q.x);
        ay = dadd(ay, q.y);
      }
      sc[2 * tid] = dadd(sc[2 * tid], dmul(M.shrinkage, ax));
      sc[2 * tid + 1] = dadd(sc[2 * tid + 1], dmul(M.shrinkage, ay));
    }
    __syncthreads();
  }
#if BL_WD_CLOCK
  if (tid == 0 && face == 0)
    printf("k_ert_wcl face 0 rank %u cycles: xform %lld traverse %lld accum %lld (issue %lld wait %lld bcast %lld) cluster-sync %lld\n", rank, clk[0],
           clk[1], clk[2], clk[4], clk[5], clk[6], clk[3]);
#endif
  // no CTA may exit while another could still write into its shared memory: every remote
  // write of the last level precedes the last cluster barrier, so exiting is safe here
  if (rank == 0)
    for (int c = tid; c < L2; c += bd)
      out_xy[(long long)face * L2 + c] = (c & 1) ? dadd((double)Y, dmul(sc[c], (double)H))
                                                 : dadd((double)X, dmul(sc[c], (double)W));
}

template <bool U8, int CL>
static cudaError_t launch_wcl(const Launch& L, const ErtDev& M, const void* frames, int w, int h, long long pitch,
                              long long fstride, const int* face_frame, const int* boxes, int box_stride,
                              const int* n_faces, int cap, double* out_xy, uint8_t* leaf_out,
                              long long leaf_out_stride, int* err) {
  const int nchunk = (int)div_up(M.K, kLeafChunk);
  const int my_chunks = (nchunk + CL - 1) / CL;
  const int threads = (int)std::min<long long>(256, div_up(std::max(my_chunks * std::max(kLeafChunk, M.L), 32), 32) * 32);
  const size_t smem = wcl_smem(M.L, M.K, M.S, CL, threads).total;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cap * CL);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = L.st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (CL > 8) cudaFuncSetAttribute(k_ert_wcl<U8, CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return cudaLaunchKernelEx(&cfg, k_ert_wcl<U8, CL>, M, frames, w, h, pitch, fstride, face_frame, boxes, box_stride,
                            n_faces, cap, out_xy, leaf_out, leaf_out_stride, err);
}

bool ert_wide_fits(const ErtDev& M) { return 2 * M.L <= kMaxL2; }

void launch_ert_wide(const Launch& L, const ErtDev& M, const void* frames, int u8, int w, int h, long long pitch,
                     long long fstride, const int* face_frame, const int* boxes, int box_stride, const int* n_faces,
                     int cap, double* out_xy, uint8_t* leaf_out, long long leaf_out_stride, int* err, int cl_req) {
  const int cl = cl_req;  // 1: one CTA per face; 2, 4, 8: a cluster of that many CTAs per face
  if (cl == 2 || cl == 4 || cl == 8 || cl == 16) {
    cudaError_t r = cudaSuccess;
    if (cl == 2)
      r = u8 ? launch_wcl<true, 2>(L, M, frames, w, h, pitch, fstride, face_frame, boxes, box_stride, n_faces, cap, out_xy, leaf_out, leaf_out_stride, err)
             : launch_wcl<false, 2>(L, M, frames, w, h, pitch, fstride, face_frame, boxes, box_stride, n_faces, cap, out_xy, leaf_out, leaf_out_stride, err);
    else if (cl == 4)
      r = u8 ? launch_wcl<true, 4>(L, M, frames, w, h, pitch, fstride, face_frame, boxes, box_stride, n_faces, cap, out_xy, leaf_out, leaf_out_stride, err)
             : launch_wcl<false, 4>(L, M, frames, w, h, pitch, fstride, face_frame, boxes, box_stride, n_faces, cap, out_xy, leaf_out, leaf_out_stride, err);
    else if (cl == 8)
      r = u8 ? launch_wcl<true, 8>(L, M, frames, w, h, pitch, fstride, face_frame, boxes, box_stride, n_faces, cap, out_xy, leaf_out, leaf_out_stride, err)
             : launch_wcl<false, 8>(L, M, frames, w, h, pitch, fstride, face_frame, boxes, box_stride, n_faces, cap, out_xy, leaf_out, leaf_out_stride, err);
    else  // 16: a non-portable cluster size
      r = u8 ? launch_wcl<true, 16>(L, M, frames, w, h, pitch, fstride, face_frame, boxes, box_stride, n_faces, cap, out_xy, leaf_out, leaf_out_stride, err)
             : launch_wcl<false, 16>(L, M, frames, w, h, pitch, fstride, face_frame, boxes, box_stride, n_faces, cap, out_xy, leaf_out, leaf_out_stride, err);
    (void)r;
    ++*L.counter;
    return;
  }
  const long long nchunk = div_up(M.K, kLeafChunk);
  const size_t smem = sizeof(double) * 4 * M.L + sizeof(double2) * (1 + nchunk * M.L) + (size_t)M.K;
  const int threads = ert_wide_threads(M);
  if (u8)
    k_ert_wide<true><<<(unsigned)cap, threads, smem, L.st>>>(M, frames, w, h, pitch, fstride, face_frame, boxes,
                                                              box_stride, n_faces, cap, out_xy, leaf_out,
                                                              leaf_out_stride, err);
  else
    k_ert_wide<false><<<(unsigned)cap, threads, smem, L.st>>>(M, frames, w, h, pitch, fstride, face_frame, boxes,
                                                               box_stride, n_faces, cap, out_xy, leaf_out,
                                                               leaf_out_stride, err);
  ++*L.counter;
}

bool ert_cascade_fits(const ErtDev& M) {
  return M.L * kFcFaces <= kFcThreads && 2 * M.L <= kMaxL2;
}

void launch_ert_cascade(const Launch& L, const ErtDev& M, const void* frames, int u8, int w, int h, long long pitch,
                        long long fstride, const int* face_frame, const int* boxes, int box_stride,
                        const int* n_faces, int cap, double* out_xy, uint8_t* leaf_out, long long leaf_out_stride,
                        int* err) {
  const size_t smem =
      sizeof(double) * kFcFaces * 2 * M.L + sizeof(double2) * kFcFaces + (size_t)kFcFaces * fc_sli_stride(M.K);
  const unsigned grid = (unsigned)div_up(cap, kFcFaces);
  if (u8)
    k_ert_cascade<true><<<grid, kFcThreads, smem, L.st>>>(M, frames, w, h, pitch, fstride, face_frame, boxes, box_stride,
                                                   n_faces, cap, out_xy, leaf_out, leaf_out_stride, err);
  else
    k_ert_cascade<false><<<grid, kFcThreads, smem, L.st>>>(M, frames, w, h, pitch, fstride, face_frame, boxes, box_stride,
                                                    n_faces, cap, out_xy, leaf_out, leaf_out_stride, err);
  ++*L.counter;
}

__global__ void k_ert_finish(ErtDev M, const int* __restrict__ boxes, int box_stride,
                             const int* __restrict__ n_faces, int cap, const double* __restrict__ cur,
                             double* __restrict__ out) {
  const int n = min(*n_faces, cap);
  const int L2 = 2 * M.L;
  const long long total = (long long)n * L2;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long face = i / L2;
    const int c = (int)(i - face * L2);
    const int* b = boxes + face * box_stride;
    // ert.cpp:132-133: box.x + p.x * box.w, box.y + p.y * box.h
    out[i] = (c & 1) ? dadd((double)b[1], dmul(cur[i], (double)b[3]))
                     : dadd((double)b[0], dmul(cur[i], (double)b[2]));
  }
}

void launch_ert_finish(const Launch& L, const ErtDev& M, const int* boxes, int box_stride,
                       const int* n_faces, int cap, const double* cur, double* out_xy) {
  k_ert_finish<<<148 * 4, 256, 0, L.st>>>(M, boxes, box_stride, n_faces, cap, cur, out_xy);
  ++*L.counter;
}

void configure_ert_kernels(int optin) {  // per device, see configure_screen_tc_kernels
  smem_optin(k_ert_wide<true>, optin);
  smem_optin(k_ert_wide<false>, optin);
  smem_optin(k_ert_cascade<true>, optin);
  smem_optin(k_ert_cascade<false>, optin);
  smem_optin(k_ert_wcl<true, 2>, optin);
  smem_optin(k_ert_wcl<false, 2>, optin);
  smem_optin(k_ert_wcl<true, 4>, optin);
  smem_optin(k_ert_wcl<false, 4>, optin);
  smem_optin(k_ert_wcl<true, 8>, optin);
  smem_optin(k_ert_wcl<false, 8>, optin);
  smem_optin(k_ert_wcl<true, 16>, optin);
  smem_optin(k_ert_wcl<false, 16>, optin);
}

}  // namespace blb
