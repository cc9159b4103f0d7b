// Ensemble-of-regression-trees 68-landmark cascade (ert.cpp:15-136) on the device.
//
// The cascade levels are strictly sequential (ert.cpp:108); within a level every face and
// every tree is independent.  Per level three fully parallel kernels:
//   1. k_ert_xform    thread per face: similarity transform current -> mean (ert.cpp:26-69),
//                     sums sequential in the reference's order (bit-identical), then CUDA's
//                     hypot/atan2/cos/sin (<= 2 ulp from glibc: the only non-bit-exact step);
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

// (1) similarity_transform(current, mean) per face, ert.cpp:26-69: sequential sums in the
// reference's order (bit-identical), then CUDA hypot/atan2/cos/sin.  Stores the linear part
// (scale*cos, scale*sin) that apply_linear recomputes for every sample (ert.cpp:21-22).
__global__ void __launch_bounds__(128) k_ert_xform(ErtDev M, const int* __restrict__ n_faces, int cap,
                                                   const double* __restrict__ cur_g, double2* __restrict__ tf,
                                                   int* __restrict__ err) {
  const int n = min(*n_faces, cap);
  const int face = blockIdx.x * blockDim.x + threadIdx.x;
  if (face >= n) return;
  const double* cur = cur_g + (long long)face * 2 * M.L;
  double mfx = 0.0, mfy = 0.0;
  for (int i = 0; i < M.L; ++i) {
    mfx = dadd(mfx, cur[2 * i]);
    mfy = dadd(mfy, cur[2 * i + 1]);
  }
  mfx = ddiv(mfx, (double)M.L);
  mfy = ddiv(mfy, (double)M.L);
  double sff = 0.0, sre = 0.0, sim = 0.0;
  for (int i = 0; i < M.L; ++i) {
    const double fx = dsub(cur[2 * i], mfx);
    const double fy = dsub(cur[2 * i + 1], mfy);
    const double txp = dsub(__ldg(M.mean_xy + 2 * i), M.mean_cx);
    const double typ = dsub(__ldg(M.mean_xy + 2 * i + 1), M.mean_cy);
    sff = dadd(sff, dadd(dmul(fx, fx), dmul(fy, fy)));
    sre = dadd(sre, dadd(dmul(fx, txp), dmul(fy, typ)));
    sim = dadd(sim, dsub(dmul(fx, typ), dmul(fy, txp)));
  }
  double A = 0.0, B = 0.0;
  if (!(sff > 0.0)) {
    atomicExch(err, 1);  // "source shape has no spread" (ert.cpp:56-57)
  } else {
    const double a = ddiv(sre, sff), b = ddiv(sim, sff);
    const double scale = hypot(a, b);
    if (!(scale > 0.0)) {
      atomicExch(err, 2);  // "target shape has no spread" (ert.cpp:62-63)
    } else {
      const double rot = atan2(b, a);
      A = dmul(scale, cos(rot));
      B = dmul(scale, sin(rot));
    }
  }
  tf[face] = make_double2(A, B);
}

// (2) one thread per (face, tree): traverse_tree (ert.cpp:87-97) with sample_intensity
// (ert.cpp:71-85) on the ORIGINAL frame; writes the leaf index.
template <bool U8>
__global__ void __launch_bounds__(256) k_ert_traverse(ErtDev M, int t, const void* __restrict__ frames, int w,
                                                      int h, long long pitch, long long fstride,
                                                      const int* __restrict__ face_frame,
                                                      const int* __restrict__ boxes, int box_stride,
                                                      const int* __restrict__ n_faces, int cap,
                                                      const double* __restrict__ cur_g,
                                                      const double2* __restrict__ tf,
                                                      uint8_t* __restrict__ leaf_idx, long long leaf_stride) {
  const int n = min(*n_faces, cap);
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int K = M.K, S = M.S;
  if (g >= (long long)n * K) return;
  const int face = (int)(g / K), k = (int)(g - (long long)face * K);
  const double2 ab = tf[face];
  const double* cur = cur_g + (long long)face * 2 * M.L;
  const int* bx = boxes + (long long)face * box_stride;
  const int X = bx[0], Y = bx[1], W = bx[2], H = bx[3];
  const void* fr = (const char*)frames + (long long)face_frame[face] * fstride * (U8 ? 1 : 8);
  const long long tree = (long long)t * K + k;
  int node = 0;
  while (node < S) {
    const long long sn = tree * S + node;
    const short2 an = *reinterpret_cast<const short2*>(M.anchors + 2 * sn);
    const double* sp = M.split + 5 * sn;
    const double ia = sample_px<U8>(fr, w, h, pitch, X, Y, W, H, cur, ab.x, ab.y, an.x, __ldg(sp), __ldg(sp + 1));
    const double ib = sample_px<U8>(fr, w, h, pitch, X, Y, W, H, cur, ab.x, ab.y, an.y, __ldg(sp + 2), __ldg(sp + 3));
    node = dsub(ia, ib) > __ldg(sp + 4) ? 2 * node + 1 : 2 * node + 2;
  }
  leaf_idx[(long long)face * leaf_stride + k] = (uint8_t)(node - S);
}

// (3) one thread per (face, coordinate): sum the K selected leaf rows IN TREE ORDER in fp64
// (ert.cpp:118-121), then cur += shrinkage * delta (ert.cpp:123-126).  Consecutive threads
// read consecutive coordinates of one leaf row (coalesced, L2-resident for the level); the
// loads of 16 trees are issued ahead of their adds.
__global__ void __launch_bounds__(256) k_ert_accum(ErtDev M, int t, const int* __restrict__ n_faces, int cap,
                                                   double* __restrict__ cur_g,
                                                   const uint8_t* __restrict__ leaf_idx, long long leaf_stride) {
  const int n = min(*n_faces, cap);
  const int L2 = 2 * M.L, K = M.K, NL = M.NL;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (long long)n * L2) return;
  const int face = (int)(g / L2), c = (int)(g - (long long)face * L2);
  const uint8_t* li = leaf_idx + (long long)face * leaf_stride;
  const double* lv = M.leaves + (long long)t * K * NL * L2 + c;
  double acc = 0.0;
  int k = 0;
  for (; k + 16 <= K; k += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldg(lv + ((long long)(k + u) * NL + li[k + u]) * L2);
#pragma unroll
    for (int u = 0; u < 16; ++u) acc = dadd(acc, v[u]);
  }
  for (; k < K; ++k) acc = dadd(acc, __ldg(lv + ((long long)k * NL + li[k]) * L2));
  double* cur = cur_g + (long long)face * L2 + c;
  *cur = dadd(*cur, dmul(M.shrinkage, acc));
}

void launch_ert_level(const Launch& L, const ErtDev& M, int t, const void* frames, int u8, int w, int h,
                      long long pitch, long long fstride, const int* face_frame, const int* boxes, int box_stride,
                      const int* n_faces, int cap, double* cur, double2* tf, uint8_t* leaf_idx,
                      long long leaf_stride, int* err) {
  k_ert_xform<<<(unsigned)div_up(cap, 128), 128, 0, L.st>>>(M, n_faces, cap, cur, tf, err);
  const long long pairs = (long long)cap * M.K;
  if (u8)
    k_ert_traverse<true><<<(unsigned)div_up(pairs, 256), 256, 0, L.st>>>(
        M, t, frames, w, h, pitch, fstride, face_frame, boxes, box_stride, n_faces, cap, cur, tf, leaf_idx, leaf_stride);
  else
    k_ert_traverse<false><<<(unsigned)div_up(pairs, 256), 256, 0, L.st>>>(
        M, t, frames, w, h, pitch, fstride, face_frame, boxes, box_stride, n_faces, cap, cur, tf, leaf_idx, leaf_stride);
  k_ert_accum<<<(unsigned)div_up((long long)cap * 2 * M.L, 256), 256, 0, L.st>>>(M, t, n_faces, cap, cur, leaf_idx,
                                                                                leaf_stride);
  *L.counter += 3;
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

}  // namespace blb
