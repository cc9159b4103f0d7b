/* TEST INFRASTRUCTURE ONLY -- see blink_oracle.h.
 *
 * Plain-C restatement of the reference hot path.  Every function cites the reference
 * file:line it follows (paths relative to /root/reference/proj).  Expressions are written
 * in the reference's evaluation order; with -ffp-contract=off (oracle/Makefile) each
 * double operation rounds exactly as the reference's -O2 x86-64 build does. */
#define _GNU_SOURCE
#include "blink_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return -1;
}

const char* orc_last_error(void) { return g_err; }

/* std::clamp(v, lo, hi) = v < lo ? lo : (hi < v ? hi : v) */
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }
static int clampi(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }
/* std::min(a, b) = (b < a) ? b : a */
static double mind(double a, double b) { return (b < a) ? b : a; }

/* ------------------------------------------------------------------ image ---- */

/* image.cpp:129-156 */
int orc_downscale_bilinear(const double* px, int w, int h, double* out) {
  if (w < 2 || h < 2) return fail("downscale_bilinear: output dimension would be 0");
  const int dw = w * 5 / 6, dh = h * 5 / 6;
  const double rx = (double)w / dw;
  const double ry = (double)h / dh;
  for (int y = 0; y < dh; ++y) {
    double sy = (y + 0.5) * ry - 0.5;
    sy = clampd(sy, 0.0, (double)(h - 1));
    const int y0 = (int)sy;
    const int y1 = (y0 + 1 < h - 1) ? y0 + 1 : h - 1;
    const double fy = sy - y0;
    for (int x = 0; x < dw; ++x) {
      double sx = (x + 0.5) * rx - 0.5;
      sx = clampd(sx, 0.0, (double)(w - 1));
      const int x0 = (int)sx;
      const int x1 = (x0 + 1 < w - 1) ? x0 + 1 : w - 1;
      const double fx = sx - x0;
      const double top = px[(size_t)y0 * w + x0] * (1.0 - fx) + px[(size_t)y0 * w + x1] * fx;
      const double bot = px[(size_t)y1 * w + x0] * (1.0 - fx) + px[(size_t)y1 * w + x1] * fx;
      out[(size_t)y * dw + x] = top * (1.0 - fy) + bot * fy;
    }
  }
  return 0;
}

/* image.cpp:158-172.  Levels are written back to back into `out` (if non-NULL and
 * large enough); dims[2k], dims[2k+1] and scales[k] describe level k.  Returns the
 * level count (which may exceed max_levels: only the first max_levels are described). */
int orc_build_pyramid(const double* px, int w, int h, int window, double* out, size_t out_cap,
                      int* dims, double* scales, int max_levels) {
  int n = 0;
  size_t off = 0;
  int cw = w, ch = h;
  const double* cur = px;
  double* tmp_prev = NULL;
  for (;;) {
    if (n < max_levels) {
      dims[2 * n] = cw;
      dims[2 * n + 1] = ch;
      scales[n] = n == 0 ? 1.0 : pow(5.0 / 6.0, (double)n);
    }
    const size_t sz = (size_t)cw * ch;
    if (out && off + sz <= out_cap) memcpy(out + off, cur, sz * sizeof(double));
    off += sz;
    ++n;
    if (cw < 2 || ch < 2) break;
    const int nw = cw * 5 / 6, nh = ch * 5 / 6;
    if (nw < window || nh < window) break;
    double* next = (double*)malloc((size_t)nw * nh * sizeof(double));
    orc_downscale_bilinear(cur, cw, ch, next);
    free(tmp_prev);
    tmp_prev = next;
    cur = next;
    cw = nw;
    ch = nh;
  }
  free(tmp_prev);
  return n;
}

/* -------------------------------------------------------------------- hog ---- */

/* hog.cpp:12-24: the 18 signed directions, from glibc cos/sin. */
void orc_direction_table(double* ux, double* uy) {
  for (int d = 0; d < 18; ++d) {
    const double a = 2.0 * M_PI * d / 18;
    ux[d] = cos(a);
    uy[d] = sin(a);
  }
}

/* hog.cpp:28-56 */
int orc_compute_gradients(const double* px, int w, int h, uint8_t* ori, double* mag) {
  if (w < 3 || h < 3) return fail("compute_gradients: image must be at least 3x3");
  double ux[18], uy[18];
  orc_direction_table(ux, uy);
  memset(ori, 0, (size_t)w * h);
  for (size_t i = 0; i < (size_t)w * h; ++i) mag[i] = 0.0;
  for (int y = 1; y + 1 < h; ++y) {
    for (int x = 1; x + 1 < w; ++x) {
      const double gx = px[(size_t)y * w + x + 1] - px[(size_t)y * w + x - 1];
      const double gy = px[(size_t)(y + 1) * w + x] - px[(size_t)(y - 1) * w + x];
      int best = 0;
      double best_dot = gx * ux[0] + gy * uy[0];
      for (int d = 1; d < 18; ++d) {
        const double dot = gx * ux[d] + gy * uy[d];
        if (dot > best_dot) {
          best_dot = dot;
          best = d;
        }
      }
      ori[(size_t)y * w + x] = (uint8_t)best;
      mag[(size_t)y * w + x] = sqrt(gx * gx + gy * gy);
    }
  }
  return 0;
}

/* hog.cpp:58-90 (scatter in pixel raster order) */
int orc_histogramize(const uint8_t* ori, const double* mag, int w, int h, double* bins) {
  const int cw = w / 8, ch = h / 8;
  for (size_t i = 0; i < (size_t)cw * ch * 18; ++i) bins[i] = 0.0;
  if (cw == 0 || ch == 0) return 0;
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      const double m = mag[(size_t)y * w + x];
      if (m == 0.0) continue;
      const int bin = ori[(size_t)y * w + x];
      const double cxf = (x - 3.5) / 8;
      const double cyf = (y - 3.5) / 8;
      const int cx0 = (int)floor(cxf);
      const int cy0 = (int)floor(cyf);
      const double wx1 = cxf - cx0;
      const double wy1 = cyf - cy0;
      const int cxs[4] = {cx0, cx0 + 1, cx0, cx0 + 1};
      const int cys[4] = {cy0, cy0, cy0 + 1, cy0 + 1};
      double v[4];
      v[0] = m * (1.0 - wx1) * (1.0 - wy1);
      v[1] = m * wx1 * (1.0 - wy1);
      v[2] = m * (1.0 - wx1) * wy1;
      v[3] = m * wx1 * wy1;
      for (int q = 0; q < 4; ++q) {
        if (cxs[q] < 0 || cys[q] < 0 || cxs[q] >= cw || cys[q] >= ch) continue;
        bins[((size_t)cys[q] * cw + cxs[q]) * 18 + bin] += v[q];
      }
    }
  }
  return 0;
}

/* hog.cpp:92-109 */
int orc_cell_energy(const double* bins, int cw, int ch, double* energy) {
  for (size_t c = 0; c < (size_t)cw * ch; ++c) {
    const double* b = bins + c * 18;
    double e = 0.0;
    for (int n = 0; n < 9; ++n) {
      const double s = b[n] + b[n + 9];
      e += s * s;
    }
    energy[c] = e;
  }
  return 0;
}

/* hog.cpp:111-166 */
int orc_compute_features(const double* bins, const double* energy, int cw, int ch, double* feat) {
  const double kEps = 1e-10, kTrunc = 0.2, kTextureScale = 0.2357;
#define E_AT(X, Y) (((X) < 0 || (Y) < 0 || (X) >= cw || (Y) >= ch) ? 0.0 : energy[(size_t)(Y) * cw + (X)])
  for (int cy = 0; cy < ch; ++cy) {
    for (int cx = 0; cx < cw; ++cx) {
      const double* b = bins + ((size_t)cy * cw + cx) * 18;
      double* f = feat + ((size_t)cy * cw + cx) * 31;
      double norm[4];
      int t = 0;
      for (int a = -1; a <= 1; a += 2) {
        for (int bb = -1; bb <= 1; bb += 2) {
          const double e = E_AT(cx, cy) + E_AT(cx + a, cy) + E_AT(cx, cy + bb) + E_AT(cx + a, cy + bb);
          norm[t++] = 1.0 / sqrt(e + kEps);
        }
      }
      double texture[4] = {0.0, 0.0, 0.0, 0.0};
      for (int d = 0; d < 18; ++d) {
        double s = 0.0;
        for (int k = 0; k < 4; ++k) {
          const double hh = mind(b[d] * norm[k], kTrunc);
          s += hh;
          texture[k] += hh;
        }
        f[d] = 0.5 * s;
      }
      for (int u = 0; u < 9; ++u) {
        const double sum = b[u] + b[u + 9];
        double s = 0.0;
        for (int k = 0; k < 4; ++k) s += mind(sum * norm[k], kTrunc);
        f[18 + u] = 0.5 * s;
      }
      for (int k = 0; k < 4; ++k) f[27 + k] = kTextureScale * texture[k];
    }
  }
#undef E_AT
  return 0;
}

/* hog.cpp:168-173 */
int orc_extract_features(const double* px, int w, int h, double* feat) {
  const size_t n = (size_t)w * h;
  uint8_t* ori = (uint8_t*)malloc(n);
  double* mag = (double*)malloc(n * sizeof(double));
  const int cw = w / 8, ch = h / 8;
  double* bins = (double*)malloc(((size_t)cw * ch * 18 + 1) * sizeof(double));
  double* en = (double*)malloc(((size_t)cw * ch + 1) * sizeof(double));
  int rc = orc_compute_gradients(px, w, h, ori, mag);
  if (rc == 0) {
    orc_histogramize(ori, mag, w, h, bins);
    orc_cell_energy(bins, cw, ch, en);
    orc_compute_features(bins, en, cw, ch, feat);
  }
  free(ori);
  free(mag);
  free(bins);
  free(en);
  return rc;
}

/* --------------------------------------------------------------- detector ---- */

/* detector.cpp:16-28 */
double orc_iou(int ax, int ay, int aw, int ah, int bx, int by, int bw, int bh) {
  const long long ix0 = ax > bx ? ax : bx;
  const long long iy0 = ay > by ? ay : by;
  const long long ae = (long long)ax + aw, be = (long long)bx + bw;
  const long long af = (long long)ay + ah, bf = (long long)by + bh;
  const long long ix1 = ae < be ? ae : be;
  const long long iy1 = af < bf ? af : bf;
  const long long iw = ix1 - ix0, ih = iy1 - iy0;
  if (iw <= 0 || ih <= 0) return 0.0;
  const double inter = (double)iw * (double)ih;
  const double uni = (double)aw * ah + (double)bw * bh - inter;
  if (uni <= 0.0) return 0.0;
  return inter / uni;
}

/* detector.cpp:34-39 */
static int check_scorable(int cw, int ch) {
  if (cw < 10 || ch < 10) return fail("feature image smaller than the 10x10 detection window");
  return 0;
}

/* detector.cpp:45-64 */
int orc_score_dense(const double* feat, int cw, int ch, const double* weights, double bias,
                    double* scores) {
  if (check_scorable(cw, ch)) return -1;
  const int sw = cw - 9, sh = ch - 9;
  for (int cy = 0; cy < sh; ++cy) {
    for (int cx = 0; cx < sw; ++cx) {
      double acc = 0.0;
      for (int j = 0; j < 10; ++j) {
        const double* strip = feat + ((size_t)(cy + j) * cw + cx) * 31;
        const double* wr = weights + (size_t)j * 310;
        for (int k = 0; k < 310; ++k) acc += strip[k] * wr[k];
      }
      scores[(size_t)cy * sw + cx] = acc + bias;
    }
  }
  return 0;
}

/* detector.cpp:66-100 */
int orc_score_separable(const double* feat, int cw, int ch, const double* weights, double bias,
                        double* scores) {
  if (check_scorable(cw, ch)) return -1;
  const int aw = cw - 9, sh = ch - 9;
  double* scratch = (double*)malloc((size_t)aw * ch * 10 * sizeof(double));
  for (int y = 0; y < ch; ++y) {
    for (int x = 0; x < aw; ++x) {
      const double* strip = feat + ((size_t)y * cw + x) * 31;
      double* o = scratch + ((size_t)y * aw + x) * 10;
      for (int j = 0; j < 10; ++j) {
        const double* wr = weights + (size_t)j * 310;
        double acc = 0.0;
        for (int k = 0; k < 310; ++k) acc += strip[k] * wr[k];
        o[j] = acc;
      }
    }
  }
  for (int cy = 0; cy < sh; ++cy) {
    for (int cx = 0; cx < aw; ++cx) {
      double acc = 0.0;
      for (int j = 0; j < 10; ++j) acc += scratch[((size_t)(cy + j) * aw + cx) * 10 + j];
      scores[(size_t)cy * aw + cx] = acc + bias;
    }
  }
  free(scratch);
  return 0;
}

/* detector.cpp:41 */
static int round_half_up(double v) { return (int)floor(v + 0.5); }

/* detector.cpp:102-122 */
int orc_threshold_detections(const double* scores, int sw, int sh, double thr, int window_cells,
                             int cell_px, int scale_num, int scale_den, int scale_index,
                             int rotation_index, orc_det* out, int cap) {
  const double c = pow((double)scale_num / scale_den, (double)scale_index);
  const int side = round_half_up((window_cells * cell_px) / c);
  int n = 0;
  for (int cy = 0; cy < sh; ++cy) {
    for (int cx = 0; cx < sw; ++cx) {
      const double s = scores[(size_t)cy * sw + cx];
      if (s > thr) {
        if (n < cap) {
          orc_det d;
          d.x = round_half_up(cx * cell_px / c);
          d.y = round_half_up(cy * cell_px / c);
          d.w = side;
          d.h = side;
          d.score = s;
          d.scale_index = scale_index;
          d.rotation_index = rotation_index;
          out[n] = d;
        }
        ++n;
      }
    }
  }
  return n;
}

/* detector.cpp:125-129: score desc, then (y, x, scale, rotation) asc */
static int det_cmp(const void* pa, const void* pb) {
  const orc_det* a = (const orc_det*)pa;
  const orc_det* b = (const orc_det*)pb;
  if (a->score != b->score) return a->score > b->score ? -1 : 1;
  if (a->y != b->y) return a->y < b->y ? -1 : 1;
  if (a->x != b->x) return a->x < b->x ? -1 : 1;
  if (a->scale_index != b->scale_index) return a->scale_index < b->scale_index ? -1 : 1;
  if (a->rotation_index != b->rotation_index) return a->rotation_index < b->rotation_index ? -1 : 1;
  return 0;
}

/* detector.cpp:124-142 */
int orc_nms(const orc_det* in, int n, double iou_thr, orc_det* out) {
  orc_det* d = (orc_det*)malloc(((size_t)n + 1) * sizeof(orc_det));
  memcpy(d, in, (size_t)n * sizeof(orc_det));
  qsort(d, (size_t)n, sizeof(orc_det), det_cmp);
  int kept = 0;
  for (int i = 0; i < n; ++i) {
    int suppressed = 0;
    for (int k = 0; k < kept; ++k) {
      if (orc_iou(d[i].x, d[i].y, d[i].w, d[i].h, out[k].x, out[k].y, out[k].w, out[k].h) >
          iou_thr) {
        suppressed = 1;
        break;
      }
    }
    if (!suppressed) out[kept++] = d[i];
  }
  free(d);
  return kept;
}

/* detector.cpp:144-155 */
int orc_eligible_scales(int w, int h, int window_cells, int cell_px, int scale_num, int scale_den,
                        double min_face_ratio, int n_levels, int* out) {
  const double min_face = min_face_ratio * (w < h ? w : h);
  int n = 0;
  for (int k = 0; k < n_levels; ++k) {
    const double detectable =
        (window_cells * cell_px) / pow((double)scale_num / scale_den, (double)k);
    if (detectable >= min_face * (1.0 - 1e-9)) out[n++] = k;
  }
  return n;
}

/* detector.cpp:157-176 */
int orc_detect_faces(const double* px, int w, int h, const orc_detector* m, orc_det* out, int cap) {
  const int window = m->window_cells * m->cell_px;
  int dims[128];
  double scales[64];
  const int n_levels = orc_build_pyramid(px, w, h, window, NULL, 0, dims, scales, 64);
  if (n_levels > 64) return fail("pyramid deeper than 64 levels");
  int levels[64];
  const int n_el = orc_eligible_scales(w, h, m->window_cells, m->cell_px, m->scale_num,
                                       m->scale_den, m->min_face_ratio, n_levels, levels);
  /* Re-walk the chain, keeping each level as it is produced. */
  size_t total = 0;
  for (int k = 0; k < n_levels; ++k) total += (size_t)dims[2 * k] * dims[2 * k + 1];
  double* all = (double*)malloc(total * sizeof(double));
  orc_build_pyramid(px, w, h, window, all, total, dims, scales, 64);
  size_t offs[64];
  size_t off = 0;
  for (int k = 0; k < n_levels; ++k) {
    offs[k] = off;
    off += (size_t)dims[2 * k] * dims[2 * k + 1];
  }
  int cap_pool = 1024, n_pool = 0;
  orc_det* pool = (orc_det*)malloc((size_t)cap_pool * sizeof(orc_det));
  for (int e = 0; e < n_el; ++e) {
    const int k = levels[e];
    const int lw = dims[2 * k], lh = dims[2 * k + 1];
    if (lw / m->cell_px < m->window_cells || lh / m->cell_px < m->window_cells) continue;
    const int cw = lw / 8, ch = lh / 8;
    double* feat = (double*)malloc((size_t)cw * ch * 31 * sizeof(double));
    orc_extract_features(all + offs[k], lw, lh, feat);
    const int sw = cw - 9, sh = ch - 9;
    double* sc = (double*)malloc((size_t)sw * sh * sizeof(double));
    for (int r = 0; r < 5; ++r) {
      orc_score_separable(feat, cw, ch, m->weights + (size_t)r * 3100, m->biases[r], sc);
      const int nd = orc_threshold_detections(sc, sw, sh, m->threshold, m->window_cells,
                                              m->cell_px, m->scale_num, m->scale_den, k, r, NULL, 0);
      if (n_pool + nd > cap_pool) {
        while (n_pool + nd > cap_pool) cap_pool *= 2;
        pool = (orc_det*)realloc(pool, (size_t)cap_pool * sizeof(orc_det));
      }
      orc_threshold_detections(sc, sw, sh, m->threshold, m->window_cells, m->cell_px,
                               m->scale_num, m->scale_den, k, r, pool + n_pool, nd);
      n_pool += nd;
    }
    free(sc);
    free(feat);
  }
  orc_det* kept = (orc_det*)malloc(((size_t)n_pool + 1) * sizeof(orc_det));
  const int nk = orc_nms(pool, n_pool, 0.5, kept);
  for (int i = 0; i < nk && i < cap; ++i) out[i] = kept[i];
  free(kept);
  free(pool);
  free(all);
  return nk;
}

/* -------------------------------------------------------------------- ert ---- */

/* ert.cpp:26-69 ; out4 = (scale, rotation, tx, ty) */
int orc_similarity_transform(const double* from, const double* to, int L, double* out4) {
  if (L < 2) return fail("similarity_transform: shapes must share L >= 2 points");
  double mfx = 0, mfy = 0, mtx = 0, mty = 0;
  for (int i = 0; i < L; ++i) {
    mfx += from[2 * i];
    mfy += from[2 * i + 1];
    mtx += to[2 * i];
    mty += to[2 * i + 1];
  }
  mfx /= (double)L;
  mfy /= (double)L;
  mtx /= (double)L;
  mty /= (double)L;
  double sff = 0.0, sre = 0.0, sim = 0.0;
  for (int i = 0; i < L; ++i) {
    const double fx = from[2 * i] - mfx;
    const double fy = from[2 * i + 1] - mfy;
    const double txp = to[2 * i] - mtx;
    const double typ = to[2 * i + 1] - mty;
    sff += fx * fx + fy * fy;
    sre += fx * txp + fy * typ;
    sim += fx * typ - fy * txp;
  }
  if (sff <= 0.0) return fail("similarity_transform: source shape has no spread");
  const double a = sre / sff, b = sim / sff;
  const double scale = hypot(a, b);
  if (scale <= 0.0) return fail("similarity_transform: target shape has no spread");
  out4[0] = scale;
  out4[1] = atan2(b, a);
  out4[2] = mtx - (a * mfx - b * mfy);
  out4[3] = mty - (b * mfx + a * mfy);
  return 0;
}

/* ert.cpp:20-24 + 71-85 */
double orc_sample_intensity(const double* px, int w, int h, int bx, int by, int bw, int bh,
                            const double* shape_xy, const double* tform4, int anchor, double ox,
                            double oy) {
  const double a = tform4[0] * cos(tform4[1]);
  const double b = tform4[0] * sin(tform4[1]);
  const double offx = a * ox - b * oy;
  const double offy = b * ox + a * oy;
  const double nx = shape_xy[2 * anchor] + offx;
  const double ny = shape_xy[2 * anchor + 1] + offy;
  const double pxx = bx + nx * bw;
  const double pyy = by + ny * bh;
  int ix = (int)llround(pxx);
  int iy = (int)llround(pyy);
  ix = clampi(ix, 0, w - 1);
  iy = clampi(iy, 0, h - 1);
  return px[(size_t)iy * w + ix];
}

/* ert.cpp:99-136 (traverse_tree ert.cpp:87-97 inlined).  leaf_idx (optional) receives
 * T*K leaf indices in cascade order. */
int orc_predict_landmarks(const double* px, int w, int h, int bx, int by, int bw, int bh,
                          const orc_ert* m, double* out_xy, uint8_t* leaf_idx, uint64_t* evals) {
  if (bw <= 0 || bh <= 0) return fail("predict_landmarks: face box must have positive area");
  const int L = m->L;
  if (L < 2) return fail("predict_landmarks: model has no mean shape");
  const int S = (1 << m->F) - 1, NL = 1 << m->F;
  double* cur = (double*)malloc((size_t)L * 2 * sizeof(double));
  double* delta = (double*)malloc((size_t)L * 2 * sizeof(double));
  memcpy(cur, m->mean_xy, (size_t)L * 2 * sizeof(double));
  uint64_t ev = 0;
  size_t q = 0;
  for (int t = 0; t < m->T; ++t) {
    double tf[4];
    if (orc_similarity_transform(cur, m->mean_xy, L, tf)) {
      free(cur);
      free(delta);
      return -1;
    }
    for (int i = 0; i < 2 * L; ++i) delta[i] = 0.0;
    for (int k = 0; k < m->K; ++k) {
      const size_t tk = (size_t)t * m->K + k;
      int node = 0;
      while (node < S) {
        const int32_t* an = m->anchors + (tk * S + node) * 2;
        const double* sp = m->split_params + (tk * S + node) * 5;
        ++ev;
        const double ia = orc_sample_intensity(px, w, h, bx, by, bw, bh, cur, tf, an[0], sp[0], sp[1]);
        const double ib = orc_sample_intensity(px, w, h, bx, by, bw, bh, cur, tf, an[1], sp[2], sp[3]);
        node = (ia - ib > sp[4]) ? 2 * node + 1 : 2 * node + 2;
      }
      const int leaf = node - S;
      if (leaf_idx) leaf_idx[q++] = (uint8_t)leaf;
      const double* lv = m->leaves + (tk * NL + leaf) * (size_t)L * 2;
      for (int i = 0; i < L; ++i) {
        delta[2 * i] += lv[2 * i];
        delta[2 * i + 1] += lv[2 * i + 1];
      }
    }
    for (int i = 0; i < L; ++i) {
      cur[2 * i] += m->shrinkage * delta[2 * i];
      cur[2 * i + 1] += m->shrinkage * delta[2 * i + 1];
    }
  }
  for (int i = 0; i < L; ++i) {
    out_xy[2 * i] = bx + cur[2 * i] * bw;
    out_xy[2 * i + 1] = by + cur[2 * i + 1] * bh;
  }
  if (evals) *evals = ev;
  free(cur);
  free(delta);
  return 0;
}
