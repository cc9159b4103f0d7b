// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// A thin extern "C" face over the UNMODIFIED reference library
// (/root/reference/proj/src/{image,hog,detector,ert}.cpp + tests/helpers.cpp),
// compiled by oracle/Makefile into oracle/_ref/libblinkline_ref.so.  Nothing
// in this file re-implements the algorithm: every entry point converts plain
// arrays into the reference's value types, calls the reference's public API
// and converts the result back.  It exists so that Python tests (ctypes) and
// bench.py's CPU-baseline leg can drive the reference without linking its
// C++ symbols next to the product's own `blinkline::` drop-in symbols.
//
// The one restatement here is `ref_ert_leaf_indices`: the reference API does
// not expose leaf indices, so it re-runs predict_landmarks' loop
// (ert.cpp:99-136) on the PUBLIC similarity_transform / sample_intensity /
// traverse_tree functions (ert.hpp:42,72-78) and records
// `&leaf - &tree.leaves[0]`.  tests/test_oracle_golden.py checks it against
// predict_landmarks bit-for-bit.

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "blinkline/blink.hpp"
#include "blinkline/detector.hpp"
#include "blinkline/pipeline.hpp"
#include "blinkline/errors.hpp"
#include "blinkline/ert.hpp"
#include "blinkline/hog.hpp"
#include "blinkline/image.hpp"
#include "helpers.hpp"

using namespace blinkline;

namespace {

thread_local std::string g_err;

GrayImage to_image(const double* px, int w, int h) {
  GrayImage img = make_image(w, h);
  std::memcpy(img.pixels.data(), px, sizeof(double) * std::size_t(w) * h);
  return img;
}

DetectorModel to_model(const double* weights, const double* biases, double thr, int window_cells,
                       int cell_px, int scale_num, int scale_den, double min_face_ratio) {
  DetectorModel m;
  for (int r = 0; r < 5; ++r) {
    m.filters[r].weights.assign(weights + std::size_t(r) * kFilterWeights,
                                weights + std::size_t(r + 1) * kFilterWeights);
    m.filters[r].bias = biases[r];
  }
  m.detection_threshold = thr;
  m.window_cells = window_cells;
  m.cell_px = cell_px;
  m.scale_num = scale_num;
  m.scale_den = scale_den;
  m.min_face_ratio = min_face_ratio;
  return m;
}

struct RefDet {  // same layout as blinkline::Detection and bl_detection
  int32_t x, y, w, h;
  double score;
  int32_t scale_index, rotation_index;
};
static_assert(sizeof(RefDet) == sizeof(Detection), "layout");

RefDet to_ref(const Detection& d) {
  return RefDet{d.box.x, d.box.y, d.box.w, d.box.h, d.score, d.scale_index, d.rotation_index};
}

void put_dets(const std::vector<Detection>& d, RefDet* out, int cap) {
  for (int i = 0; i < int(d.size()) && i < cap; ++i) {
    out[i] = RefDet{d[i].box.x, d[i].box.y, d[i].box.w, d[i].box.h, d[i].score,
                    d[i].scale_index, d[i].rotation_index};
  }
}

std::vector<Detection> get_dets(const RefDet* in, int n) {
  std::vector<Detection> d(n);
  for (int i = 0; i < n; ++i) {
    d[i].box = Box{in[i].x, in[i].y, in[i].w, in[i].h};
    d[i].score = in[i].score;
    d[i].scale_index = in[i].scale_index;
    d[i].rotation_index = in[i].rotation_index;
  }
  return d;
}

Shape to_shape(const double* xy, int L) {
  Shape s;
  s.frame = ShapeFrame::normalized;
  s.points.resize(L);
  for (int i = 0; i < L; ++i) s.points[i] = {xy[2 * i], xy[2 * i + 1]};
  return s;
}

}  // namespace

#define REF_TRY try {
#define REF_CATCH                    \
  }                                  \
  catch (const std::exception& e) {  \
    g_err = e.what();                \
    return -1;                       \
  }

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- image ----
int ref_build_pyramid(const double* px, int w, int h, int window, double* out, int out_cap,
                      int* dims, double* scales, int max_levels) {
  REF_TRY
  const Pyramid p = build_pyramid(to_image(px, w, h), window);
  const int n = int(p.levels.size());
  std::size_t off = 0;
  for (int k = 0; k < n && k < max_levels; ++k) {
    dims[2 * k] = p.levels[k].width;
    dims[2 * k + 1] = p.levels[k].height;
    scales[k] = p.cumulative_scale[k];
    const std::size_t sz = p.levels[k].pixels.size();
    if (out && off + sz <= std::size_t(out_cap))
      std::memcpy(out + off, p.levels[k].pixels.data(), sz * sizeof(double));
    off += sz;
  }
  return n;
  REF_CATCH
}

int ref_downscale_bilinear(const double* px, int w, int h, double* out) {
  REF_TRY
  const GrayImage o = downscale_bilinear(to_image(px, w, h));
  std::memcpy(out, o.pixels.data(), o.pixels.size() * sizeof(double));
  return 0;
  REF_CATCH
}

// ------------------------------------------------------------------ hog ----
int ref_compute_gradients(const double* px, int w, int h, uint8_t* ori, double* mag) {
  REF_TRY
  const GradientField g = compute_gradients(to_image(px, w, h));
  std::memcpy(ori, g.orientation.data(), g.orientation.size());
  std::memcpy(mag, g.magnitude.data(), g.magnitude.size() * sizeof(double));
  return 0;
  REF_CATCH
}

int ref_histogramize(const uint8_t* ori, const double* mag, int w, int h, double* bins) {
  REF_TRY
  GradientField g;
  g.width = w;
  g.height = h;
  g.orientation.assign(ori, ori + std::size_t(w) * h);
  g.magnitude.assign(mag, mag + std::size_t(w) * h);
  const CellGrid c = histogramize(g);
  std::memcpy(bins, c.bins.data(), c.bins.size() * sizeof(double));
  return 0;
  REF_CATCH
}

int ref_cell_energy(const double* bins, int cw, int ch, double* energy) {
  REF_TRY
  CellGrid c;
  c.cells_w = cw;
  c.cells_h = ch;
  c.bins.assign(bins, bins + std::size_t(cw) * ch * kOrientationBins);
  const EnergyGrid e = cell_energy(c);
  std::memcpy(energy, e.energy.data(), e.energy.size() * sizeof(double));
  return 0;
  REF_CATCH
}

int ref_compute_features(const double* bins, const double* energy, int cw, int ch, double* feat) {
  REF_TRY
  CellGrid c;
  c.cells_w = cw;
  c.cells_h = ch;
  c.bins.assign(bins, bins + std::size_t(cw) * ch * kOrientationBins);
  EnergyGrid e;
  e.cells_w = cw;
  e.cells_h = ch;
  e.energy.assign(energy, energy + std::size_t(cw) * ch);
  const FeatureImage f = compute_features(c, e);
  std::memcpy(feat, f.values.data(), f.values.size() * sizeof(double));
  return 0;
  REF_CATCH
}

int ref_extract_features(const double* px, int w, int h, double* feat) {
  REF_TRY
  const FeatureImage f = extract_features(to_image(px, w, h));
  std::memcpy(feat, f.values.data(), f.values.size() * sizeof(double));
  return 0;
  REF_CATCH
}

// ------------------------------------------------------------- detector ----
static int score_common(bool dense, const double* feat, int cw, int ch, const double* weights,
                        double bias, double* scores) {
  FeatureImage f;
  f.cells_w = cw;
  f.cells_h = ch;
  f.values.assign(feat, feat + std::size_t(cw) * ch * kCellFeatures);
  LinearFilter lf;
  lf.weights.assign(weights, weights + kFilterWeights);
  lf.bias = bias;
  const SaliencyMap s = dense ? score_dense(f, lf) : score_separable(f, lf);
  std::memcpy(scores, s.scores.data(), s.scores.size() * sizeof(double));
  return 0;
}

int ref_score_dense(const double* feat, int cw, int ch, const double* weights, double bias,
                    double* scores) {
  REF_TRY
  return score_common(true, feat, cw, ch, weights, bias, scores);
  REF_CATCH
}

int ref_score_separable(const double* feat, int cw, int ch, const double* weights, double bias,
                        double* scores) {
  REF_TRY
  return score_common(false, feat, cw, ch, weights, bias, scores);
  REF_CATCH
}

int ref_threshold_detections(const double* scores, int sw, int sh, double thr, int window_cells,
                             int cell_px, int scale_num, int scale_den, int scale_index,
                             int rotation_index, RefDet* out, int cap) {
  REF_TRY
  DetectorModel m;
  m.detection_threshold = thr;
  m.window_cells = window_cells;
  m.cell_px = cell_px;
  m.scale_num = scale_num;
  m.scale_den = scale_den;
  SaliencyMap s;
  s.width = sw;
  s.height = sh;
  s.scores.assign(scores, scores + std::size_t(sw) * sh);
  const auto d = threshold_detections(s, m, scale_index, rotation_index);
  put_dets(d, out, cap);
  return int(d.size());
  REF_CATCH
}

int ref_nms(const RefDet* in, int n, double iou_thr, RefDet* out) {
  REF_TRY
  const auto k = nms(get_dets(in, n), iou_thr);
  put_dets(k, out, n);
  return int(k.size());
  REF_CATCH
}

double ref_iou(int ax, int ay, int aw, int ah, int bx, int by, int bw, int bh) {
  return iou(Box{ax, ay, aw, ah}, Box{bx, by, bw, bh});
}

int ref_eligible_scales(int w, int h, int window_cells, int cell_px, int scale_num, int scale_den,
                        double min_face_ratio, int n_levels, int* out) {
  REF_TRY
  DetectorModel m;
  m.window_cells = window_cells;
  m.cell_px = cell_px;
  m.scale_num = scale_num;
  m.scale_den = scale_den;
  m.min_face_ratio = min_face_ratio;
  const auto e = eligible_scales(w, h, m, n_levels);
  for (std::size_t i = 0; i < e.size(); ++i) out[i] = e[i];
  return int(e.size());
  REF_CATCH
}

int ref_detect_faces(const double* px, int w, int h, const double* weights, const double* biases,
                     double thr, int window_cells, int cell_px, int scale_num, int scale_den,
                     double min_face_ratio, RefDet* out, int cap) {
  REF_TRY
  const DetectorModel m =
      to_model(weights, biases, thr, window_cells, cell_px, scale_num, scale_den, min_face_ratio);
  const auto d = detect_faces(to_image(px, w, h), m);
  put_dets(d, out, cap);
  return int(d.size());
  REF_CATCH
}

// ------------------------------------------------------------------ ert ----
struct RefErt {
  ErtModel model;
};

void* ref_ert_create(int L, int T, int K, int F, double shrinkage, const double* mean_xy,
                     const int32_t* anchors, const double* split_params, const double* leaves) {
  try {
    auto* r = new RefErt;
    r->model.shrinkage = shrinkage;
    r->model.mean_shape = to_shape(mean_xy, L);
    const int S = (1 << F) - 1, NL = 1 << F;
    for (int t = 0; t < T; ++t) {
      std::vector<RegressionTree> level;
      for (int k = 0; k < K; ++k) {
        RegressionTree tree;
        tree.depth = F;
        const std::size_t tk = std::size_t(t) * K + k;
        for (int s = 0; s < S; ++s) {
          const int32_t* a = anchors + (tk * S + s) * 2;
          const double* p = split_params + (tk * S + s) * 5;
          SplitNode n;
          n.anchor_a = a[0];
          n.anchor_b = a[1];
          n.offset_a = {p[0], p[1]};
          n.offset_b = {p[2], p[3]};
          n.threshold = p[4];
          tree.splits.push_back(n);
        }
        for (int l = 0; l < NL; ++l) {
          const double* lv = leaves + (tk * NL + l) * std::size_t(L) * 2;
          std::vector<Point2> pts(L);
          for (int i = 0; i < L; ++i) pts[i] = {lv[2 * i], lv[2 * i + 1]};
          tree.leaves.push_back(std::move(pts));
        }
        level.push_back(std::move(tree));
      }
      r->model.cascade.push_back(std::move(level));
    }
    return r;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_ert_destroy(void* h) { delete static_cast<RefErt*>(h); }

int ref_predict_landmarks(const double* px, int w, int h, int bx, int by, int bw, int bh,
                          const void* ert, double* out_xy, uint64_t* evals) {
  REF_TRY
  PredictStats st;
  const Shape s = predict_landmarks(to_image(px, w, h), Box{bx, by, bw, bh},
                                    static_cast<const RefErt*>(ert)->model, &st);
  for (std::size_t i = 0; i < s.points.size(); ++i) {
    out_xy[2 * i] = s.points[i].x;
    out_xy[2 * i + 1] = s.points[i].y;
  }
  if (evals) *evals = st.intensity_diffs;
  return 0;
  REF_CATCH
}

// Instrumented restatement of predict_landmarks on the public API, recording
// leaf indices (ert.cpp:99-136 loop shape; leaf index = &leaf - &leaves[0]).
int ref_ert_leaf_indices(const double* px, int w, int h, int bx, int by, int bw, int bh,
                         const void* ert, uint8_t* leaf_idx, double* out_xy) {
  REF_TRY
  const ErtModel& model = static_cast<const RefErt*>(ert)->model;
  const GrayImage img = to_image(px, w, h);
  const Box box{bx, by, bw, bh};
  const int L = model.landmark_count();
  Shape current = model.mean_shape;
  std::size_t q = 0;
  for (const auto& level : model.cascade) {
    const SimilarityTransform tform = similarity_transform(current, model.mean_shape);
    std::vector<Point2> delta(L, Point2{0, 0});
    for (const RegressionTree& tree : level) {
      const std::vector<Point2>& leaf =
          traverse_tree(tree, [&](const SplitNode& s) -> std::pair<double, double> {
            return {sample_intensity(img, box, current, tform, s.anchor_a, s.offset_a),
                    sample_intensity(img, box, current, tform, s.anchor_b, s.offset_b)};
          });
      leaf_idx[q++] = uint8_t(&leaf - &tree.leaves[0]);
      for (int i = 0; i < L; ++i) {
        delta[i].x += leaf[i].x;
        delta[i].y += leaf[i].y;
      }
    }
    for (int i = 0; i < L; ++i) {
      current.points[i].x += model.shrinkage * delta[i].x;
      current.points[i].y += model.shrinkage * delta[i].y;
    }
  }
  for (int i = 0; i < L; ++i) {
    out_xy[2 * i] = box.x + current.points[i].x * box.w;
    out_xy[2 * i + 1] = box.y + current.points[i].y * box.h;
  }
  return 0;
  REF_CATCH
}

int ref_similarity_transform(const double* from_xy, const double* to_xy, int L, double* out4) {
  REF_TRY
  const SimilarityTransform t = similarity_transform(to_shape(from_xy, L), to_shape(to_xy, L));
  out4[0] = t.scale;
  out4[1] = t.rotation;
  out4[2] = t.tx;
  out4[3] = t.ty;
  return 0;
  REF_CATCH
}

double ref_sample_intensity(const double* px, int w, int h, int bx, int by, int bw, int bh,
                            const double* shape_xy, int L, const double* tform4, int anchor,
                            double ox, double oy) {
  SimilarityTransform t;
  t.scale = tform4[0];
  t.rotation = tform4[1];
  t.tx = tform4[2];
  t.ty = tform4[3];
  return sample_intensity(to_image(px, w, h), Box{bx, by, bw, bh}, to_shape(shape_xy, L), t,
                          anchor, Point2{ox, oy});
}

// ------------------------------------------------------------- fixtures ----
// The reference's own seeded generators (tests/helpers.cpp), exposed so the
// golden fixtures are built from exactly the inputs the reference tests use.
int ref_pattern_detector(double* weights3100, double* bias, double* thr) {
  REF_TRY
  const DetectorModel& m = testutil::pattern_detector();
  std::memcpy(weights3100, m.filters[0].weights.data(), sizeof(double) * kFilterWeights);
  *bias = m.filters[0].bias;
  *thr = m.detection_threshold;
  return 0;
  REF_CATCH
}

void ref_face68_mean_shape(double* xy) {
  const Shape s = testutil::face68_mean_shape();
  for (int i = 0; i < 68; ++i) {
    xy[2 * i] = s.points[i].x;
    xy[2 * i + 1] = s.points[i].y;
  }
}

void ref_random_image(int w, int h, uint64_t seed, double lo, double hi, double* out) {
  std::mt19937_64 rng(seed);
  const GrayImage img = testutil::random_image(w, h, rng, lo, hi);
  std::memcpy(out, img.pixels.data(), img.pixels.size() * sizeof(double));
}

// make_image(w,h,20) + add_noise(mt19937_64(seed), 1.5) + draw_pattern(cx,cy,size),
// then rounded exactly as save_pgm/load_pgm would round-trip it
// (helpers.cpp:203-216, image.cpp:116-127).
void ref_ring_frame(int w, int h, uint64_t seed, double cx, double cy, double size, int round_u8,
                    double* out) {
  GrayImage img = make_image(w, h, 20.0);
  std::mt19937_64 rng(seed);
  testutil::add_noise(img, rng, 1.5);
  if (size > 0) testutil::draw_pattern(img, cx, cy, size);
  for (std::size_t i = 0; i < img.pixels.size(); ++i) {
    double v = img.pixels[i];
    if (round_u8) v = double(std::llround(std::clamp(v, 0.0, 255.0)));
    out[i] = v;
  }
}

// --------------------------------------------------------- CPU baseline ----
// detect_faces on every frame, then predict_landmarks on every kept
// detection -- the reference pipeline's detect_frame/landmark_frame work
// (pipeline.cpp:159-190) without PGM decode -- frame-parallel over `threads`
// std::threads as the reference's own pipelined runtime does.  Returns the
// total number of landmarked faces; per-frame counts and an order-independent
// checksum of all landmark coordinates go to the out-params.
long long ref_run_batch_u8(const uint8_t* frames, int n, int w, int h, const double* weights,
                           const double* biases, double thr, const void* ert, int threads,
                           int* counts, double* checksum) {
  try {
    const DetectorModel m = to_model(weights, biases, thr, 10, 8, 5, 6, 0.2);
    const ErtModel* em = ert ? &static_cast<const RefErt*>(ert)->model : nullptr;
    std::atomic<int> next{0};
    std::vector<double> sums(std::max(1, threads), 0.0);
    std::atomic<long long> faces{0};
    auto work = [&](int tid) {
      GrayImage img = make_image(w, h);
      for (int f = next++; f < n; f = next++) {
        const uint8_t* src = frames + std::size_t(f) * w * h;
        for (std::size_t i = 0; i < img.pixels.size(); ++i) img.pixels[i] = src[i];
        const auto dets = detect_faces(img, m);
        counts[f] = int(dets.size());
        if (em) {
          for (const Detection& d : dets) {
            const Shape s = predict_landmarks(img, d.box, *em);
            for (const Point2& p : s.points) sums[tid] += p.x + p.y;
          }
          faces += (long long)dets.size();
        }
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(work, t);
    for (auto& t : pool) t.join();
    double s = 0;
    for (double v : sums) s += v;
    if (checksum) *checksum = s;
    return faces.load();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ERT-only batch (config C4): boxes over frames, box-parallel.
int ref_landmarks_batch_u8(const uint8_t* frames, int w, int h, const int32_t* frame_of_box,
                           const int32_t* boxes, int n_boxes, const void* ert, int threads,
                           double* out_xy) {
  try {
    const ErtModel& em = static_cast<const RefErt*>(ert)->model;
    const int L = em.landmark_count();
    std::atomic<int> next{0};
    auto work = [&]() {
      GrayImage img = make_image(w, h);
      int loaded = -1;
      for (int b = next++; b < n_boxes; b = next++) {
        const int f = frame_of_box[b];
        if (f != loaded) {
          const uint8_t* src = frames + std::size_t(f) * w * h;
          for (std::size_t i = 0; i < img.pixels.size(); ++i) img.pixels[i] = src[i];
          loaded = f;
        }
        const Box box{boxes[4 * b], boxes[4 * b + 1], boxes[4 * b + 2], boxes[4 * b + 3]};
        const Shape s = predict_landmarks(img, box, em);
        if (out_xy)
          for (int i = 0; i < L; ++i) {
            out_xy[(std::size_t(b) * L + i) * 2] = s.points[i].x;
            out_xy[(std::size_t(b) * L + i) * 2 + 1] = s.points[i].y;
          }
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(work);
    for (auto& t : pool) t.join();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ------------------------------------------------------ file formats (reference I/O) ----
// 0 ok, 1 io_error, 2 model_error, 3 invalid_argument / other; message via ref_last_error.
static int io_catch(const std::exception_ptr& ep) {
  try {
    std::rethrow_exception(ep);
  } catch (const io_error& e) {
    g_err = e.what();
    return 1;
  } catch (const model_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

int ref_load_pgm(const char* path, int* w, int* h, double* px, long long cap) {
  try {
    const GrayImage img = load_pgm(path);
    *w = img.width;
    *h = img.height;
    if (px && cap >= (long long)img.pixels.size()) std::memcpy(px, img.pixels.data(), sizeof(double) * img.pixels.size());
    return 0;
  } catch (...) {
    return io_catch(std::current_exception());
  }
}

int ref_save_pgm(const char* path, const double* px, int w, int h) {
  try {
    save_pgm(to_image(px, w, h), path);
    return 0;
  } catch (...) {
    return io_catch(std::current_exception());
  }
}

int ref_save_detector_json(const char* path, const double* weights, const double* biases, double thr,
                           int window_cells, int cell_px, int scale_num, int scale_den, double min_face_ratio) {
  try {
    save_model(to_model(weights, biases, thr, window_cells, cell_px, scale_num, scale_den, min_face_ratio), path);
    return 0;
  } catch (...) {
    return io_catch(std::current_exception());
  }
}

int ref_load_detector_json(const char* path, double* weights, double* biases, double* thr, int* window_cells,
                           int* cell_px, int* scale_num, int* scale_den, double* min_face_ratio) {
  try {
    const DetectorModel m = load_detector_model(path);
    for (int r = 0; r < 5; ++r) {
      if (weights) std::memcpy(weights + r * m.filters[r].weights.size(), m.filters[r].weights.data(),
                               sizeof(double) * m.filters[r].weights.size());
      biases[r] = m.filters[r].bias;
    }
    *thr = m.detection_threshold;
    *window_cells = m.window_cells;
    *cell_px = m.cell_px;
    *scale_num = m.scale_num;
    *scale_den = m.scale_den;
    *min_face_ratio = m.min_face_ratio;
    return 0;
  } catch (...) {
    return io_catch(std::current_exception());
  }
}

int ref_ert_save_json(void* h, const char* path) {
  try {
    save_model(static_cast<RefErt*>(h)->model, path);
    return 0;
  } catch (...) {
    return io_catch(std::current_exception());
  }
}

// Loads an ert-v1 file with the reference and exports it in the bl_ert_upload layout.
// dims[5] = L, T, K, F (and shrinkage in *shrink); arrays may be NULL for a dims-only call.
int ref_ert_load_json(const char* path, int* dims, double* shrink, double* mean_xy, int32_t* anchors,
                      double* split_params, double* leaves) {
  try {
    const ErtModel m = load_ert_model(path);
    const int L = m.landmark_count(), T = m.levels(), K = m.trees_per_level();
    const int F = (T > 0 && K > 0) ? m.cascade[0][0].depth : 0;
    dims[0] = L;
    dims[1] = T;
    dims[2] = K;
    dims[3] = F;
    *shrink = m.shrinkage;
    if (mean_xy)
      for (int i = 0; i < L; ++i) {
        mean_xy[2 * i] = m.mean_shape.points[i].x;
        mean_xy[2 * i + 1] = m.mean_shape.points[i].y;
      }
    std::size_t si = 0, li = 0;
    for (const auto& level : m.cascade)
      for (const RegressionTree& tree : level) {
        for (const SplitNode& n : tree.splits) {
          if (anchors) {
            anchors[2 * si] = n.anchor_a;
            anchors[2 * si + 1] = n.anchor_b;
          }
          if (split_params) {
            double* q = split_params + 5 * si;
            q[0] = n.offset_a.x;
            q[1] = n.offset_a.y;
            q[2] = n.offset_b.x;
            q[3] = n.offset_b.y;
            q[4] = n.threshold;
          }
          ++si;
        }
        for (const auto& leaf : tree.leaves) {
          if (leaves)
            for (std::size_t i = 0; i < leaf.size(); ++i) {
              leaves[2 * (li + i)] = leaf[i].x;
              leaves[2 * (li + i) + 1] = leaf[i].y;
            }
          li += leaf.size();
        }
      }
    return 0;
  } catch (...) {
    return io_catch(std::current_exception());
  }
}

// ------------------------------------------------------------- run (pipeline.cpp) ----
// The reference's run() over a frame directory: per frame n_dets, face (RefDet, found flag),
// landmarks [L][2], the trace sample's ear/closure values; all detections in frame order.
int ref_run(const char* dir, const double* weights, const double* biases, double thr, void* ert, double fps,
            int pipelined, int batch_size, int* n_frames, int* n_dets, int* face_found, RefDet* faces,
            double* landmarks, double* ears4, RefDet* dets, int det_cap, int* det_total, double* baselines) {
  try {
    const DetectorModel hog = to_model(weights, biases, thr, 10, 8, 5, 6, 0.2);
    PipelineConfig cfg;
    cfg.mode = pipelined ? ExecMode::pipelined : ExecMode::sequential;
    cfg.batch_size = std::size_t(batch_size);
    cfg.detect_workers = pipelined ? 2 : 1;
    cfg.landmark_workers = pipelined ? 2 : 1;
    if (pipelined >= 2) {  // `pipelined` = total worker threads (the CPU-baseline timing uses all cores)
      cfg.detect_workers = std::max(1, (2 * pipelined) / 3);
      cfg.landmark_workers = std::max(1, pipelined - cfg.detect_workers);
    }
    const RunOutput out = run(dir, hog, static_cast<RefErt*>(ert)->model, fps, cfg);
    const int n = int(out.results.size());
    *n_frames = n;
    int tot = 0;
    for (int i = 0; i < n; ++i) {
      const FrameResult& fr = out.results[i];
      n_dets[i] = int(fr.detections.size());
      face_found[i] = fr.face.has_value();
      if (fr.face) faces[i] = to_ref(*fr.face);
      if (fr.landmarks)
        for (std::size_t k = 0; k < fr.landmarks->points.size(); ++k) {
          landmarks[(std::size_t(i) * fr.landmarks->points.size() + k) * 2] = fr.landmarks->points[k].x;
          landmarks[(std::size_t(i) * fr.landmarks->points.size() + k) * 2 + 1] = fr.landmarks->points[k].y;
        }
      const BlinkSample& s = out.trace.samples[i];
      ears4[4 * i] = s.ear_left.value_or(NAN);
      ears4[4 * i + 1] = s.ear_right.value_or(NAN);
      ears4[4 * i + 2] = s.closure_left.value_or(NAN);
      ears4[4 * i + 3] = s.closure_right.value_or(NAN);
      for (const Detection& d : fr.detections)
        if (tot < det_cap) dets[tot++] = to_ref(d);
    }
    *det_total = tot;
    baselines[0] = out.trace.baseline_left;
    baselines[1] = out.trace.baseline_right;
    return 0;
  } catch (...) {
    return io_catch(std::current_exception());
  }
}

}  // extern "C"
