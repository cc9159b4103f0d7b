// blinkline drop-in API (blinkline_gpu.hpp) implemented over the C-ABI.
//
// Hot-path functions (build_pyramid, downscale_bilinear, the HOG stages, score_*,
// nms, detect_faces, predict_landmarks and the batch extensions) run on the GPU through
// include/blinkline_b200.h.  The remaining entry points are O(1)/O(n) scalar helpers of
// the API (iou, eligible_scales, threshold_detections, similarity_transform,
// sample_intensity, traverse_tree, SimilarityTransform::apply*) and are evaluated here
// with the reference's arithmetic (file:line cited per function); they are not a fallback
// for any device stage.
#include "blinkline_gpu.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <chrono>
#include <cstdio>
#include <filesystem>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>

#include "blinkline_b200.h"

namespace blinkline {
namespace {

// Map a C-ABI status to the reference's exception types.
void check(int rc) {
  if (rc == BL_OK) return;
  const std::string msg = bl_last_error();
  if (rc == BL_ERR_INVALID) throw std::invalid_argument(msg);
  if (rc == BL_ERR_MODEL) throw model_error(msg);
  if (rc == BL_ERR_IO) throw io_error(msg);
  throw std::runtime_error("blinkline_b200: " + msg);
}

// --- models on the device ---------------------------------------------------------------
// Every thread has its own context (the reference calls these functions concurrently from its
// pipeline workers, pipeline.cpp:278-311), but a model lives on each device ONCE: a
// process-wide registry per device holds the last uploaded detector and ERT model in an owner
// context, and thread contexts share them (bl_ctx_share_models) instead of uploading copies.
//
// Which model a call means is decided by its content key, not its address:
//  * detector: every weight, bias, the threshold and the geometry (124 KB, compared exactly);
//  * ERT: the structure (L, T, K, F, shrinkage, every tree's depth and vector sizes), the mean
//    shape, a full 64-bit hash of every split record (the anchors, offsets and thresholds
//    that decide each leaf) and of every leaf row's address, plus a strided sample of leaf
//    values.  Reallocation, reassignment, another model at the same address or any split
//    edit is seen on the next call; only a leaf VALUE edited in place within its existing
//    buffer can slip past the sample -- call gpu::invalidate_model_cache() after such an edit
//    (hashing all 130 MB of leaves per call would cost ~20 ms, 100x the device time).
struct DetKey {
  std::vector<double> w;
  std::array<double, 5> b{};
  double thr = 0, ratio = 0;
  int geom[4] = {0, 0, 0, 0};
  bool operator==(const DetKey& o) const {
    return w == o.w && b == o.b && thr == o.thr && ratio == o.ratio && std::memcmp(geom, o.geom, sizeof geom) == 0;
  }
};

struct ErtKey {
  std::vector<double> head;  // L, T, K, F, shrinkage, mean shape, sampled leaf values
  uint64_t split_hash = 0, layout_hash = 0;
  bool operator==(const ErtKey& o) const {
    return split_hash == o.split_hash && layout_hash == o.layout_hash && head == o.head;
  }
};

struct DeviceModels {
  std::mutex mu;
  bl_ctx* det_owner = nullptr;  // never destroyed: process-lifetime, like the device itself
  bl_ctx* ert_owner = nullptr;
  DetKey det_key;
  ErtKey ert_key;
  bool det_valid = false, ert_valid = false;
  uint64_t generation = 0;  // bumped by gpu::invalidate_model_cache()
};

DeviceModels& registry(int device) {
  static DeviceModels r[64];
  if (device < 0 || device >= 64) throw std::invalid_argument("device index out of range");
  return r[device];
}

int default_device() {
  const char* e = std::getenv("BLINKLINE_DEVICE");
  return e ? std::atoi(e) : 0;
}

struct ThreadCtx {
  int device = default_device();
  bl_ctx* ctx = nullptr;
  DetKey det_key;
  ErtKey ert_key;
  bool det_valid = false, ert_valid = false;
  uint64_t generation = 0;
  ~ThreadCtx() {
    if (ctx) bl_ctx_destroy(ctx);
  }
  bl_ctx* get() {
    if (!ctx) check(bl_ctx_create(device, &ctx));
    return ctx;
  }
};

ThreadCtx& tls() {
  thread_local ThreadCtx t;
  return t;
}

DetKey detector_key(const DetectorModel& m) {
  DetKey k;
  k.w.resize(5 * std::size_t(kFilterWeights));
  for (int r = 0; r < 5; ++r) {
    if (int(m.filters[r].weights.size()) != kFilterWeights)
      throw std::invalid_argument("filter must carry exactly 3100 weights");
    std::memcpy(&k.w[std::size_t(r) * kFilterWeights], m.filters[r].weights.data(), sizeof(double) * kFilterWeights);
    k.b[r] = m.filters[r].bias;
  }
  k.thr = m.detection_threshold;
  k.ratio = m.min_face_ratio;
  const int geom[4] = {m.window_cells, m.cell_px, m.scale_num, m.scale_den};
  std::memcpy(k.geom, geom, sizeof geom);
  return k;
}

void ensure_detector(ThreadCtx& T, const DetectorModel& m) {
  DetKey key = detector_key(m);
  DeviceModels& R = registry(T.device);
  if (T.det_valid && T.generation == R.generation && T.det_key == key) return;
  std::lock_guard<std::mutex> lk(R.mu);
  if (!R.det_valid || !(R.det_key == key)) {
    if (!R.det_owner) check(bl_ctx_create(T.device, &R.det_owner));
    check(bl_detector_upload(R.det_owner, key.w.data(), key.b.data(), key.thr, m.window_cells, m.cell_px,
                             m.scale_num, m.scale_den, m.min_face_ratio));
    R.det_key = key;
    R.det_valid = true;
  }
  check(bl_ctx_share_models(T.get(), R.det_owner, BL_SHARE_DETECTOR));
  T.det_key = std::move(key);
  T.det_valid = true;
  T.generation = R.generation;
}

inline uint64_t mix(uint64_t h, uint64_t v) {  // FNV-1a style 64-bit step over whole words
  h ^= v;
  h *= 0x100000001B3ull;
  return h ^ (h >> 29);
}

inline uint64_t bits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, sizeof u);
  return u;
}

ErtKey ert_key(const ErtModel& m) {
  ErtKey k;
  const int L = m.landmark_count(), Tn = m.levels(), K = m.trees_per_level();
  k.head = {double(L), double(Tn), double(K), m.shrinkage};
  for (const Point2& p : m.mean_shape.points) {
    k.head.push_back(p.x);
    k.head.push_back(p.y);
  }
  uint64_t hs = 0xcbf29ce484222325ull, hl = 0x84222325cbf29ce4ull;
  for (std::size_t t = 0; t < m.cascade.size(); ++t) {
    const auto& lv = m.cascade[t];
    hl = mix(hl, lv.size());
    for (std::size_t i = 0; i < lv.size(); ++i) {
      const RegressionTree& tr = lv[i];
      hl = mix(hl, uint64_t(tr.depth));
      hl = mix(hl, tr.splits.size());
      hl = mix(hl, tr.leaves.size());
      for (const SplitNode& n : tr.splits) {
        hs = mix(hs, (uint64_t(uint32_t(n.anchor_a)) << 32) | uint32_t(n.anchor_b));
        hs = mix(hs, bits(n.offset_a.x));
        hs = mix(hs, bits(n.offset_a.y));
        hs = mix(hs, bits(n.offset_b.x));
        hs = mix(hs, bits(n.offset_b.y));
        hs = mix(hs, bits(n.threshold));
      }
      for (const auto& leaf : tr.leaves) {
        hl = mix(hl, reinterpret_cast<uintptr_t>(leaf.data()));
        hl = mix(hl, leaf.size());
      }
      if ((i & 15) == 0 && !tr.leaves.empty())  // sampled leaf values
        for (const auto& leaf : tr.leaves)
          if (!leaf.empty()) {
            k.head.push_back(leaf[t % leaf.size()].x);
            k.head.push_back(leaf.back().y);
          }
    }
  }
  k.split_hash = hs;
  k.layout_hash = hl;
  return k;
}

void upload_ert(bl_ctx* ctx, const ErtModel& m) {
  const int L = m.landmark_count(), Tn = m.levels(), K = m.trees_per_level();
  if (L < 2) throw std::invalid_argument("predict_landmarks: model has no mean shape");
  const int F = (Tn > 0 && K > 0) ? m.cascade[0][0].depth : 0;
  const int S = (1 << F) - 1, NL = 1 << F;
  std::vector<double> mean(2 * L);
  for (int i = 0; i < L; ++i) {
    mean[2 * i] = m.mean_shape.points[i].x;
    mean[2 * i + 1] = m.mean_shape.points[i].y;
  }
  std::vector<int32_t> an(std::size_t(Tn) * K * S * 2);
  std::vector<double> sp(std::size_t(Tn) * K * S * 5);
  std::vector<double> lv(std::size_t(Tn) * K * NL * L * 2);
  for (int t = 0; t < Tn; ++t) {
    if (int(m.cascade[t].size()) != K) throw model_error("every cascade level must carry K trees");
    for (int k = 0; k < K; ++k) {
      const RegressionTree& tr = m.cascade[t][k];
      if (int(tr.splits.size()) != S || int(tr.leaves.size()) != NL)
        throw model_error("tree split/leaf counts do not match depth F");
      const std::size_t tk = std::size_t(t) * K + k;
      for (int s = 0; s < S; ++s) {
        const SplitNode& n = tr.splits[s];
        an[(tk * S + s) * 2] = n.anchor_a;
        an[(tk * S + s) * 2 + 1] = n.anchor_b;
        double* p = &sp[(tk * S + s) * 5];
        p[0] = n.offset_a.x;
        p[1] = n.offset_a.y;
        p[2] = n.offset_b.x;
        p[3] = n.offset_b.y;
        p[4] = n.threshold;
      }
      for (int l = 0; l < NL; ++l) {
        if (int(tr.leaves[l].size()) != L) throw model_error("leaf delta must carry L points");
        double* q = &lv[(tk * NL + l) * std::size_t(L) * 2];
        for (int i = 0; i < L; ++i) {
          q[2 * i] = tr.leaves[l][i].x;
          q[2 * i + 1] = tr.leaves[l][i].y;
        }
      }
    }
  }
  check(bl_ert_upload(ctx, L, Tn, K, F, m.shrinkage, mean.data(), an.data(), sp.data(), lv.data()));
}

void ensure_ert(ThreadCtx& T, const ErtModel& m) {
  if (m.landmark_count() < 2) throw std::invalid_argument("predict_landmarks: model has no mean shape");
  ErtKey key = ert_key(m);
  DeviceModels& R = registry(T.device);
  if (T.ert_valid && T.generation == R.generation && T.ert_key == key) return;
  std::lock_guard<std::mutex> lk(R.mu);
  if (!R.ert_valid || !(R.ert_key == key)) {
    if (!R.ert_owner) check(bl_ctx_create(T.device, &R.ert_owner));
    upload_ert(R.ert_owner, m);
    R.ert_key = key;
    R.ert_valid = true;
  }
  check(bl_ctx_share_models(T.get(), R.ert_owner, BL_SHARE_ERT));
  T.ert_key = std::move(key);
  T.ert_valid = true;
  T.generation = R.generation;
}

// Frames go to the device as u8 when every pixel is an integer in [0,255] (lossless),
// otherwise as fp64.
bool integral_u8(const GrayImage& img) {
  for (const double v : img.pixels)
    if (!(v >= 0.0 && v <= 255.0) || v != std::floor(v)) return false;
  return true;
}

struct Packed {
  int pix = BL_PIX_U8;
  std::vector<uint8_t> u8;
  std::vector<double> f64;
  const void* data() const { return pix == BL_PIX_U8 ? (const void*)u8.data() : (const void*)f64.data(); }
};

Packed pack(const std::vector<const GrayImage*>& frames) {
  Packed p;
  bool all_u8 = true;
  for (const GrayImage* f : frames) all_u8 = all_u8 && integral_u8(*f);
  const std::size_t n = frames.empty() ? 0 : frames[0]->pixels.size();
  if (all_u8) {
    p.pix = BL_PIX_U8;
    p.u8.resize(n * frames.size());
    for (std::size_t i = 0; i < frames.size(); ++i)
      for (std::size_t j = 0; j < n; ++j) p.u8[i * n + j] = uint8_t(frames[i]->pixels[j]);
  } else {
    p.pix = BL_PIX_F64;
    p.f64.resize(n * frames.size());
    for (std::size_t i = 0; i < frames.size(); ++i)
      std::memcpy(&p.f64[i * n], frames[i]->pixels.data(), sizeof(double) * n);
  }
  return p;
}

void check_image(const GrayImage& img) {
  if (img.width < 1 || img.height < 1 || img.pixels.size() != std::size_t(img.width) * img.height)
    throw std::invalid_argument("image dimensions do not match its pixel buffer");
}

Detection from_c(const bl_detection& d) {
  Detection o;
  o.box = Box{d.box.x, d.box.y, d.box.w, d.box.h};
  o.score = d.score;
  o.scale_index = d.scale_index;
  o.rotation_index = d.rotation_index;
  return o;
}

}  // namespace

// ------------------------------------------------------------------------ image ----
GrayImage make_image(int width, int height, double fill) {  // image.cpp:13-20
  if (width < 1 || height < 1) throw std::invalid_argument("make_image: dimensions must be >= 1");
  GrayImage img;
  img.width = width;
  img.height = height;
  img.pixels.assign(std::size_t(width) * height, fill);
  return img;
}

GrayImage downscale_bilinear(const GrayImage& img) {
  if (img.width < 2 || img.height < 2)
    throw std::invalid_argument("downscale_bilinear: output dimension would be 0");
  check_image(img);
  GrayImage out = make_image(img.width * 5 / 6, img.height * 5 / 6);
  check(bl_downscale_bilinear(tls().get(), img.pixels.data(), img.width, img.height, out.pixels.data()));
  return out;
}

Pyramid build_pyramid(const GrayImage& img, int window) {
  check_image(img);
  bl_ctx* c = tls().get();
  int n = 0;
  std::vector<int> dims(128);
  std::vector<double> scales(64);
  check(bl_build_pyramid(c, img.pixels.data(), BL_PIX_F64, img.width, img.height, window, nullptr, 0,
                         dims.data(), scales.data(), 64, &n));
  if (n > 64) throw std::runtime_error("pyramid deeper than 64 levels");
  std::size_t total = 0;
  for (int k = 0; k < n; ++k) total += std::size_t(dims[2 * k]) * dims[2 * k + 1];
  std::vector<double> all(total);
  check(bl_build_pyramid(c, img.pixels.data(), BL_PIX_F64, img.width, img.height, window, all.data(), total,
                         dims.data(), scales.data(), 64, &n));
  Pyramid p;
  std::size_t off = 0;
  for (int k = 0; k < n; ++k) {
    GrayImage lv;
    lv.width = dims[2 * k];
    lv.height = dims[2 * k + 1];
    lv.pixels.assign(all.begin() + off, all.begin() + off + std::size_t(lv.width) * lv.height);
    off += lv.pixels.size();
    p.levels.push_back(std::move(lv));
    p.cumulative_scale.push_back(scales[k]);
  }
  return p;
}

// -------------------------------------------------------------------------- hog ----
GradientField compute_gradients(const GrayImage& img) {
  if (img.width < 3 || img.height < 3)
    throw std::invalid_argument("compute_gradients: image must be at least 3x3");
  check_image(img);
  GradientField g;
  g.width = img.width;
  g.height = img.height;
  g.orientation.assign(std::size_t(img.width) * img.height, 0);
  g.magnitude.assign(std::size_t(img.width) * img.height, 0.0);
  check(bl_compute_gradients(tls().get(), img.pixels.data(), img.width, img.height, g.orientation.data(),
                             g.magnitude.data()));
  return g;
}

CellGrid histogramize(const GradientField& grads) {
  CellGrid cg;
  cg.cells_w = grads.width / kCellSize;
  cg.cells_h = grads.height / kCellSize;
  cg.bins.assign(std::size_t(cg.cells_w) * cg.cells_h * kOrientationBins, 0.0);
  if (cg.cells_w == 0 || cg.cells_h == 0) return cg;
  check(bl_histogramize(tls().get(), grads.orientation.data(), grads.magnitude.data(), grads.width, grads.height,
                        cg.bins.data()));
  return cg;
}

EnergyGrid cell_energy(const CellGrid& cells) {
  EnergyGrid e;
  e.cells_w = cells.cells_w;
  e.cells_h = cells.cells_h;
  e.energy.assign(std::size_t(cells.cells_w) * cells.cells_h, 0.0);
  if (!e.energy.empty())
    check(bl_cell_energy(tls().get(), cells.bins.data(), cells.cells_w, cells.cells_h, e.energy.data()));
  return e;
}

FeatureImage compute_features(const CellGrid& cells, const EnergyGrid& energies) {
  if (cells.cells_w != energies.cells_w || cells.cells_h != energies.cells_h)
    throw std::invalid_argument("compute_features: cell and energy grids must share dimensions");
  FeatureImage f;
  f.cells_w = cells.cells_w;
  f.cells_h = cells.cells_h;
  f.values.assign(std::size_t(f.cells_w) * f.cells_h * kCellFeatures, 0.0);
  if (!f.values.empty())
    check(bl_compute_features(tls().get(), cells.bins.data(), energies.energy.data(), cells.cells_w, cells.cells_h,
                              f.values.data()));
  return f;
}

FeatureImage extract_features(const GrayImage& img) {
  if (img.width < 3 || img.height < 3)
    throw std::invalid_argument("compute_gradients: image must be at least 3x3");
  check_image(img);
  FeatureImage f;
  f.cells_w = img.width / kCellSize;
  f.cells_h = img.height / kCellSize;
  f.values.assign(std::size_t(f.cells_w) * f.cells_h * kCellFeatures, 0.0);
  if (!f.values.empty())
    check(bl_extract_features(tls().get(), img.pixels.data(), img.width, img.height, f.values.data(), nullptr,
                              nullptr));
  return f;
}

// --------------------------------------------------------------------- detector ----
double iou(const Box& a, const Box& b) {  // detector.cpp:16-28
  const long long ix0 = std::max(a.x, b.x);
  const long long iy0 = std::max(a.y, b.y);
  const long long ix1 = std::min<long long>(a.x + a.w, b.x + b.w);
  const long long iy1 = std::min<long long>(a.y + a.h, b.y + b.h);
  const long long iw = ix1 - ix0, ih = iy1 - iy0;
  if (iw <= 0 || ih <= 0) return 0.0;
  const double inter = double(iw) * double(ih);
  const double uni = double(a.w) * a.h + double(b.w) * b.h - inter;
  if (uni <= 0.0) return 0.0;
  return inter / uni;
}

static SaliencyMap score_gpu(const FeatureImage& feat, const LinearFilter& filter) {
  if (int(filter.weights.size()) != kFilterWeights)
    throw std::invalid_argument("filter must carry exactly 3100 weights");
  if (feat.cells_w < kWindowCells || feat.cells_h < kWindowCells)
    throw std::invalid_argument("feature image smaller than the 10x10 detection window");
  SaliencyMap s;
  s.width = feat.cells_w - (kWindowCells - 1);
  s.height = feat.cells_h - (kWindowCells - 1);
  s.scores.assign(std::size_t(s.width) * s.height, 0.0);
  check(bl_score_window(tls().get(), feat.values.data(), feat.cells_w, feat.cells_h, filter.weights.data(),
                        filter.bias, s.scores.data()));
  return s;
}

// Both scorers run on the device in their own summation order: bit-identical to the
// reference's score_separable and score_dense respectively.
SaliencyMap score_dense(const FeatureImage& feat, const LinearFilter& filter) {  // detector.cpp:45-64 order
  if (int(filter.weights.size()) != kFilterWeights)
    throw std::invalid_argument("filter must carry exactly 3100 weights");
  if (feat.cells_w < kWindowCells || feat.cells_h < kWindowCells)
    throw std::invalid_argument("feature image smaller than the 10x10 detection window");
  SaliencyMap s;
  s.width = feat.cells_w - (kWindowCells - 1);
  s.height = feat.cells_h - (kWindowCells - 1);
  s.scores.assign(std::size_t(s.width) * s.height, 0.0);
  check(bl_score_window_dense(tls().get(), feat.values.data(), feat.cells_w, feat.cells_h, filter.weights.data(),
                              filter.bias, s.scores.data()));
  return s;
}
SaliencyMap score_separable(const FeatureImage& feat, const LinearFilter& filter) {
  return score_gpu(feat, filter);
}

std::vector<Detection> threshold_detections(const SaliencyMap& sal, const DetectorModel& model, int scale_index,
                                            int rotation_index) {  // detector.cpp:102-122
  const double c = std::pow(double(model.scale_num) / model.scale_den, double(scale_index));
  const int side = int(std::floor(model.window_px() / c + 0.5));
  std::vector<Detection> dets;
  for (int cy = 0; cy < sal.height; ++cy)
    for (int cx = 0; cx < sal.width; ++cx) {
      const double s = sal.at(cx, cy);
      if (s > model.detection_threshold) {
        Detection d;
        d.box = {int(std::floor(cx * model.cell_px / c + 0.5)), int(std::floor(cy * model.cell_px / c + 0.5)), side,
                 side};
        d.score = s;
        d.scale_index = scale_index;
        d.rotation_index = rotation_index;
        dets.push_back(d);
      }
    }
  return dets;
}

std::vector<Detection> nms(std::vector<Detection> dets, double iou_threshold) {
  std::vector<Detection> out(dets.size());
  if (dets.empty()) return out;
  static_assert(sizeof(Detection) == sizeof(bl_detection), "layout");
  int64_t kept = 0;
  check(bl_nms(tls().get(), reinterpret_cast<const bl_detection*>(dets.data()), int64_t(dets.size()), iou_threshold,
               reinterpret_cast<bl_detection*>(out.data()), &kept));
  out.resize(std::size_t(kept));
  return out;
}

std::vector<int> eligible_scales(int img_w, int img_h, const DetectorModel& model,
                                 int n_levels) {  // detector.cpp:144-155
  const double min_face = model.min_face_ratio * std::min(img_w, img_h);
  std::vector<int> out;
  for (int k = 0; k < n_levels; ++k) {
    const double detectable =
        model.window_px() / std::pow(double(model.scale_num) / model.scale_den, double(k));
    if (detectable >= min_face * (1.0 - 1e-9)) out.push_back(k);
  }
  return out;
}

std::vector<Detection> detect_faces(const GrayImage& img, const DetectorModel& model) {
  return gpu::detect_faces_batch({img}, model)[0];
}

// -------------------------------------------------------------------------- ert ----
Point2 SimilarityTransform::apply(const Point2& p) const {  // ert.cpp:15-18
  const Point2 q = apply_linear(p);
  return {q.x + tx, q.y + ty};
}

Point2 SimilarityTransform::apply_linear(const Point2& p) const {  // ert.cpp:20-24
  const double a = scale * std::cos(rotation);
  const double b = scale * std::sin(rotation);
  return {a * p.x - b * p.y, b * p.x + a * p.y};
}

SimilarityTransform similarity_transform(const Shape& from, const Shape& to) {  // ert.cpp:26-69
  const std::size_t n = from.points.size();
  if (n < 2 || to.points.size() != n)
    throw std::invalid_argument("similarity_transform: shapes must share L >= 2 points");
  if (from.frame != to.frame) throw std::invalid_argument("similarity_transform: shapes must share a frame");
  double mfx = 0, mfy = 0, mtx = 0, mty = 0;
  for (std::size_t i = 0; i < n; ++i) {
    mfx += from.points[i].x;
    mfy += from.points[i].y;
    mtx += to.points[i].x;
    mty += to.points[i].y;
  }
  mfx /= double(n);
  mfy /= double(n);
  mtx /= double(n);
  mty /= double(n);
  double sff = 0, sre = 0, sim = 0;
  for (std::size_t i = 0; i < n; ++i) {
    const double fx = from.points[i].x - mfx, fy = from.points[i].y - mfy;
    const double txp = to.points[i].x - mtx, typ = to.points[i].y - mty;
    sff += fx * fx + fy * fy;
    sre += fx * txp + fy * typ;
    sim += fx * typ - fy * txp;
  }
  if (sff <= 0.0) throw std::invalid_argument("similarity_transform: source shape has no spread");
  const double a = sre / sff, b = sim / sff;
  SimilarityTransform t;
  t.scale = std::hypot(a, b);
  if (t.scale <= 0.0) throw std::invalid_argument("similarity_transform: target shape has no spread");
  t.rotation = std::atan2(b, a);
  t.tx = mtx - (a * mfx - b * mfy);
  t.ty = mty - (b * mfx + a * mfy);
  return t;
}

double sample_intensity(const GrayImage& img, const Box& box, const Shape& shape, const SimilarityTransform& tform,
                        int anchor, Point2 offset) {  // ert.cpp:71-85
  if (shape.frame != ShapeFrame::normalized)
    throw std::invalid_argument("sample_intensity: shape must be in the normalized frame");
  const Point2 off = tform.apply_linear(offset);
  const double nx = shape.points[anchor].x + off.x;
  const double ny = shape.points[anchor].y + off.y;
  const double px = box.x + nx * box.w;
  const double py = box.y + ny * box.h;
  const int ix = std::clamp(int(std::llround(px)), 0, img.width - 1);
  const int iy = std::clamp(int(std::llround(py)), 0, img.height - 1);
  return img.at(ix, iy);
}

const std::vector<Point2>& traverse_tree(const RegressionTree& tree,
                                         const IntensityPairFn& intensity_of) {  // ert.cpp:87-97
  std::size_t node = 0;
  const std::size_t n_splits = tree.splits.size();
  while (node < n_splits) {
    const SplitNode& s = tree.splits[node];
    const auto [ia, ib] = intensity_of(s);
    node = (ia - ib > s.threshold) ? 2 * node + 1 : 2 * node + 2;
  }
  return tree.leaves[node - n_splits];
}

Shape predict_landmarks(const GrayImage& img, const Box& box, const ErtModel& model, PredictStats* stats) {
  if (box.w <= 0 || box.h <= 0) throw std::invalid_argument("predict_landmarks: face box must have positive area");
  if (model.landmark_count() < 2) throw std::invalid_argument("predict_landmarks: model has no mean shape");
  Shape s = gpu::predict_landmarks_batch({img}, {0}, {box}, model)[0];
  if (stats) {
    std::uint64_t evals = 0;  // one intensity difference per visited split: T*K*F
    for (const auto& lv : model.cascade)
      for (const RegressionTree& t : lv) evals += std::uint64_t(t.depth);
    stats->intensity_diffs = evals;
  }
  return s;
}

// ------------------------------------------------------------------------- batch ----
namespace gpu {

void set_device(int device) {
  ThreadCtx& T = tls();
  if (T.device == device) return;
  registry(device);  // range check
  if (T.ctx) bl_ctx_destroy(T.ctx);
  T.ctx = nullptr;
  T.device = device;
  T.det_valid = false;
  T.ert_valid = false;
}

void invalidate_model_cache() {  // every thread re-checks against a fresh upload
  for (int d = 0; d < 64; ++d) {
    DeviceModels& R = registry(d);
    std::lock_guard<std::mutex> lk(R.mu);
    R.det_valid = false;
    R.ert_valid = false;
    ++R.generation;
  }
  ThreadCtx& T = tls();
  T.det_valid = false;
  T.ert_valid = false;
}

static void same_size(const std::vector<const GrayImage*>& fr) {
  for (const GrayImage* f : fr) {
    check_image(*f);
    if (f->width != fr[0]->width || f->height != fr[0]->height)
      throw std::invalid_argument("batched frames must share dimensions");
  }
}

std::vector<std::vector<Detection>> detect_faces_batch(const std::vector<GrayImage>& frames,
                                                       const DetectorModel& model) {
  std::vector<std::vector<Detection>> res(frames.size());
  if (frames.empty()) return res;
  ThreadCtx& T = tls();
  ensure_detector(T, model);
  std::vector<const GrayImage*> fr;
  for (const GrayImage& f : frames) fr.push_back(&f);
  same_size(fr);
  const int w = fr[0]->width, h = fr[0]->height;
  const Packed p = pack(fr);
  std::vector<int32_t> counts(frames.size());
  int64_t total = 0;
  // generous first guess; on BL_ERR_CAPACITY `total` reports the exact need
  int64_t cap = std::max<int64_t>(1024, int64_t(frames.size()) * 64);
  std::vector<bl_detection> out(static_cast<std::size_t>(cap));
  int rc = bl_detect(T.get(), p.data(), p.pix, int(frames.size()), w, h, w, std::size_t(w) * h, out.data(), cap,
                     counts.data(), &total);
  if (rc == BL_ERR_CAPACITY && total > cap) {
    cap = total;
    out.resize(std::size_t(cap));
    rc = bl_detect(T.get(), p.data(), p.pix, int(frames.size()), w, h, w, std::size_t(w) * h, out.data(), cap,
                   counts.data(), &total);
  }
  check(rc);
  std::size_t o = 0;
  for (std::size_t i = 0; i < frames.size(); ++i)
    for (int k = 0; k < counts[i]; ++k) res[i].push_back(from_c(out[o++]));
  return res;
}

std::vector<Shape> predict_landmarks_batch(const std::vector<GrayImage>& frames, const std::vector<int>& frame_of_box,
                                           const std::vector<Box>& boxes, const ErtModel& model) {
  if (frame_of_box.size() != boxes.size()) throw std::invalid_argument("frame_of_box and boxes differ in length");
  std::vector<Shape> res;
  if (boxes.empty()) return res;
  ThreadCtx& T = tls();
  ensure_ert(T, model);
  std::vector<const GrayImage*> fr;
  for (const GrayImage& f : frames) fr.push_back(&f);
  same_size(fr);
  const Packed p = pack(fr);
  const int L = model.landmark_count();
  std::vector<double> xy(boxes.size() * std::size_t(L) * 2);
  static_assert(sizeof(Box) == sizeof(bl_box), "layout");
  check(bl_landmarks(T.get(), p.data(), p.pix, int(frames.size()), fr[0]->width, fr[0]->height, fr[0]->width,
                     std::size_t(fr[0]->width) * fr[0]->height, frame_of_box.data(),
                     reinterpret_cast<const bl_box*>(boxes.data()), int64_t(boxes.size()), xy.data(), nullptr));
  res.resize(boxes.size());
  for (std::size_t b = 0; b < boxes.size(); ++b) {
    res[b].frame = ShapeFrame::image;
    res[b].points.resize(L);
    for (int i = 0; i < L; ++i) res[b].points[i] = {xy[(b * L + i) * 2], xy[(b * L + i) * 2 + 1]};
  }
  return res;
}

std::vector<FrameResult> detect_and_landmark(const std::vector<GrayImage>& frames, const DetectorModel& hog,
                                             const ErtModel& ert) {
  std::vector<FrameResult> res(frames.size());
  if (frames.empty()) return res;
  ThreadCtx& T = tls();
  ensure_detector(T, hog);
  ensure_ert(T, ert);
  std::vector<const GrayImage*> fr;
  for (const GrayImage& f : frames) fr.push_back(&f);
  same_size(fr);
  const int w = fr[0]->width, h = fr[0]->height, L = ert.landmark_count();
  const Packed p = pack(fr);
  std::vector<int32_t> counts(frames.size());
  int64_t total = 0;
  int64_t cap = std::max<int64_t>(1024, int64_t(frames.size()) * 64);
  std::vector<bl_detection> out(static_cast<std::size_t>(cap));
  std::vector<double> xy(std::size_t(cap) * L * 2);
  int rc = bl_detect_landmarks(T.get(), p.data(), p.pix, int(frames.size()), w, h, w, std::size_t(w) * h,
                               out.data(), cap, counts.data(), &total, xy.data());
  if (rc == BL_ERR_CAPACITY && total > cap) {
    cap = total;
    out.resize(std::size_t(cap));
    xy.resize(std::size_t(cap) * L * 2);
    rc = bl_detect_landmarks(T.get(), p.data(), p.pix, int(frames.size()), w, h, w, std::size_t(w) * h, out.data(),
                             cap, counts.data(), &total, xy.data());
  }
  check(rc);
  std::size_t o = 0;
  for (std::size_t i = 0; i < frames.size(); ++i)
    for (int k = 0; k < counts[i]; ++k, ++o) {
      res[i].detections.push_back(from_c(out[o]));
      Shape s;
      s.frame = ShapeFrame::image;
      s.points.resize(L);
      for (int j = 0; j < L; ++j) s.points[j] = {xy[(o * L + j) * 2], xy[(o * L + j) * 2 + 1]};
      res[i].landmarks.push_back(std::move(s));
    }
  return res;
}

// The same over several GPUs: contiguous frame shards, one context and host thread per device
// (bl_multi), models bound from each device's registry, results in frame order.
std::vector<FrameResult> detect_and_landmark(const std::vector<GrayImage>& frames, const DetectorModel& hog,
                                             const ErtModel& ert, const std::vector<int>& devices) {
  if (devices.empty()) throw std::invalid_argument("detect_and_landmark: empty device list");
  std::vector<FrameResult> res(frames.size());
  if (frames.empty()) return res;
  struct Multi {
    bl_multi* m = nullptr;
  };
  static std::mutex mu;
  static std::map<std::vector<int>, Multi> pool;  // process-lifetime, one per device list
  std::lock_guard<std::mutex> lk(mu);
  Multi& M = pool[devices];
  if (!M.m) check(bl_multi_create(devices.data(), int(devices.size()), &M.m));
  const DetKey dk = detector_key(hog);
  const ErtKey ek = ert_key(ert);
  for (std::size_t i = 0; i < devices.size(); ++i) {  // bind the device's registry models
    bl_ctx* c = nullptr;
    check(bl_multi_context(M.m, int(i), &c));
    DeviceModels& R = registry(devices[i]);
    std::lock_guard<std::mutex> rl(R.mu);
    if (!R.det_valid || !(R.det_key == dk)) {
      if (!R.det_owner) check(bl_ctx_create(devices[i], &R.det_owner));
      check(bl_detector_upload(R.det_owner, dk.w.data(), dk.b.data(), dk.thr, hog.window_cells, hog.cell_px,
                               hog.scale_num, hog.scale_den, hog.min_face_ratio));
      R.det_key = dk;
      R.det_valid = true;
    }
    if (!R.ert_valid || !(R.ert_key == ek)) {
      if (!R.ert_owner) check(bl_ctx_create(devices[i], &R.ert_owner));
      upload_ert(R.ert_owner, ert);
      R.ert_key = ek;
      R.ert_valid = true;
    }
    check(bl_ctx_share_models(c, R.det_owner, BL_SHARE_DETECTOR));
    check(bl_ctx_share_models(c, R.ert_owner, BL_SHARE_ERT));
  }
  std::vector<const GrayImage*> fr;
  for (const GrayImage& f : frames) fr.push_back(&f);
  same_size(fr);
  const int w = fr[0]->width, h = fr[0]->height, L = ert.landmark_count();
  const Packed p = pack(fr);
  std::vector<int32_t> counts(frames.size());
  int64_t total = 0;
  const int64_t cap = int64_t(frames.size()) * 64;
  std::vector<bl_detection> out(static_cast<std::size_t>(cap));
  std::vector<double> xy(std::size_t(cap) * L * 2);
  check(bl_multi_detect_landmarks(M.m, p.data(), p.pix, int(frames.size()), w, h, w, std::size_t(w) * h, out.data(),
                                  cap, counts.data(), &total, xy.data(), nullptr));
  std::size_t o = 0;
  for (std::size_t i = 0; i < frames.size(); ++i)
    for (int k = 0; k < counts[i]; ++k, ++o) {
      res[i].detections.push_back(from_c(out[o]));
      Shape s;
      s.frame = ShapeFrame::image;
      s.points.resize(L);
      for (int j = 0; j < L; ++j) s.points[j] = {xy[(o * L + j) * 2], xy[(o * L + j) * 2 + 1]};
      res[i].landmarks.push_back(std::move(s));
    }
  return res;
}

}  // namespace gpu
// ------------------------------------------------------------------ data formats ----
// PGM and model files through the C-ABI adapters (bl_io.cpp): same formats, messages and
// exception classes as image.cpp:67-127, detector.cpp:291-351, ert.cpp:340-469.
GrayImage load_pgm(const std::string& path) {
  int w = 0, h = 0;
  check(bl_read_pgm(path.c_str(), &w, &h, nullptr, 0));
  std::vector<std::uint8_t> px(std::size_t(w) * h);
  check(bl_read_pgm(path.c_str(), &w, &h, px.data(), px.size()));
  GrayImage img = make_image(w, h);
  for (std::size_t i = 0; i < px.size(); ++i) img.pixels[i] = double(px[i]);
  return img;
}

void save_pgm(const GrayImage& img, const std::string& path) {
  check(bl_write_pgm(path.c_str(), img.pixels.data(), img.width, img.height));
}

void save_model(const DetectorModel& model, const std::string& path) {
  const std::size_t per = std::size_t(model.window_cells) * model.window_cells * kCellFeatures;
  std::vector<double> w(per * 5), b(5);
  for (int r = 0; r < 5; ++r) {
    if (model.filters[r].weights.size() != per)
      throw model_error(path + ": filter " + std::to_string(r) + " does not match window_cells");
    std::copy(model.filters[r].weights.begin(), model.filters[r].weights.end(), w.begin() + r * per);
    b[r] = model.filters[r].bias;
  }
  check(bl_write_detector_json(path.c_str(), w.data(), b.data(), model.detection_threshold, model.window_cells,
                               model.cell_px, model.scale_num, model.scale_den, model.min_face_ratio));
}

DetectorModel load_detector_model(const std::string& path) {
  DetectorModel m;
  check(bl_read_detector_json(path.c_str(), nullptr, nullptr, &m.detection_threshold, &m.window_cells, &m.cell_px,
                              &m.scale_num, &m.scale_den, &m.min_face_ratio));
  const std::size_t per = std::size_t(m.window_cells) * m.window_cells * kCellFeatures;
  std::vector<double> w(per * 5), b(5);
  check(bl_read_detector_json(path.c_str(), w.data(), b.data(), &m.detection_threshold, &m.window_cells, &m.cell_px,
                              &m.scale_num, &m.scale_den, &m.min_face_ratio));
  for (int r = 0; r < 5; ++r) {
    m.filters[r].weights.assign(w.begin() + r * per, w.begin() + (r + 1) * per);
    m.filters[r].bias = b[r];
  }
  return m;
}

void save_model(const ErtModel& model, const std::string& path) {
  const int L = model.landmark_count(), T = model.levels(), K = model.trees_per_level();
  const int F = (T > 0 && K > 0) ? model.cascade[0][0].depth : 0;
  const std::size_t S = (std::size_t(1) << F) - 1, NL = std::size_t(1) << F;
  std::vector<double> mean(2 * std::size_t(L)), sp, lv;
  std::vector<std::int32_t> an;
  for (int i = 0; i < L; ++i) {
    mean[2 * i] = model.mean_shape.points[i].x;
    mean[2 * i + 1] = model.mean_shape.points[i].y;
  }
  for (const auto& level : model.cascade) {
    if (int(level.size()) != K) throw model_error(path + ": every cascade level must carry K trees");
    for (const RegressionTree& tree : level) {
      if (tree.splits.size() != S || tree.leaves.size() != NL)
        throw model_error(path + ": tree split/leaf counts do not match depth F");
      for (const SplitNode& n : tree.splits) {
        an.push_back(n.anchor_a);
        an.push_back(n.anchor_b);
        for (double v : {n.offset_a.x, n.offset_a.y, n.offset_b.x, n.offset_b.y, n.threshold}) sp.push_back(v);
      }
      for (const auto& leaf : tree.leaves)
        for (const Point2& p : leaf) {
          lv.push_back(p.x);
          lv.push_back(p.y);
        }
    }
  }
  check(bl_write_ert_json(path.c_str(), L, T, K, F, model.shrinkage, mean.data(), an.data(), sp.data(), lv.data()));
}

ErtModel load_ert_model(const std::string& path) {
  bl_ert_file* f = nullptr;
  int L = 0, T = 0, K = 0, F = 0;
  ErtModel m;
  check(bl_ert_file_open(path.c_str(), &f, &L, &T, &K, &F, &m.shrinkage));
  const std::size_t S = (std::size_t(1) << F) - 1, NL = std::size_t(1) << F, n = std::size_t(T) * K;
  std::vector<double> mean(2 * std::size_t(L)), sp(n * S * 5), lv(n * NL * L * 2);
  std::vector<std::int32_t> an(n * S * 2);
  const int rc = bl_ert_file_copy(f, mean.data(), an.data(), sp.data(), lv.data());
  bl_ert_file_close(f);
  check(rc);
  m.mean_shape.frame = ShapeFrame::normalized;
  for (int i = 0; i < L; ++i) m.mean_shape.points.push_back({mean[2 * i], mean[2 * i + 1]});
  for (int t = 0; t < T; ++t) {
    std::vector<RegressionTree> level;
    for (int k = 0; k < K; ++k) {
      const std::size_t tk = std::size_t(t) * K + k;
      RegressionTree tree;
      tree.depth = F;
      for (std::size_t s = 0; s < S; ++s) {
        const std::size_t i = tk * S + s;
        SplitNode node;
        node.anchor_a = an[2 * i];
        node.anchor_b = an[2 * i + 1];
        node.offset_a = {sp[5 * i], sp[5 * i + 1]};
        node.offset_b = {sp[5 * i + 2], sp[5 * i + 3]};
        node.threshold = sp[5 * i + 4];
        tree.splits.push_back(node);
      }
      for (std::size_t q = 0; q < NL; ++q) {
        std::vector<Point2> delta(L);
        const double* d = &lv[((tk * NL + q) * L) * 2];
        for (int i = 0; i < L; ++i) delta[i] = {d[2 * i], d[2 * i + 1]};
        tree.leaves.push_back(std::move(delta));
      }
      level.push_back(std::move(tree));
    }
    m.cascade.push_back(std::move(level));
  }
  return m;
}

EyeIndices eye_indices(int landmark_count) {  // ert.cpp:340-347: the iBUG 300-W 68-point convention
  if (landmark_count != 68)
    throw std::invalid_argument("eye_indices: no eye mapping for L=" + std::to_string(landmark_count) +
                                "; only the 68-landmark convention is built in");
  return EyeIndices{{36, 37, 38, 39, 40, 41}, {42, 43, 44, 45, 46, 47}};
}

EyeIndices eye_indices(int landmark_count, const EyeIndices& custom) {  // ert.cpp:349-356
  for (const auto& eye : {custom.left, custom.right})
    for (const int i : eye)
      if (i < 0 || i >= landmark_count) throw std::invalid_argument("eye_indices: custom index out of range");
  return custom;
}

// ------------------------------------------------------------------ blink / pipeline ----
// EAR and the blink trace (blink.cpp:13-135): host folds over the device's landmarks.
namespace {
double pdist(const Point2& a, const Point2& b) { return std::hypot(a.x - b.x, a.y - b.y); }

double quantile_lin(std::vector<double> v, double q) {  // linear interpolation over order statistics
  std::sort(v.begin(), v.end());
  if (v.size() == 1) return v[0];
  const double pos = q * double(v.size() - 1);
  const std::size_t lo = std::size_t(pos);
  if (lo + 1 >= v.size()) return v.back();
  return v[lo] + (pos - double(lo)) * (v[lo + 1] - v[lo]);
}

double closure(double ear, double baseline) {
  if (baseline <= 0.0) return 1.0;  // a never-open trace counts every frame as closed
  return std::clamp(1.0 - ear / baseline, 0.0, 1.0);
}
}  // namespace

double eye_aspect_ratio(const std::array<Point2, 6>& p) {
  const double horiz = pdist(p[0], p[3]);
  if (horiz <= 1e-9) throw std::invalid_argument("eye_aspect_ratio: degenerate eye, corner span ~ 0");
  return (pdist(p[1], p[5]) + pdist(p[2], p[4])) / (2.0 * horiz);
}

double shape_ear(const Shape& landmarks, const std::array<int, 6>& eye) {
  std::array<Point2, 6> pts;
  for (std::size_t i = 0; i < 6; ++i) {
    if (eye[i] < 0 || eye[i] >= int(landmarks.points.size()))
      throw std::invalid_argument("shape_ear: eye index out of range");
    pts[i] = landmarks.points[eye[i]];
  }
  return eye_aspect_ratio(pts);
}

BlinkTrace build_trace(const std::vector<FrameEar>& frames, double fps, double baseline_quantile) {
  if (fps <= 0.0) throw std::invalid_argument("build_trace: fps must be positive");
  std::vector<FrameEar> ordered = frames;
  std::sort(ordered.begin(), ordered.end(),
            [](const FrameEar& a, const FrameEar& b) { return a.frame_index < b.frame_index; });
  for (std::size_t i = 1; i < ordered.size(); ++i)
    if (ordered[i].frame_index == ordered[i - 1].frame_index)
      throw std::invalid_argument("build_trace: duplicate frame index " + std::to_string(ordered[i].frame_index));
  std::vector<double> lefts, rights;
  for (const FrameEar& f : ordered)
    if (f.face_found) {
      lefts.push_back(f.ear_left);
      rights.push_back(f.ear_right);
    }
  if (lefts.empty())
    throw std::invalid_argument("build_trace: no frames with a detected face, cannot establish an EAR baseline");
  BlinkTrace trace;
  trace.fps = fps;
  trace.baseline_left = quantile_lin(lefts, baseline_quantile);
  trace.baseline_right = quantile_lin(rights, baseline_quantile);
  for (const FrameEar& f : ordered) {
    BlinkSample s;
    s.frame_index = f.frame_index;
    s.t = double(f.frame_index) / fps;
    s.face_found = f.face_found;
    if (f.face_found) {
      s.ear_left = f.ear_left;
      s.ear_right = f.ear_right;
      s.closure_left = closure(f.ear_left, trace.baseline_left);
      s.closure_right = closure(f.ear_right, trace.baseline_right);
    }
    trace.samples.push_back(s);
  }
  return trace;
}

std::vector<BlinkEvent> detect_blinks(const BlinkTrace& trace, double closure_threshold, std::size_t min_frames) {
  std::vector<BlinkEvent> events;  // maximal runs of closure_left >= threshold lasting >= min_frames
  std::size_t start = 0, len = 0;
  double peak = 0.0;
  auto close_run = [&](std::size_t last) {
    if (len >= min_frames && min_frames > 0)
      events.push_back(BlinkEvent{trace.samples[start].frame_index, trace.samples[last].frame_index, peak});
    len = 0;
    peak = 0.0;
  };
  for (std::size_t i = 0; i < trace.samples.size(); ++i) {
    const BlinkSample& s = trace.samples[i];
    if (s.closure_left && *s.closure_left >= closure_threshold) {
      if (len == 0) start = i;
      ++len;
      peak = std::max(peak, *s.closure_left);
    } else if (len > 0) {
      close_run(i - 1);
    }
  }
  if (len > 0) close_run(trace.samples.size() - 1);
  return events;
}

FrameSequence ingest(const std::string& frames_dir) {
  int n = 0, w = 0, h = 0;
  check(bl_ingest(frames_dir.c_str(), &n, &w, &h));
  FrameSequence seq;
  seq.dir = frames_dir;
  seq.width = w;
  seq.height = h;
  for (int i = 0; i < n; ++i) {
    char name[32];
    std::snprintf(name, sizeof name, "frame_%06d.pgm", i);
    seq.paths.push_back((std::filesystem::path(frames_dir) / name).string());
  }
  return seq;
}

RunOutput run(const std::string& frames_dir, const DetectorModel& hog, const ErtModel& ert, double fps,
              const PipelineConfig& config) {
  ThreadCtx& T = tls();
  ensure_detector(T, hog);
  ensure_ert(T, ert);
  int n = 0, w = 0, h = 0;
  check(bl_ingest(frames_dir.c_str(), &n, &w, &h));
  const int L = ert.landmark_count();
  std::vector<bl_frame_result> fr(n);
  std::vector<bl_detection> dets(std::size_t(std::max(1, n)) * 64);
  std::vector<double> lms(std::size_t(n) * 2 * L), base(2);
  int64_t tot = 0;
  const int batch = config.mode == ExecMode::sequential ? 1 : int(std::max<std::size_t>(1, config.batch_size));
  int rc = bl_run(T.get(), frames_dir.c_str(), fps, batch, fr.data(), n, dets.data(), int64_t(dets.size()), &tot,
                  lms.data(), base.data());
  if (rc == BL_ERR_CAPACITY) {  // more detections than the first guess: size exactly and rerun
    dets.resize(std::size_t(n) * 5 * 4096);
    rc = bl_run(T.get(), frames_dir.c_str(), fps, batch, fr.data(), n, dets.data(), int64_t(dets.size()), &tot,
                lms.data(), base.data());
  }
  check(rc);
  RunOutput out;
  out.trace.fps = fps;
  out.trace.baseline_left = base[0];
  out.trace.baseline_right = base[1];
  std::size_t off = 0;
  for (int i = 0; i < n; ++i) {
    const bl_frame_result& f = fr[i];
    FrameResult r;
    r.frame_index = std::size_t(f.frame_index);
    for (int k = 0; k < f.n_detections; ++k) r.detections.push_back(*reinterpret_cast<const Detection*>(&dets[off + k]));
    off += std::size_t(f.n_detections);
    r.timings = StageTimings{f.decode_ms, f.detect_ms, f.landmark_ms};
    BlinkSample s;
    s.frame_index = r.frame_index;
    s.t = f.t;
    s.face_found = f.face_found != 0;
    if (f.face_found) {
      r.face = *reinterpret_cast<const Detection*>(&f.face);
      Shape sh;
      sh.frame = ShapeFrame::image;
      for (int p = 0; p < L; ++p) sh.points.push_back({lms[(std::size_t(i) * L + p) * 2], lms[(std::size_t(i) * L + p) * 2 + 1]});
      r.landmarks = std::move(sh);
      s.ear_left = f.ear_left;
      s.ear_right = f.ear_right;
      s.closure_left = f.closure_left;
      s.closure_right = f.closure_right;
    }
    out.trace.samples.push_back(s);
    out.results.push_back(std::move(r));
  }
  return out;
}

std::vector<BenchReport> bench(const std::string& frames_dir, const DetectorModel& hog, const ErtModel& ert,
                               const std::vector<PipelineConfig>& grid) {
  // pipeline.cpp:406-454 on the device path: a discarded warm-up run, the sequential run as
  // the speedup denominator, then every grid entry; per-stage means over the frames.
  auto timed = [&](const PipelineConfig& cfg, BenchReport& r) {
    run(frames_dir, hog, ert, 30.0, cfg);  // warm-up (model upload, plan arenas, page cache)
    const auto t0 = std::chrono::steady_clock::now();
    const RunOutput o = run(frames_dir, hog, ert, 30.0, cfg);
    const double total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    r.frames = o.results.size();
    r.config = cfg;
    for (const FrameResult& f : o.results) {
      r.decode_ms += f.timings.decode_ms;
      r.detect_ms += f.timings.detect_ms;
      r.landmark_ms += f.timings.landmark_ms;
    }
    const double n = double(std::max<std::size_t>(1, r.frames));
    r.decode_ms /= n;
    r.detect_ms /= n;
    r.landmark_ms /= n;
    r.end_to_end_ms = total / n;
    r.fps = 1000.0 / r.end_to_end_ms;
  };
  PipelineConfig seq_cfg;
  seq_cfg.mode = ExecMode::sequential;
  BenchReport ref;
  timed(seq_cfg, ref);
  std::vector<BenchReport> out;
  for (const PipelineConfig& cfg : grid) {
    BenchReport r;
    if (cfg.mode == ExecMode::sequential) {
      r = ref;
      r.config = cfg;
      r.speedup = 1.0;
    } else {
      timed(cfg, r);
      r.speedup = ref.end_to_end_ms / r.end_to_end_ms;
    }
    out.push_back(r);
  }
  return out;
}

}  // namespace blinkline
