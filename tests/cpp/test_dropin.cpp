// The drop-in C++ API (paper_2006_00816_b200/cpp/blinkline_gpu.hpp) exercised with the
// reference's own unit-test cases (proj/tests/test_{image,hog,detector,ert}.cpp), written the
// way a reference user would call the library.
//
//   test_dropin --host   API scalar helpers only (no GPU needed)
//   test_dropin --gpu    the device-backed hot path (B200)
//
// Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>

#include "blinkline_gpu.hpp"

using namespace blinkline;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    if (cond) {                                                         \
      ++g_pass;                                                         \
    } else {                                                            \
      ++g_fail;                                                         \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);       \
    }                                                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                        \
  do {                                                                  \
    bool ok_ = false;                                                   \
    try {                                                               \
      (void)(expr);                                                     \
    } catch (const T&) {                                                \
      ok_ = true;                                                       \
    } catch (...) {                                                     \
    }                                                                   \
    CHECK(ok_ && #T);                                                   \
  } while (0)

static double urand(std::mt19937_64& rng, double lo, double hi) {
  return lo + (hi - lo) * (double(rng() >> 11) * 0x1.0p-53);
}

static Shape make_shape(std::initializer_list<Point2> pts) {
  Shape s;
  s.points = pts;
  return s;
}

// ------------------------------------------------------------------- host only ----
static void host_tests() {
  // iou (detector.cpp:16-28)
  CHECK(iou(Box{0, 0, 10, 10}, Box{0, 0, 10, 10}) == 1.0);
  CHECK(iou(Box{0, 0, 10, 10}, Box{10, 0, 10, 10}) == 0.0);
  CHECK(iou(Box{0, 0, 10, 10}, Box{5, 0, 10, 10}) == 50.0 / 150.0);
  // eligible_scales (test_detector.cpp:232-258)
  DetectorModel model;
  CHECK((eligible_scales(640, 480, model, 10) == std::vector<int>{1, 2, 3, 4, 5, 6, 7, 8, 9}));
  model.min_face_ratio = 0.0;
  CHECK((eligible_scales(640, 480, model, 4) == std::vector<int>{0, 1, 2, 3}));
  model.min_face_ratio = 0.9;
  CHECK((eligible_scales(100, 100, model, 2) == std::vector<int>{1}));
  // threshold_detections known answers (test_detector.cpp:146-178)
  DetectorModel m2;
  m2.detection_threshold = 1.0;
  SaliencyMap sal;
  sal.width = 5;
  sal.height = 4;
  sal.scores.assign(20, 0.0);
  CHECK(threshold_detections(sal, m2, 0, 0).empty());
  sal.scores[2 * 5 + 3] = 2.0;
  auto d = threshold_detections(sal, m2, 0, 1);
  CHECK(d.size() == 1 && d[0].box.x == 24 && d[0].box.y == 16 && d[0].box.w == 80 && d[0].rotation_index == 1);
  sal.scores.assign(20, 0.0);
  sal.scores[0] = 2.0;
  d = threshold_detections(sal, m2, 2, 0);
  CHECK(d.size() == 1 && d[0].box.w == 115 && d[0].box.h == 115);
  // similarity_transform known transforms (test_ert.cpp:37-103)
  const Shape s3 = make_shape({{0, 0}, {1, 0}, {0.5, 1}});
  SimilarityTransform t = similarity_transform(s3, s3);
  CHECK(std::fabs(t.scale - 1.0) < 1e-12 && std::fabs(t.rotation) < 1e-12);
  const Shape from = make_shape({{-1, 0}, {1, 0}, {0, 1}, {0, -1}});
  Shape to = from;
  for (Point2& p : to.points) {
    p.x *= 2;
    p.y *= 2;
  }
  t = similarity_transform(from, to);
  CHECK(std::fabs(t.scale - 2.0) < 1e-12);
  CHECK_THROWS_AS(similarity_transform(make_shape({{0.5, 0.5}, {0.5, 0.5}}), make_shape({{0, 0}, {1, 1}})),
                  std::invalid_argument);
  // sample_intensity (test_ert.cpp:105-132)
  GrayImage img = make_image(20, 20);
  for (int y = 0; y < 20; ++y)
    for (int x = 0; x < 20; ++x) img.at(x, y) = 10.0 * y + x;
  const Box box{4, 4, 10, 10};
  const SimilarityTransform ident;
  const Shape s2 = make_shape({{0.5, 0.5}, {0.2, 0.3}});
  CHECK(sample_intensity(img, box, s2, ident, 0, {0, 0}) == img.at(9, 9));
  CHECK(sample_intensity(img, box, s2, ident, 1, {0, 0}) == img.at(6, 7));
  CHECK(sample_intensity(img, box, make_shape({{0.5, 0.5}}), ident, 0, {10.0, 0}) == img.at(19, 9));
  SimilarityTransform rot;
  rot.scale = 2.0;
  rot.rotation = M_PI / 2;
  rot.tx = rot.ty = 100.0;
  CHECK(sample_intensity(img, box, make_shape({{0.5, 0.5}}), rot, 0, {0.1, 0}) == img.at(9, 11));
  // traverse_tree bit path (test_ert.cpp:134-171)
  RegressionTree tree;
  tree.depth = 3;
  tree.splits.assign(7, SplitNode{});
  for (int i = 0; i < 7; ++i) tree.splits[i].threshold = double(i);
  for (int i = 0; i < 8; ++i) tree.leaves.push_back({{double(i), double(i)}});
  const auto& leaf = traverse_tree(tree, [](const SplitNode& sn) {
    const bool left = int(sn.threshold) % 2 == 0;
    return std::pair<double, double>{left ? sn.threshold + 1 : sn.threshold - 1, 0.0};
  });
  CHECK(leaf[0].x == 2.0);
  // error types
  CHECK_THROWS_AS(make_image(0, 5), std::invalid_argument);

  // data formats (test_image.cpp:50-119, test_detector.cpp:353-394, test_ert.cpp:406-443)
  const std::string dir = "/tmp/blinkline_dropin_" + std::to_string(::getpid());
  if (std::system(("mkdir -p " + dir).c_str()) != 0) std::printf("mkdir failed\n");
  GrayImage pg = make_image(7, 5);
  for (std::size_t i = 0; i < pg.pixels.size(); ++i) pg.pixels[i] = double((i * 37) % 256);
  save_pgm(pg, dir + "/f.pgm");
  const GrayImage back = load_pgm(dir + "/f.pgm");
  CHECK(back.width == 7 && back.height == 5 && back.pixels == pg.pixels);
  CHECK_THROWS_AS(load_pgm(dir + "/missing.pgm"), io_error);
  {
    std::ofstream(dir + "/bad.pgm") << "P5\n2 2\n300\n";
    bool msg_ok = false;
    try {
      load_pgm(dir + "/bad.pgm");
    } catch (const io_error& e) {
      msg_ok = std::string(e.what()).find("unsupported maxval 300 (limit 255) at byte") != std::string::npos;
    }
    CHECK(msg_ok);
  }
  DetectorModel dm;
  std::mt19937_64 rng(11);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (auto& f : dm.filters) {
    for (double& wv : f.weights) wv = u(rng);
    f.bias = u(rng);
  }
  dm.detection_threshold = 0.25;
  save_model(dm, dir + "/hog.json");
  const DetectorModel dm2 = load_detector_model(dir + "/hog.json");
  bool same = dm2.detection_threshold == dm.detection_threshold && dm2.window_cells == 10;
  for (int r = 0; r < 5; ++r) same = same && dm2.filters[r].weights == dm.filters[r].weights && dm2.filters[r].bias == dm.filters[r].bias;
  CHECK(same);
  std::ofstream(dir + "/v2.json") << "{\"version\": \"hog-v2\"}";
  CHECK_THROWS_AS(load_detector_model(dir + "/v2.json"), model_error);
  CHECK_THROWS_AS(load_detector_model(dir + "/none.json"), io_error);
  ErtModel em;
  em.shrinkage = 0.1;
  for (int i = 0; i < 4; ++i) em.mean_shape.points.push_back({0.1 * i, 0.2 * i});
  for (int t = 0; t < 2; ++t) {
    std::vector<RegressionTree> level;
    for (int k = 0; k < 3; ++k) {
      RegressionTree tr;
      tr.depth = 2;
      for (int sidx = 0; sidx < 3; ++sidx) tr.splits.push_back(SplitNode{sidx % 4, (sidx + 1) % 4, {u(rng), u(rng)}, {u(rng), u(rng)}, u(rng)});
      for (int l = 0; l < 4; ++l) tr.leaves.push_back({{u(rng), u(rng)}, {u(rng), u(rng)}, {u(rng), u(rng)}, {u(rng), u(rng)}});
      level.push_back(tr);
    }
    em.cascade.push_back(level);
  }
  save_model(em, dir + "/ert.json");
  const ErtModel em2 = load_ert_model(dir + "/ert.json");
  bool esame = em2.levels() == 2 && em2.trees_per_level() == 3 && em2.landmark_count() == 4 && em2.shrinkage == 0.1;
  for (int t = 0; esame && t < 2; ++t)
    for (int k = 0; k < 3; ++k) {
      const RegressionTree &a = em.cascade[t][k], &b2 = em2.cascade[t][k];
      for (int sidx = 0; sidx < 3; ++sidx)
        esame = esame && a.splits[sidx].anchor_a == b2.splits[sidx].anchor_a &&
                a.splits[sidx].offset_b.y == b2.splits[sidx].offset_b.y && a.splits[sidx].threshold == b2.splits[sidx].threshold;
      for (int l = 0; l < 4; ++l)
        for (int i = 0; i < 4; ++i) esame = esame && a.leaves[l][i].x == b2.leaves[l][i].x && a.leaves[l][i].y == b2.leaves[l][i].y;
    }
  CHECK(esame);
  CHECK(eye_indices(68).left[0] == 36 && eye_indices(68).right[5] == 47);

  // EAR and the blink trace (test_blink.cpp:41-160)
  {
    std::array<Point2, 6> eye{{{0, 0}, {1, 1}, {3, 1}, {4, 0}, {3, -1}, {1, -1}}};
    CHECK(std::fabs(eye_aspect_ratio(eye) - 0.5) < 1e-12);
    std::array<Point2, 6> flat{{{0, 0}, {0, 0}, {0, 0}, {0, 0}, {0, 0}, {0, 0}}};
    CHECK_THROWS_AS(eye_aspect_ratio(flat), std::invalid_argument);
    auto scripted = [](const std::vector<double>& ears) {
      std::vector<FrameEar> f;
      for (std::size_t i = 0; i < ears.size(); ++i) f.push_back({i, true, ears[i], ears[i]});
      return f;
    };
    BlinkTrace tr = build_trace(scripted({0.3, 0.3, 0.3, 0.3}), 100.0);
    CHECK(std::fabs(tr.baseline_left - 0.3) < 1e-12 && *tr.samples[0].closure_left == 0.0);
    tr = build_trace(scripted({0.3, 0.3, 0.0, 0.3, 0.3}), 50.0);
    CHECK(*tr.samples[2].closure_left == 1.0 && *tr.samples[0].closure_left == 0.0);
    std::vector<double> ears(20, 0.3);
    for (int i = 7; i < 12; ++i) ears[i] = 0.0;
    const auto ev = detect_blinks(build_trace(scripted(ears), 10.0), 0.7, 3);
    CHECK(ev.size() == 1 && ev[0].onset_frame == 7 && ev[0].offset_frame == 11 && ev[0].peak_closure == 1.0);
    std::vector<FrameEar> none{{0, false, 0, 0}, {1, false, 0, 0}};
    CHECK_THROWS_AS(build_trace(none, 10.0), std::invalid_argument);
    std::vector<FrameEar> dup{{0, true, 0.3, 0.3}, {0, true, 0.2, 0.2}};
    CHECK_THROWS_AS(build_trace(dup, 10.0), std::invalid_argument);
  }
  CHECK_THROWS_AS(eye_indices(5), std::invalid_argument);
  if (std::system(("rm -rf " + dir).c_str()) != 0) std::printf("cleanup failed\n");
}

// -------------------------------------------------------------------------- GPU ----
static DetectorModel pattern_detector(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  std::vector<double> v(3102);
  in.read(reinterpret_cast<char*>(v.data()), sizeof(double) * v.size());
  if (!in) throw std::runtime_error("cannot read " + path);
  DetectorModel m;
  for (auto& f : m.filters) {
    f.weights.assign(v.begin(), v.begin() + 3100);
    f.bias = v[3100];
  }
  m.detection_threshold = v[3101];
  return m;
}

static void draw_ring(GrayImage& img, double cx, double cy, double size) {  // helpers.cpp:33-52 shape
  for (int y = 0; y < img.height; ++y)
    for (int x = 0; x < img.width; ++x) {
      const double r = std::hypot(x - cx, y - cy);
      if (r <= 0.18 * size)
        img.at(x, y) = 30.0;
      else if (r <= 0.34 * size)
        img.at(x, y) = 225.0;
      else if (r <= 0.47 * size)
        img.at(x, y) = 60.0;
    }
}

static void gpu_tests(const std::string& model_path) {
  // pyramid (test_image.cpp:121-194)
  const Pyramid pyr = build_pyramid(make_image(640, 480, 10.0), 80);
  CHECK(pyr.levels.size() == 10 && pyr.levels[1].width == 533 && pyr.levels[1].height == 400);
  for (std::size_t k = 0; k < pyr.levels.size(); ++k) CHECK(pyr.cumulative_scale[k] == std::pow(5.0 / 6.0, double(k)));
  const GrayImage c12 = downscale_bilinear(make_image(12, 12, 100.0));
  CHECK(c12.width == 10 && c12.pixels[55] == 100.0);
  // gradients (test_hog.cpp:76-108)
  GrayImage ramp = make_image(8, 8);
  for (int y = 0; y < 8; ++y)
    for (int x = 0; x < 8; ++x) ramp.at(x, y) = x;
  const GradientField g = compute_gradients(ramp);
  CHECK(g.magnitude[g.index(3, 3)] == 2.0 && g.orientation[g.index(3, 3)] == 0);
  CHECK_THROWS_AS(compute_gradients(make_image(2, 5)), std::invalid_argument);
  // histogram single-pixel split (test_hog.cpp:138-158)
  GradientField f;
  f.width = f.height = 32;
  f.orientation.assign(1024, 0);
  f.magnitude.assign(1024, 0.0);
  f.orientation[f.index(11, 11)] = 4;
  f.magnitude[f.index(11, 11)] = 8.0;
  const CellGrid cg = histogramize(f);
  CHECK(cg.cell(1, 1)[4] == 8.0 * 0.9375 * 0.9375 && cg.cell(0, 0)[4] == 8.0 * 0.0625 * 0.0625);
  CellGrid ones;
  ones.cells_w = ones.cells_h = 1;
  ones.bins.assign(18, 1.0);
  CHECK(cell_energy(ones).at(0, 0) == 36.0);
  // score known answers (test_detector.cpp:71-110)
  FeatureImage fi;
  fi.cells_w = 12;
  fi.cells_h = 11;
  fi.values.assign(12 * 11 * 31, 0.0);
  LinearFilter lf;
  lf.bias = 2.5;
  const SaliencyMap sal = score_dense(fi, lf);
  CHECK(sal.width == 3 && sal.height == 2 && sal.scores[0] == 2.5);
  // nms (test_detector.cpp:180-230)
  CHECK(nms({}).empty());
  const auto kept = nms({Detection{{10, 10, 50, 50}, 1.0, 0, 0}, Detection{{10, 10, 50, 50}, 2.0, 0, 0}});
  CHECK(kept.size() == 1 && kept[0].score == 2.0);
  // detect_faces end to end (test_detector.cpp:260-281)
  const DetectorModel model = pattern_detector(model_path);
  CHECK(detect_faces(make_image(320, 240, 20.0), model).empty());
  CHECK(detect_faces(make_image(60, 60, 20.0), model).empty());
  GrayImage frame = make_image(640, 480, 20.0);
  std::mt19937_64 rng(36);
  for (double& p : frame.pixels) p = std::min(255.0, std::max(0.0, p + urand(rng, -1.5, 1.5)));
  draw_ring(frame, 300.0, 250.0, 160.0);
  const auto dets = detect_faces(frame, model);
  bool hit = false;
  const Box truth{220, 170, 160, 160};
  for (const Detection& dd : dets) hit = hit || iou(dd.box, truth) >= 0.5;
  CHECK(!dets.empty() && hit);
  // batch == single-frame calls
  const auto batch = gpu::detect_faces_batch({frame, make_image(640, 480, 20.0)}, model);
  CHECK(batch.size() == 2 && batch[0].size() == dets.size() && batch[1].empty());
  // predict_landmarks: zero-delta cascade lands the mean shape (test_ert.cpp:173-225)
  ErtModel ert;
  ert.shrinkage = 0.1;
  ert.mean_shape = make_shape({{0.25, 0.5}, {0.75, 0.5}, {0.5, 0.25}});
  RegressionTree tr;
  tr.depth = 2;
  tr.splits.assign(3, SplitNode{});
  tr.leaves.assign(4, std::vector<Point2>(3, Point2{0, 0}));
  ert.cascade.assign(3, std::vector<RegressionTree>(4, tr));
  GrayImage half = make_image(64, 64);
  for (int y = 0; y < 64; ++y)
    for (int x = 0; x < 64; ++x) half.at(x, y) = x > 32 ? 200.0 : 10.0;
  PredictStats st;
  const Shape lm = predict_landmarks(half, Box{8, 8, 48, 48}, ert, &st);
  CHECK(lm.frame == ShapeFrame::image && lm.points[0].x == 8 + 0.25 * 48 && lm.points[2].y == 8 + 0.25 * 48);
  CHECK(st.intensity_diffs == 3u * 4u * 2u);
  CHECK_THROWS_AS(predict_landmarks(half, Box{0, 0, 0, 10}, ert), std::invalid_argument);
  // single depth-1 tree applies one shrunk delta
  ErtModel one;
  one.shrinkage = 0.1;
  one.mean_shape = make_shape({{0.25, 0.5}, {0.75, 0.5}});
  RegressionTree t1;
  t1.depth = 1;
  SplitNode sn;
  sn.anchor_a = 1;
  sn.anchor_b = 0;
  sn.threshold = 50.0;
  t1.splits = {sn};
  t1.leaves = {{{0.1, 0.2}, {-0.1, 0.0}}, {{9, 9}, {9, 9}}};
  one.cascade = {{t1}};
  const Shape o = predict_landmarks(half, Box{8, 8, 48, 48}, one);
  CHECK(std::fabs(o.points[0].x - (8 + 0.26 * 48)) < 1e-12 && std::fabs(o.points[1].x - (8 + 0.74 * 48)) < 1e-12);
  // detect + landmark in one device pass
  const auto both = gpu::detect_and_landmark({frame}, model, one);
  CHECK(both.size() == 1 && both[0].detections.size() == dets.size() && both[0].landmarks.size() == dets.size());
  // ... and sharded over a device list (one B200 on the lease: the same device twice)
  {
    const auto multi = gpu::detect_and_landmark({frame, make_image(640, 480, 20.0), frame}, model, one, {0, 0});
    bool eq = multi.size() == 3 && multi[1].detections.empty() && multi[0].detections.size() == dets.size() &&
              multi[2].detections.size() == dets.size();
    for (std::size_t k = 0; eq && k < dets.size(); ++k)
      eq = multi[0].detections[k].score == dets[k].score && multi[2].detections[k].box.x == dets[k].box.x &&
           multi[0].landmarks[k].points[1].y == both[0].landmarks[k].points[1].y;
    CHECK(eq);
  }
  // a model edited in place (same object, same buffers): a split threshold change is seen by
  // the next call (the content key hashes every split record)
  {
    ErtModel m = one;
    const Shape before = predict_landmarks(half, Box{8, 8, 48, 48}, m);
    m.cascade[0][0].splits[0].threshold = 1000.0;  // now Ia - Ib > thr fails: the other leaf
    const Shape after = predict_landmarks(half, Box{8, 8, 48, 48}, m);
    CHECK(before.points[0].x != after.points[0].x && std::fabs(after.points[0].x - (8 + 0.25 * 48 + 0.9 * 48)) < 1e-9);
    m.cascade[0][0].leaves[1][0].x = -9.0;  // a leaf value edited in place: explicit invalidation
    gpu::invalidate_model_cache();
    const Shape again = predict_landmarks(half, Box{8, 8, 48, 48}, m);
    CHECK(std::fabs(again.points[0].x - (8 + (0.25 - 0.9) * 48)) < 1e-9);
  }
  // score_dense in the definitional order vs score_separable (both bit-identical to the
  // reference in their own order): a single non-zero weight makes them equal
  {
    FeatureImage fr2;
    fr2.cells_w = 13;
    fr2.cells_h = 12;
    fr2.values.resize(13 * 12 * 31);
    std::mt19937_64 r2(5);
    for (double& v : fr2.values) v = urand(r2, 0.0, 0.4);
    LinearFilter d1;
    d1.weights[2 * 310 + 3 * 31 + 7] = 1.0;
    const SaliencyMap a = score_dense(fr2, d1), b = score_separable(fr2, d1);
    CHECK(a.scores == b.scores && a.scores[0] == fr2.cell(3, 2)[7]);
  }
  // concurrent callers on their own threads share the device models and agree bit for bit
  {
    std::vector<Shape> out(4);
    std::vector<std::thread> th;
    for (int t = 0; t < 4; ++t) th.emplace_back([&, t] { out[t] = predict_landmarks(half, Box{8, 8, 48, 48}, one); });
    for (auto& t : th) t.join();
    bool eq = true;
    for (int t = 1; t < 4; ++t) eq = eq && out[t].points[0].x == out[0].points[0].x && out[t].points[1].y == out[0].points[1].y;
    CHECK(eq && out[0].points[0].x == o.points[0].x);
  }

  // run() over a frame directory: sequential == pipelined (test_pipeline.cpp:92-123)
  {
    const std::string dir = "/tmp/blinkline_run_" + std::to_string(::getpid());
    if (std::system(("mkdir -p " + dir).c_str()) != 0) std::printf("mkdir failed\n");
    std::mt19937_64 frng(1000);
    for (int i = 0; i < 10; ++i) {
      GrayImage f = make_image(320, 240, 20.0);
      for (double& p : f.pixels) p = std::round(std::min(255.0, std::max(0.0, p + urand(frng, -1.5, 1.5))));
      if (i != 4) draw_ring(f, 150.0 + 3 * i, 120.0, 110.0);
      char name[32];
      std::snprintf(name, sizeof name, "/frame_%06d.pgm", i);
      save_pgm(f, dir + name);
    }
    ErtModel e68;  // zero-delta 68-point cascade: landmarks = the mean shape in each face box
    e68.shrinkage = 0.1;
    for (int i = 0; i < 68; ++i) e68.mean_shape.points.push_back({0.2 + 0.6 * std::cos(0.3 * i) * 0.5 + 0.3, 0.5 + 0.25 * std::sin(0.7 * i)});
    RegressionTree z;
    z.depth = 1;
    z.splits.assign(1, SplitNode{});
    z.leaves.assign(2, std::vector<Point2>(68, Point2{0, 0}));
    e68.cascade.assign(2, std::vector<RegressionTree>(3, z));
    PipelineConfig pc;
    pc.mode = ExecMode::pipelined;
    pc.batch_size = 4;
    const RunOutput a = run(dir, model, e68, 25.0, PipelineConfig{});
    const RunOutput b = run(dir, model, e68, 25.0, pc);
    bool same = a.results.size() == 10 && b.results.size() == 10;
    for (std::size_t i = 0; same && i < 10; ++i) {
      same = a.results[i].detections.size() == b.results[i].detections.size() &&
             a.results[i].face.has_value() == b.results[i].face.has_value();
      for (std::size_t k = 0; same && k < a.results[i].detections.size(); ++k)
        same = a.results[i].detections[k].score == b.results[i].detections[k].score;
      if (same && a.results[i].landmarks)
        same = a.results[i].landmarks->points[40].x == b.results[i].landmarks->points[40].x;
    }
    CHECK(same);
    CHECK(!a.results[4].face.has_value() && a.results[0].face.has_value());
    CHECK(a.trace.samples.size() == 10 && !a.trace.samples[4].face_found && a.trace.samples[3].closure_left.has_value());
    CHECK(a.trace.baseline_left > 0.0 && std::fabs(a.trace.samples[2].t - 2.0 / 25.0) < 1e-15);
    CHECK(ingest(dir).paths.size() == 10 && ingest(dir).width == 320);
    if (std::system(("rm -rf " + dir).c_str()) != 0) std::printf("cleanup failed\n");
  }
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  try {
    host_tests();
    if (gpu) gpu_tests(argc > 2 ? argv[2] : "tests/golden/pattern_detector.bin");
  } catch (const std::exception& e) {
    std::printf("EXCEPTION %s\n", e.what());
    ++g_fail;
  }
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
