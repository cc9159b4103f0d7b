// blinkline drop-in API served by the B200 device path.
//
// Declares, in namespace blinkline, the value types and hot-path functions of the
// reference library's public headers (proj/include/blinkline/{image,hog,detector,ert,
// errors}.hpp) with the same names, layouts, argument meaning and exception types, so a
// caller of the reference's detect_faces / predict_landmarks (and the stage functions they
// are built from) recompiles against this header and links libblinkline_gpu.so instead.
// Every function below is implemented on top of the C-ABI in include/blinkline_b200.h.
//
// Also what sits either side of the path: the frame-sequence runtime
// (ingest / run / bench, device-backed), PGM frames, the "hog-v1" / "ert-v1" model files and
// the EAR / blink-trace fold.  Out of scope (not declared here): the trainers, evaluation
// metrics, the trace CSV reader/writer and the CLI -- DESIGN.md §8.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace blinkline {

// ------------------------------------------------------------------ errors (errors.hpp)
struct io_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct model_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------- image (image.hpp)
struct GrayImage {
  int width = 0;
  int height = 0;
  std::vector<double> pixels;  // row-major, width * height
  double at(int x, int y) const { return pixels[std::size_t(y) * width + x]; }
  double& at(int x, int y) { return pixels[std::size_t(y) * width + x]; }
};

GrayImage make_image(int width, int height, double fill = 0.0);
// P5/P2 PGM, maxval <= 255 (image.hpp:23-28); malformed files throw io_error with the byte offset.
GrayImage load_pgm(const std::string& path);
void save_pgm(const GrayImage& img, const std::string& path);
GrayImage downscale_bilinear(const GrayImage& img);

struct Pyramid {
  std::vector<GrayImage> levels;
  std::vector<double> cumulative_scale;
};
Pyramid build_pyramid(const GrayImage& img, int window = 80);

// --------------------------------------------------------------------- hog (hog.hpp)
inline constexpr int kOrientationBins = 18;
inline constexpr int kCellSize = 8;
inline constexpr int kCellFeatures = 31;

struct GradientField {
  int width = 0;
  int height = 0;
  std::vector<std::uint8_t> orientation;
  std::vector<double> magnitude;
  std::size_t index(int x, int y) const { return std::size_t(y) * width + x; }
};

struct CellGrid {
  int cells_w = 0;
  int cells_h = 0;
  std::vector<double> bins;
  double* cell(int cx, int cy) { return &bins[(std::size_t(cy) * cells_w + cx) * kOrientationBins]; }
  const double* cell(int cx, int cy) const {
    return &bins[(std::size_t(cy) * cells_w + cx) * kOrientationBins];
  }
};

struct EnergyGrid {
  int cells_w = 0;
  int cells_h = 0;
  std::vector<double> energy;
  double at(int cx, int cy) const { return energy[std::size_t(cy) * cells_w + cx]; }
};

struct FeatureImage {
  int cells_w = 0;
  int cells_h = 0;
  std::vector<double> values;
  double* cell(int cx, int cy) { return &values[(std::size_t(cy) * cells_w + cx) * kCellFeatures]; }
  const double* cell(int cx, int cy) const {
    return &values[(std::size_t(cy) * cells_w + cx) * kCellFeatures];
  }
};

GradientField compute_gradients(const GrayImage& img);
CellGrid histogramize(const GradientField& grads);
EnergyGrid cell_energy(const CellGrid& cells);
FeatureImage compute_features(const CellGrid& cells, const EnergyGrid& energies);
FeatureImage extract_features(const GrayImage& img);

// ----------------------------------------------------------- detector (detector.hpp)
inline constexpr int kWindowCells = 10;
inline constexpr int kFilterWeights = kWindowCells * kWindowCells * kCellFeatures;

struct Box {
  int x = 0;
  int y = 0;
  int w = 0;
  int h = 0;
};

double iou(const Box& a, const Box& b);

struct LinearFilter {
  std::vector<double> weights = std::vector<double>(kFilterWeights, 0.0);
  double bias = 0.0;
};

struct DetectorModel {
  std::array<LinearFilter, 5> filters;
  double detection_threshold = 0.0;
  int window_cells = kWindowCells;
  int cell_px = kCellSize;
  int scale_num = 5;
  int scale_den = 6;
  double min_face_ratio = 0.2;
  int window_px() const { return window_cells * cell_px; }
};

struct SaliencyMap {
  int width = 0;
  int height = 0;
  std::vector<double> scores;
  double at(int cx, int cy) const { return scores[std::size_t(cy) * width + cx]; }
};

struct Detection {
  Box box;
  double score = 0.0;
  int scale_index = 0;
  int rotation_index = 0;
};

SaliencyMap score_dense(const FeatureImage& feat, const LinearFilter& filter);
SaliencyMap score_separable(const FeatureImage& feat, const LinearFilter& filter);
std::vector<Detection> threshold_detections(const SaliencyMap& sal, const DetectorModel& model,
                                            int scale_index, int rotation_index);
std::vector<Detection> nms(std::vector<Detection> dets, double iou_threshold = 0.5);
std::vector<int> eligible_scales(int img_w, int img_h, const DetectorModel& model, int n_levels);
std::vector<Detection> detect_faces(const GrayImage& img, const DetectorModel& model);
// JSON model file, format version "hog-v1" (detector.hpp:97-100).
void save_model(const DetectorModel& model, const std::string& path);
DetectorModel load_detector_model(const std::string& path);

// --------------------------------------------------------------------- ert (ert.hpp)
struct Point2 {
  double x = 0.0;
  double y = 0.0;
};

enum class ShapeFrame { normalized, image };

struct Shape {
  std::vector<Point2> points;
  ShapeFrame frame = ShapeFrame::normalized;
};

struct SimilarityTransform {
  double scale = 1.0;
  double rotation = 0.0;
  double tx = 0.0;
  double ty = 0.0;
  Point2 apply(const Point2& p) const;
  Point2 apply_linear(const Point2& p) const;
};

SimilarityTransform similarity_transform(const Shape& from, const Shape& to);

struct SplitNode {
  int anchor_a = 0;
  int anchor_b = 0;
  Point2 offset_a;
  Point2 offset_b;
  double threshold = 0.0;
};

struct RegressionTree {
  int depth = 0;
  std::vector<SplitNode> splits;
  std::vector<std::vector<Point2>> leaves;
};

struct ErtModel {
  Shape mean_shape;
  std::vector<std::vector<RegressionTree>> cascade;
  double shrinkage = 0.1;
  int landmark_count() const { return int(mean_shape.points.size()); }
  int levels() const { return int(cascade.size()); }
  int trees_per_level() const { return cascade.empty() ? 0 : int(cascade[0].size()); }
};

double sample_intensity(const GrayImage& img, const Box& box, const Shape& shape,
                        const SimilarityTransform& tform, int anchor, Point2 offset);

using IntensityPairFn = std::function<std::pair<double, double>(const SplitNode&)>;
const std::vector<Point2>& traverse_tree(const RegressionTree& tree, const IntensityPairFn& intensity_of);

struct PredictStats {
  std::uint64_t intensity_diffs = 0;
};

Shape predict_landmarks(const GrayImage& img, const Box& box, const ErtModel& model,
                        PredictStats* stats = nullptr);

struct EyeIndices {
  std::array<int, 6> left;
  std::array<int, 6> right;
};
// iBUG 300-W convention for 68 landmarks: left eye 36..41, right eye 42..47 (ert.hpp:116-125).
EyeIndices eye_indices(int landmark_count);
EyeIndices eye_indices(int landmark_count, const EyeIndices& custom);

// JSON model file, format version "ert-v1" (ert.hpp:127-129).
void save_model(const ErtModel& model, const std::string& path);
ErtModel load_ert_model(const std::string& path);

// --------------------------------------------------------------- blink (blink.hpp)
double eye_aspect_ratio(const std::array<Point2, 6>& p);
double shape_ear(const Shape& landmarks, const std::array<int, 6>& eye);

struct BlinkSample {
  std::size_t frame_index = 0;
  double t = 0.0;
  bool face_found = false;
  std::optional<double> ear_left;
  std::optional<double> ear_right;
  std::optional<double> closure_left;
  std::optional<double> closure_right;
};

struct BlinkTrace {
  double fps = 0.0;
  std::vector<BlinkSample> samples;
  double baseline_left = 0.0;
  double baseline_right = 0.0;
};

struct FrameEar {
  std::size_t frame_index = 0;
  bool face_found = false;
  double ear_left = 0.0;
  double ear_right = 0.0;
};

BlinkTrace build_trace(const std::vector<FrameEar>& frames, double fps, double baseline_quantile = 0.95);

struct BlinkEvent {
  std::size_t onset_frame = 0;
  std::size_t offset_frame = 0;
  double peak_closure = 0.0;
};

std::vector<BlinkEvent> detect_blinks(const BlinkTrace& trace, double closure_threshold = 0.7,
                                      std::size_t min_frames = 3);

// ------------------------------------------------------- pipeline (pipeline.hpp)
// The frame-sequence runtime with detect + landmark on the device (bl_run): frames are
// decoded on the host and pushed through in batches of batch_size (the decode of batch
// b+1 overlaps the device work on batch b); sequential mode = batches of one.  Results are
// in frame order and identical between modes.  Worker counts are accepted for API
// compatibility; the device path has one decode thread and one device stream per context.
enum class ExecMode { sequential, pipelined };

struct PipelineConfig {
  ExecMode mode = ExecMode::sequential;
  std::size_t batch_size = 16;
  int detect_workers = 1;
  int landmark_workers = 1;
  std::size_t queue_capacity = 4;
};

struct FrameSequence {
  std::string dir;
  std::vector<std::string> paths;
  int width = 0;
  int height = 0;
};

FrameSequence ingest(const std::string& frames_dir);

struct StageTimings {
  double decode_ms = 0.0;
  double detect_ms = 0.0;
  double landmark_ms = 0.0;
};

struct FrameResult {
  std::size_t frame_index = 0;
  std::vector<Detection> detections;
  std::optional<Detection> face;
  std::optional<Shape> landmarks;
  StageTimings timings;
};

struct RunOutput {
  std::vector<FrameResult> results;
  BlinkTrace trace;
};

RunOutput run(const std::string& frames_dir, const DetectorModel& hog, const ErtModel& ert, double fps,
              const PipelineConfig& config);

struct BenchReport {
  std::size_t frames = 0;
  PipelineConfig config;
  double decode_ms = 0.0;
  double detect_ms = 0.0;
  double landmark_ms = 0.0;
  double end_to_end_ms = 0.0;
  double fps = 0.0;
  double speedup = 1.0;
};

std::vector<BenchReport> bench(const std::string& frames_dir, const DetectorModel& hog, const ErtModel& ert,
                               const std::vector<PipelineConfig>& grid);

// ------------------------------------------------------------ batch extensions (new)
namespace gpu {

// Device used by this thread's context (default: $BLINKLINE_DEVICE or 0).
void set_device(int device);
// Models live on each device once, shared by every thread's context, and are matched by
// content: weights exactly; an ERT model by structure, mean shape, a full hash of its split
// records and leaf-row addresses, and sampled leaf values.  After editing leaf VALUES of an
// ERT model in place (same buffers), call this so the next call re-uploads.
void invalidate_model_cache();

// detect_faces over many equal-size frames in one device pass; result[i] is frame i's list.
std::vector<std::vector<Detection>> detect_faces_batch(const std::vector<GrayImage>& frames,
                                                       const DetectorModel& model);
// predict_landmarks for many (frame, box) pairs in one device pass.
std::vector<Shape> predict_landmarks_batch(const std::vector<GrayImage>& frames,
                                           const std::vector<int>& frame_of_box,
                                           const std::vector<Box>& boxes, const ErtModel& model);
// detect + landmark every kept detection (pipeline.cpp:159-190 per frame), all on device.
struct FrameResult {
  std::vector<Detection> detections;
  std::vector<Shape> landmarks;  // aligned with detections
};
std::vector<FrameResult> detect_and_landmark(const std::vector<GrayImage>& frames,
                                             const DetectorModel& hog, const ErtModel& ert);
// The same sharded over several GPUs of this process (contiguous frame shards, one host thread
// per device, results in frame order; a device may be listed more than once).
std::vector<FrameResult> detect_and_landmark(const std::vector<GrayImage>& frames,
                                             const DetectorModel& hog, const ErtModel& ert,
                                             const std::vector<int>& devices);

}  // namespace gpu
}  // namespace blinkline
