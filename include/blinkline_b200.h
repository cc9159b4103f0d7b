/* blinkline_b200 -- C-ABI of the B200-native face-detection + 68-landmark hot path.
 *
 * This is the drop-in boundary.  Plain pointers and sizes only; no CUDA, torch or C++
 * types cross it.  Every entry point replaces a reference (blinkline, /root/reference/proj)
 * interface, cited per function as  `replaces: <header>:<line>`.  The C++ drop-in API
 * (paper_2006_00816_b200/cpp/blinkline_gpu.hpp) and the Python binding
 * (paper_2006_00816_b200/__init__.py) both sit on top of this header.
 *
 * Results are bit-identical to the reference CPU implementation: pyramid levels, gradient
 * orientations/magnitudes, cell histograms, energies, features, detection scores and boxes
 * are equal to the last bit; ERT leaf indices are equal and landmarks agree to <= 1e-9 px
 * (the similarity transform goes through CUDA's hypot/atan2/cos/sin, which can differ from
 * glibc's by an ulp).  See DESIGN.md §3.
 *
 * Error convention: every function returns BL_OK (0) or a BL_ERR_* code; the message of the
 * last failure on the calling thread is bl_last_error().  The C++ layer maps
 * BL_ERR_INVALID -> std::invalid_argument, BL_ERR_MODEL -> blinkline::model_error and the
 * rest -> std::runtime_error, matching the reference's exception types.
 *
 * Threading: a bl_ctx is owned by one thread at a time (calls on one ctx are serialised
 * internally by a mutex).  Different contexts may run concurrently, on one or several GPUs.
 *
 * Memory: `frames`, `boxes` and outputs may be host (pageable or pinned) or device pointers;
 * the library inspects each pointer.  Host inputs are staged through pinned buffers. */
#ifndef BLINKLINE_B200_H
#define BLINKLINE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BL_ABI_VERSION 1

enum {
  BL_OK = 0,
  BL_ERR_INVALID = 1,  /* precondition violated        -> std::invalid_argument */
  BL_ERR_MODEL = 2,    /* model shape/content invalid  -> blinkline::model_error */
  BL_ERR_CUDA = 3,     /* CUDA runtime/device failure   -> std::runtime_error */
  BL_ERR_CAPACITY = 4, /* a fixed device capacity was exceeded -> std::runtime_error */
  BL_ERR_STATE = 5,    /* no model uploaded / context misuse */
  BL_ERR_IO = 6        /* file unreadable / malformed PGM  -> blinkline::io_error */
};

enum { BL_PIX_U8 = 0, BL_PIX_F64 = 1 };

typedef struct bl_ctx bl_ctx;

/* Same layout as blinkline::Box (detector.hpp:15-20). */
typedef struct {
  int32_t x, y, w, h;
} bl_box;

/* Same layout as blinkline::Detection (detector.hpp:52-57). */
typedef struct {
  bl_box box;
  double score;
  int32_t scale_index;
  int32_t rotation_index;
} bl_detection;

/* Per-stage device time of the last pipeline call (CUDA events), when enabled. */
enum {
  BL_STAGE_H2D = 0,
  BL_STAGE_PYRAMID,
  BL_STAGE_GRADHIST,
  BL_STAGE_FEATURES,
  BL_STAGE_SCREEN,
  BL_STAGE_RESCORE,
  BL_STAGE_NMS,
  BL_STAGE_ERT,
  BL_STAGE_D2H,
  BL_STAGE_COUNT
};

/* ------------------------------------------------------------------ context ---- */
int bl_abi_version(void);
/* Host-only geometry of a detect batch, no device work: pyramid level dims (image.cpp:158-172),
 * the scored levels -- eligible_scales (detector.cpp:144-155) with room for a window
 * (detector.cpp:163-167) -- and per scored level the scale (5/6)^k and the box side
 * round_half_up(window_px / c) (detector.cpp:104-105). */
int bl_plan_geometry(int w, int h, int window_cells, int cell_px, int scale_num, int scale_den,
                     double min_face_ratio, int* dims, int* scored, double* scale_c, int* side,
                     int max_levels, int* n_levels, int* n_scored);
const char* bl_last_error(void);
int bl_device_count(int* n);
int bl_ctx_create(int device, bl_ctx** out);
void bl_ctx_destroy(bl_ctx* ctx);
/* Run on a caller-provided cudaStream_t (passed as void*); NULL restores the ctx stream. */
int bl_ctx_set_stream(bl_ctx* ctx, void* cuda_stream);
int bl_ctx_synchronize(bl_ctx* ctx);
/* Number of kernels this context has launched so far (for launch-count accounting). */
int bl_ctx_launch_count(bl_ctx* ctx, uint64_t* out);
/* Per-stage CUDA-event timing of subsequent pipeline calls (adds events; off by default). */
int bl_ctx_enable_stage_timing(bl_ctx* ctx, int enable);
int bl_ctx_stage_times(bl_ctx* ctx, float* ms /* BL_STAGE_COUNT */, int* launches /* BL_STAGE_COUNT */);
/* CUDA graphs for the pipelined path (bl_submit, and the synchronous calls built on it; on by
 * default, BL_GRAPHS=0 in the environment disables at context creation): a batch's detection
 * launches and its landmark cascade are captured once per (lane, slot, input buffer, batch
 * shape) and replayed, so host submit is a few graph/event calls instead of ~60 launches.
 * Per-stage timing runs without graphs.  Results are identical either way. */
int bl_ctx_enable_graphs(bl_ctx* ctx, int enable);
/* Classifier screen implementation (both feed the same exact fp64 re-score, so detections
 * are bit-identical either way): BL_SCREEN_TCGEN05 -- implicit GEMM on the tensor cores
 * (tcgen05.mma kind::f16, default); BL_SCREEN_FP32 -- register-tiled CUDA-core FMA.  The
 * environment variable BL_SCREEN=fp32|tc overrides the default at context creation. */
#define BL_SCREEN_TCGEN05 0
#define BL_SCREEN_FP32 1
int bl_ctx_set_screen(bl_ctx* ctx, int mode);

/* ------------------------------------------------------------------- models ---- */
/* replaces: the DetectorModel value passed to detect_faces (detector.hpp:31-41,87).
 * weights: 5 x (window_cells*window_cells*31) row-major (cell-y, cell-x, feature). */
int bl_detector_upload(bl_ctx* ctx, const double* weights, const double* biases, double threshold,
                       int window_cells, int cell_px, int scale_num, int scale_den,
                       double min_face_ratio);
/* replaces: the ErtModel value passed to predict_landmarks (ert.hpp:44-68,86).
 * anchors: T*K*S x 2 int32 (S = 2^F-1, level order), split_params: T*K*S x 5
 * (offset_a.x, offset_a.y, offset_b.x, offset_b.y, threshold), leaves: T*K*2^F x L x 2. */
int bl_ert_upload(bl_ctx* ctx, int L, int T, int K, int F, double shrinkage, const double* mean_xy,
                  const int32_t* anchors, const double* split_params, const double* leaves);

/* Share src's uploaded detector and/or ERT model with dst (same device): one device copy
 * serves every context of a process (e.g. the C++ drop-in's per-thread contexts).  Models are
 * immutable once uploaded; a later upload on either context replaces only that context's
 * model.  BL_ERR_STATE while dst has uncollected batches. */
#define BL_SHARE_DETECTOR 1
#define BL_SHARE_ERT 2
int bl_ctx_share_models(bl_ctx* dst, bl_ctx* src, int what);

/* --------------------------------------------------------------- hot path ---- */
/* replaces: detect_faces (detector.hpp:87, detector.cpp:157-176), batched over n frames of
 * equal size.  Frame i starts at frames + i*frame_stride elements; rows are `pitch`
 * elements apart.  Kept detections of all frames are written back to back into `out`
 * (capacity `cap` entries) in each frame's NMS order; counts[i] = detections of frame i.
 * *total (optional) = sum of counts.  BL_ERR_CAPACITY if cap is too small. */
int bl_detect(bl_ctx* ctx, const void* frames, int pixel_type, int n, int w, int h, size_t pitch,
              size_t frame_stride, bl_detection* out, int64_t cap, int32_t* counts, int64_t* total);

/* replaces: predict_landmarks (ert.hpp:86-87, ert.cpp:99-136), batched over boxes.
 * out_xy: n_boxes x L x 2 image-pixel coordinates; leaf_idx (optional): n_boxes x T*K. */
int bl_landmarks(bl_ctx* ctx, const void* frames, int pixel_type, int n_frames, int w, int h,
                 size_t pitch, size_t frame_stride, const int32_t* frame_of_box, const bl_box* boxes,
                 int64_t n_boxes, double* out_xy, uint8_t* leaf_idx);

/* replaces: the per-frame detect_frame + landmark_frame pair (pipeline.cpp:159-190): detect,
 * then landmark every kept detection, all on the device.  landmarks: cap x L x 2, aligned
 * with `out`. */
int bl_detect_landmarks(bl_ctx* ctx, const void* frames, int pixel_type, int n, int w, int h,
                        size_t pitch, size_t frame_stride, bl_detection* out, int64_t cap,
                        int32_t* counts, int64_t* total, double* landmarks);

/* Pipelined mode (the paper's pipelined CPU/GPU model; the reference's
 * pipelined run(), pipeline.cpp:230-324): bl_submit enqueues a batch (H2D of host frames on
 * a copy stream, the whole detect [+ landmark] pipeline on the compute stream, result
 * metadata back) and returns at once; bl_collect waits for it and copies its results out
 * exactly like bl_detect / bl_detect_landmarks.  Up to BL_MAX_IN_FLIGHT batches may be in
 * flight, so later batches' H2D, the landmark cascade of an earlier one (its own stream) and
 * result copies overlap detection.  Tickets are collected in submission order. */
#define BL_MAX_IN_FLIGHT 4
/* with_landmarks: 0 = detection only; BL_LANDMARKS_ALL = every kept detection (landmarks of
 * bl_collect aligned with `out`); BL_LANDMARKS_BEST = the first (best) detection of each frame
 * only, as the reference's run() does (pipeline.cpp:167-190): bl_collect's landmarks then hold
 * one row per FRAME (n x L x 2), rows of frames without a detection undefined. */
#define BL_LANDMARKS_ALL 1
#define BL_LANDMARKS_BEST 2
int bl_submit(bl_ctx* ctx, const void* frames, int pixel_type, int n, int w, int h, size_t pitch,
              size_t frame_stride, int with_landmarks, uint64_t* ticket);
int bl_collect(bl_ctx* ctx, uint64_t ticket, bl_detection* out, int64_t cap, int32_t* counts,
               int64_t* total, double* landmarks);
/* Device capacity of landmarked faces per frame for the landmark pipelines (default 64); the
 * synchronous calls grow it automatically, bl_collect reports BL_ERR_CAPACITY. */
int bl_ctx_set_face_capacity(bl_ctx* ctx, int faces_per_frame);
int bl_ctx_get_face_capacity(bl_ctx* ctx, int* faces_per_frame);
/* Page-locked host memory (cudaMallocHost) for frames and results: H2D / D2H then run at full
 * PCIe rate and overlap device work. */
int bl_host_alloc(size_t bytes, void** out);
void bl_host_free(void* p);

/* ------------------------------------------------------------- multi-device ---- */
/* Frame sharding over several GPUs in one process (replaces the reference's
 * frame-parallel worker pool, pipeline.cpp:230-324, with one worker per device).  One context
 * per listed device (a device may be listed more than once), each driven by its own host
 * thread.  Frames are independent: a batch is split into contiguous per-device shards (sizes
 * differ by at most one, lower slots take the extra frame), every device runs detect +
 * landmarks on its shard through bl_submit/bl_collect with its own model replica, and the
 * results are gathered in frame order.  No collective: the gather is on the host. */
typedef struct bl_multi bl_multi;
int bl_multi_create(const int* devices, int n_devices, bl_multi** out);
void bl_multi_destroy(bl_multi* m);
int bl_multi_size(bl_multi* m, int* n_devices);
/* The context of device slot i (configuration, model files via bl_ert_file_upload). */
int bl_multi_context(bl_multi* m, int i, bl_ctx** ctx);
/* Frames per submitted batch = max(1, pixels_per_submit / (w*h)) (default 160 Mi pixels). */
int bl_multi_set_batch_pixels(bl_multi* m, int64_t pixels_per_submit);
/* Replicate a model to every device (arguments as bl_detector_upload / bl_ert_upload). */
int bl_multi_detector_upload(bl_multi* m, const double* weights, const double* biases, double threshold,
                             int window_cells, int cell_px, int scale_num, int scale_den,
                             double min_face_ratio);
int bl_multi_ert_upload(bl_multi* m, int L, int T, int K, int F, double shrinkage, const double* mean_xy,
                        const int32_t* anchors, const double* split_params, const double* leaves);
/* replaces: detect_frame + landmark_frame over a frame sequence (pipeline.cpp:159-190,
 * 230-324).  Outputs exactly as bl_detect_landmarks (landmarks NULL = detection only).
 * device_ms (optional, n_devices): wall time of each device's shard. */
int bl_multi_detect_landmarks(bl_multi* m, const void* frames, int pixel_type, int n, int w, int h,
                              size_t pitch, size_t frame_stride, bl_detection* out, int64_t cap,
                              int32_t* counts, int64_t* total, double* landmarks, double* device_ms);

/* ----------------------------------------------------------- stage functions ---- */
/* Device implementations of the reference's stage API, for the drop-in C++ layer and the
 * per-stage parity tests.  All buffers may be host or device memory. */

/* replaces: build_pyramid (image.hpp:43, image.cpp:158-172).  Levels are written back to
 * back as doubles into out (capacity out_cap doubles; may be NULL to query); dims[2k..2k+1]
 * = level k's (w,h); scales[k] = (5/6)^k.  *n_levels receives the level count. */
int bl_build_pyramid(bl_ctx* ctx, const void* image, int pixel_type, int w, int h, int window,
                     double* out, size_t out_cap, int* dims, double* scales, int max_levels,
                     int* n_levels);
/* replaces: downscale_bilinear (image.hpp:33, image.cpp:129-156). */
int bl_downscale_bilinear(bl_ctx* ctx, const double* image, int w, int h, double* out);
/* replaces: compute_gradients (hog.hpp:65, hog.cpp:28-56). */
int bl_compute_gradients(bl_ctx* ctx, const double* image, int w, int h, uint8_t* orientation,
                         double* magnitude);
/* replaces: histogramize (hog.hpp:70, hog.cpp:58-90) on an arbitrary gradient field. */
int bl_histogramize(bl_ctx* ctx, const uint8_t* orientation, const double* magnitude, int w, int h,
                    double* bins);
/* replaces: cell_energy (hog.hpp:73, hog.cpp:92-109). */
int bl_cell_energy(bl_ctx* ctx, const double* bins, int cells_w, int cells_h, double* energy);
/* replaces: compute_features (hog.hpp:75, hog.cpp:111-166). */
int bl_compute_features(bl_ctx* ctx, const double* bins, const double* energy, int cells_w,
                        int cells_h, double* features);
/* replaces: extract_features (hog.hpp:78, hog.cpp:168-173): the fused gradHist + feature
 * kernels on one image; bins/energy may be NULL. */
int bl_extract_features(bl_ctx* ctx, const double* image, int w, int h, double* features,
                        double* bins, double* energy);
/* replaces: score_separable / score_dense (detector.hpp:72-78, detector.cpp:45-100).
 * scores: (cells_h-9) x (cells_w-9), bit-identical to score_separable. */
int bl_score_window(bl_ctx* ctx, const double* features, int cells_w, int cells_h,
                    const double* weights, double bias, double* scores);
/* replaces: score_dense (detector.hpp:72-74, detector.cpp:45-64): the definitional order (one
 * accumulator over all 3100 terms), bit-identical to the reference's score_dense. */
int bl_score_window_dense(bl_ctx* ctx, const double* features, int cells_w, int cells_h,
                          const double* weights, double bias, double* scores);
/* replaces: nms (detector.hpp:80, detector.cpp:124-142).  *kept = kept count. */
int bl_nms(bl_ctx* ctx, const bl_detection* dets, int64_t n, double iou_threshold,
           bl_detection* out, int64_t* kept);
/* Device orientation argmax on explicit (gx, gy) pairs (hog.cpp:41-49 semantics). */
int bl_orientation_bins(bl_ctx* ctx, const double* gx, const double* gy, int64_t n, uint8_t* bins);

/* Self-check of the device gradient-magnitude square root (sqrt_fast, bl_hog.cu) against
 * IEEE __dsqrt_rn on the same inputs (inputs in [1e-300, 1e300]). */
int bl_debug_sqrt(bl_ctx* ctx, const double* in, int64_t n, double* fast, double* ieee);
/* Raw tcgen05 screen sums (filter r, without bias) of every anchor of one feature image
 * (cells_w x cells_h x 31 doubles) against the uploaded detector: scores[r][sh][sw], with
 * the rigorous per-filter error bound the candidate cut uses in delta[r]. */
int bl_debug_screen_tc(bl_ctx* ctx, const double* features, int cells_w, int cells_h, float* scores,
                       double* delta);

/* ---------------------------------------------------- data formats (host only) ---- */
/* Frames.  replaces: load_pgm (image.hpp:25, image.cpp:67-114).  P5 or P2, maxval <= 255,
 * parsed straight to u8 (exact: PGM samples are integers).  pixels == NULL: header only
 * (dimensions).  Errors: BL_ERR_IO with the reference's message and byte offset. */
int bl_read_pgm(const char* path, int* w, int* h, uint8_t* pixels, size_t capacity);
/* replaces: save_pgm (image.hpp:28, image.cpp:116-127): P5, values clamped and rounded. */
int bl_write_pgm(const char* path, const double* pixels, int w, int h);

/* Detector model file "hog-v1".  replaces: load_detector_model / save_model
 * (detector.hpp:99-100, detector.cpp:291-351).  weights: 5 x window_cells^2 x 31 doubles
 * (filter-major, the bl_detector_upload layout); NULL -> scalars only (call once for
 * window_cells, again with buffers).  Errors: BL_ERR_IO (cannot open), BL_ERR_MODEL. */
int bl_read_detector_json(const char* path, double* weights, double* biases, double* threshold,
                          int* window_cells, int* cell_px, int* scale_num, int* scale_den,
                          double* min_face_ratio);
int bl_write_detector_json(const char* path, const double* weights, const double* biases,
                           double threshold, int window_cells, int cell_px, int scale_num,
                           int scale_den, double min_face_ratio);

/* ERT model file "ert-v1".  replaces: load_ert_model / save_model (ert.hpp:128-129,
 * ert.cpp:358-469).  Open parses once into the bl_ert_upload layout (anchors [T][K][S][2],
 * split_params [T][K][S][5] = ox_a, oy_a, ox_b, oy_b, thr, leaves [T][K][2^F][L][2]); copy
 * the arrays out, or upload them to a context, then close. */
typedef struct bl_ert_file bl_ert_file;
int bl_ert_file_open(const char* path, bl_ert_file** out, int* L, int* T, int* K, int* F,
                     double* shrinkage);
int bl_ert_file_copy(const bl_ert_file* file, double* mean_xy, int32_t* anchors, double* split_params,
                     double* leaves);
int bl_ert_file_upload(const bl_ert_file* file, bl_ctx* ctx);
void bl_ert_file_close(bl_ert_file* file);
int bl_write_ert_json(const char* path, int L, int T, int K, int F, double shrinkage,
                      const double* mean_xy, const int32_t* anchors, const double* split_params,
                      const double* leaves);

/* -------------------------------------------------- frame-sequence runtime ---- */
/* One frame of a run (pipeline.hpp:41-47 FrameResult + blink.hpp:20-28 BlinkSample). */
typedef struct {
  int32_t frame_index;
  int32_t n_detections;  /* this frame's post-NMS detections, consecutive in `dets` */
  int32_t face_found;    /* the frame has a face: its first (best) detection */
  int32_t pad;
  bl_detection face;
  double ear_left, ear_right;          /* valid iff face_found */
  double closure_left, closure_right;  /* valid iff face_found */
  double t;                            /* frame_index / fps */
  double decode_ms, detect_ms, landmark_ms;
} bl_frame_result;

/* Landmark count of the context's ERT model (BL_ERR_STATE when none is uploaded). */
int bl_ctx_model_info(bl_ctx* ctx, int* landmark_count);
/* replaces: ingest (pipeline.hpp:33, pipeline.cpp:358-394): frame_%06d.pgm numbered from 0
 * without gaps, all with equal dimensions (read from the headers). */
int bl_ingest(const char* frames_dir, int* n_frames, int* w, int* h);
/* replaces: run (pipeline.hpp:59-60, pipeline.cpp:396-404) with the uploaded detector and
 * ERT model: decode -> detect -> landmark the best detection of each frame -> EAR -> blink
 * trace (blink.cpp:47-93, baseline quantile 0.95), in batches of batch_size frames on the
 * device (1 = the reference's sequential mode; results identical for any batch size).
 * frames[n_frames]; dets receives every frame's detections in frame order (det_cap);
 * landmarks[n_frames][L][2] (rows of frames without a face are untouched);
 * baselines[2] = left / right EAR baselines. */
int bl_run(bl_ctx* ctx, const char* frames_dir, double fps, int batch_size, bl_frame_result* frames,
           int64_t frames_cap, bl_detection* dets, int64_t det_cap, int64_t* det_total, double* landmarks,
           double* baselines);

#ifdef __cplusplus
}
#endif
#endif /* BLINKLINE_B200_H */
