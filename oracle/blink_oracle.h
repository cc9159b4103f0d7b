/* TEST INFRASTRUCTURE ONLY -- the CPU oracle for the face + landmark hot path.
 *
 * A plain-C restatement of the reference algorithm (blinkline, /root/reference/proj),
 * following its operation order exactly so that, compiled without FP contraction
 * (oracle/Makefile), it is bit-identical to the reference.  Pinned against golden
 * vectors produced by the unmodified reference (tests/golden/, oracle/make_golden.py)
 * and against the reference's own known-answer cases (tests/test_oracle_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this
 * library, and only as the checker.  The product (paper_2006_00816_b200/) never links it.
 *
 * Layouts are the reference's: row-major pixels; cell-major bins (cy, cx, 18) and
 * features (cy, cx, 31); filters (5, 10, 10, 31) row-major; detections laid out like
 * blinkline::Detection (detector.hpp:52-57). */
#ifndef BLINK_ORACLE_H
#define BLINK_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t x, y, w, h;
  double score;
  int32_t scale_index, rotation_index;
} orc_det;

typedef struct {
  const double* weights; /* 5 x 3100 */
  const double* biases;  /* 5 */
  double threshold;
  int window_cells, cell_px, scale_num, scale_den;
  double min_face_ratio;
} orc_detector;

typedef struct {
  int L, T, K, F;
  double shrinkage;
  const double* mean_xy;      /* L x 2 */
  const int32_t* anchors;     /* T*K*S x 2   (S = 2^F - 1) */
  const double* split_params; /* T*K*S x 5   (oax, oay, obx, oby, thr) */
  const double* leaves;       /* T*K*2^F x L x 2 */
} orc_ert;

/* image.cpp:129-172 */
int orc_downscale_bilinear(const double* px, int w, int h, double* out);
int orc_build_pyramid(const double* px, int w, int h, int window, double* out, size_t out_cap,
                      int* dims, double* scales, int max_levels);
/* hog.cpp:12-173 */
void orc_direction_table(double* ux, double* uy);
int orc_compute_gradients(const double* px, int w, int h, uint8_t* ori, double* mag);
int orc_histogramize(const uint8_t* ori, const double* mag, int w, int h, double* bins);
int orc_cell_energy(const double* bins, int cw, int ch, double* energy);
int orc_compute_features(const double* bins, const double* energy, int cw, int ch, double* feat);
int orc_extract_features(const double* px, int w, int h, double* feat);
/* detector.cpp:16-176 */
double orc_iou(int ax, int ay, int aw, int ah, int bx, int by, int bw, int bh);
int orc_score_dense(const double* feat, int cw, int ch, const double* weights, double bias,
                    double* scores);
int orc_score_separable(const double* feat, int cw, int ch, const double* weights, double bias,
                        double* scores);
int orc_threshold_detections(const double* scores, int sw, int sh, double thr, int window_cells,
                             int cell_px, int scale_num, int scale_den, int scale_index,
                             int rotation_index, orc_det* out, int cap);
int orc_nms(const orc_det* in, int n, double iou_thr, orc_det* out);
int orc_eligible_scales(int w, int h, int window_cells, int cell_px, int scale_num, int scale_den,
                        double min_face_ratio, int n_levels, int* out);
int orc_detect_faces(const double* px, int w, int h, const orc_detector* m, orc_det* out, int cap);
/* ert.cpp:15-136 */
int orc_similarity_transform(const double* from_xy, const double* to_xy, int L, double* out4);
double orc_sample_intensity(const double* px, int w, int h, int bx, int by, int bw, int bh,
                            const double* shape_xy, const double* tform4, int anchor, double ox,
                            double oy);
int orc_predict_landmarks(const double* px, int w, int h, int bx, int by, int bw, int bh,
                          const orc_ert* m, double* out_xy, uint8_t* leaf_idx, uint64_t* evals);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
