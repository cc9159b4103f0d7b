// Host side of blinkline_b200: device contexts, batch plans (geometry + pre-sized device
// arenas, the paper's "allocate once" scheme), the per-batch pipeline
// and every extern "C" entry point of include/blinkline_b200.h.
//
// No computation of the hot path happens on the host: the host computes geometry
// (pyramid dims, eligibility, per-level scale constants -- with the same libm calls the
// reference makes, so the constants are bit-identical) and launches kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "bl_internal.cuh"

using namespace blb;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

}  // namespace

namespace blb {
// The thread-local error message, for the host-only translation units (bl_io.cpp).
void set_last_error(const char* msg) { g_err = msg; }
}  // namespace blb

namespace {

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return set_err(BL_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                     __FILE__, __LINE__);                                                 \
  } while (0)

#define TRY(call)              \
  do {                         \
    int rc_ = (call);          \
    if (rc_ != BL_OK) return rc_; \
  } while (0)

// Bumped by every device (re)allocation: a captured CUDA graph bakes buffer addresses into its
// kernel arguments, so a graph captured before the latest allocation is recaptured.
std::atomic<uint64_t> g_alloc_epoch{1};

// Device buffer that only grows.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int device = -1;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) {
      int cur = 0;
      cudaGetDevice(&cur);
      if (device >= 0 && device != cur) cudaSetDevice(device);
      cudaFree(p);
      if (device >= 0 && device != cur) cudaSetDevice(cur);
    }
    p = nullptr;
    bytes = 0;
  }
  int ensure(size_t n, bool zero = false) {
    if (n <= bytes && p) return BL_OK;
    release();
    const size_t alloc = std::max<size_t>(n, 256);
    cudaError_t e = cudaMalloc(&p, alloc);
    if (e != cudaSuccess) {
      p = nullptr;
      return set_err(BL_ERR_CUDA, "cudaMalloc(%zu) failed: %s", alloc, cudaGetErrorString(e));
    }
    cudaGetDevice(&device);
    bytes = alloc;
    g_alloc_epoch.fetch_add(1);
    if (zero) {
      e = cudaMemset(p, 0, alloc);
      if (e != cudaSuccess) return set_err(BL_ERR_CUDA, "cudaMemset failed: %s", cudaGetErrorString(e));
    }
    return BL_OK;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int round_half_up_host(double v) { return int(std::floor(v + 0.5)); }  // detector.cpp:41

constexpr int kLevelMargin = 8;  // readable doubles either side of every arena level row

// Round a double to the nearest fp16 (ties to even, like cvt.rn.f16.f64); |x| < 65520.
uint16_t half_rn_host(double x) {
  const uint16_t sign = std::signbit(x) ? 0x8000 : 0;
  const double a = std::fabs(x);
  if (std::isnan(x)) return 0x7e00;
  if (a >= 65520.0) return (uint16_t)(sign | 0x7c00);  // rounds to infinity
  if (a == 0.0) return sign;
  int e = 0;
  std::frexp(a, &e);  // a = m 2^e, m in [0.5, 1): binade exponent e - 1
  if (e - 1 < -14) {  // subnormal: quantum 2^-24
    const double q = std::nearbyint(std::ldexp(a, 24));
    return (uint16_t)(sign | (uint16_t)q);  // q = 1024 encodes the smallest normal
  }
  double q = std::nearbyint(std::ldexp(a, 11 - e));  // 11 significant bits, in [1024, 2048]
  if (q == 2048.0) {
    q = 1024.0;
    ++e;
  }
  return (uint16_t)(sign | (uint16_t)((e - 1 + 15) << 10) | (uint16_t)((int)q - 1024));
}

struct DetectorState {
  bool ready = false;
  double thr = 0;
  int window_cells = 10, cell_px = 8, scale_num = 5, scale_den = 6;
  double min_face_ratio = 0.2;
  double bias[kFilters] = {0};
  float cut[kFilters] = {0};
  float cut_tc[2 * kFilters] = {0};  // [0, 5): cut in the screen's scaled domain, [5, 10): 2^-scale
  double delta_tc[kFilters] = {0};
  DevBuf w64, w64t, w32, bias64, cut32, w_tc, cuttc;
};

struct ErtState {
  bool ready = false;
  ErtDev dev{};
  DevBuf mean, mean_c, split, leaves;
};

// A batch plan: geometry + device arenas for (n, w, h, pixel type, detector geometry).
struct Plan {
  bool valid = false;
  int n = 0, w = 0, h = 0, pix = 0;
  int window = 80, cell_px = 8, window_cells = 10, scale_num = 5, scale_den = 6;
  double min_face_ratio = 0.2;
  int screen = BL_SCREEN_TCGEN05;
  int n_levels = 0;
  std::vector<int> lw, lh;
  std::vector<long long> arena_off;  // levels >= 1, in doubles
  std::vector<int> lpitch;           // levels >= 1: row pitch in doubles (multiple of 4)
  long long arena_elems = 0;
  std::vector<int> scored;           // pyramid level of each scored slot
  PlanDesc host{};
  DevBuf desc;
  long long cap_pf = 0;              // raw detections per frame (all anchors x 5 filters)
  long long cand_cap = 0;
  long long f32_elems = 0;
  long long gkeys_pf = 0;
  DevBuf arena, bins, energy, feat64, feat32, feat_tc, cand, n_cand, dets, det_count, kept, kept_count, gkeys,
      overflow, offsets;
  // level 0's gradHist reads only the caller's frames: it runs on `aux` beside the pyramid
  // (fork / join events, capturable into the batch's graph)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

// ERT cascade working set (current shapes, per-level transforms, leaf-index scratch).
struct ErtWork {
  DevBuf cur, tf, leafs;
};

// One in-flight batch: its staged input, its device results and pinned host mirrors.
// BL_MAX_IN_FLIGHT slots let later batches' H2D and detection overlap an earlier batch's
// landmark cascade and result copies (bl_submit/collect).
struct Slot {
  DevBuf input, flat, face_frame, meta, ert_out, best, best_frame;
  ErtWork ert;                  // the slot's cascade runs on the ERT stream, beside the next detect
  cudaEvent_t ev_det = nullptr; // detections flattened: the ERT stream may start
  int* h_meta = nullptr;
  size_t h_meta_cap = 0;
  void* h_stage = nullptr;
  size_t h_stage_cap = 0;
  cudaEvent_t ev_h2d = nullptr, ev_done = nullptr, ev_meta = nullptr, ev_out = nullptr;
  cudaStream_t d2h = nullptr;  // this slot's result copies: never queued behind the other slot
  // this slot's landmark cascade (lowest priority): overlaps the next batches' detection and,
  // at small batches where one cascade fills few SMs, the other slots' cascades
  cudaStream_t est = nullptr;
  bool busy = false;
  bool eager = false;  // results copied to h_stage with the counts (small batches: one wait)
  int n = 0, w = 0, h = 0, pix = 0, landmarks = 0;
  long long cap_faces = 0;
  uint64_t ticket = 0;
};

}  // namespace

// Detection lanes (plan arenas + compute stream): consecutive in-flight batches rotate over
// them so their detection stages overlap.  Two lanes saturate the GPU at large batches (the
// bench's 512 frames: 3-4 lanes measured 1-3% slower); small, latency-bound batches (up to
// kSmallBatchPx pixels, e.g. the 16-frame camera stream) rotate over all four.
constexpr int kLanes = 4;
constexpr int kLanesLarge = 2;
constexpr long long kSmallBatchPx = 16LL << 20;
constexpr long long kChainMaxPx = 1LL << 19;  // batches up to this many pixels: k_pyramid_chain (C1 yes, C2 no: measured)

struct bl_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t st = nullptr;
  std::mutex mu;
  uint64_t launches = 0;
  // Models: immutable once uploaded and shared between contexts on one device
  // (bl_ctx_share_models); an upload replaces the context's pointer, sharers keep theirs.
  std::shared_ptr<DetectorState> detp = std::make_shared<DetectorState>();
  std::shared_ptr<ErtState> ertp = std::make_shared<ErtState>();
  // Detection lanes (plan arenas + compute stream, see kLanes): consecutive in-flight batches
  // rotate over them, so batch i+1's pyramid / gradHist overlap batch i's later stages.
  // Lane 0 runs on the caller's stream (c->user); `plan` / `st` point at the active lane.
  Plan plans[kLanes];
  Plan* plan = &plans[0];
  cudaStream_t lanes[kLanes] = {};  // lanes[0] unused: lane 0 runs on `user`
  cudaStream_t user = nullptr;
  cudaEvent_t ev_lane = nullptr;
  // ERT working set
  ErtWork ert_work;  // bl_landmarks' cascade (on the compute stream)
  DevBuf ert_out, ert_leaf, ert_boxes, ert_frames, ert_nfaces, ert_err, ert_input;
  // scratch for stage functions
  DevBuf s_a, s_b, s_c, s_d, s_e, s_desc;
  bool timing = false;
  cudaEvent_t ev[BL_STAGE_COUNT + 1] = {};
  float stage_ms[BL_STAGE_COUNT] = {};
  int stage_launch[BL_STAGE_COUNT] = {};
  bool graphs = true;
  bool ert_serial = false;          // BL_ERT_SERIAL=1: the cascade on the lane stream (experiment)
  bool ert_conc = false;            // BL_ERT_CONC=1: large batches' cascades concurrent again (experiment)
  bool h2d_after_ert = true;        // BL_H2D_AFTER_ERT=0: large inputs copied as soon as their slot is free (A/B)
  int lanes_large = kLanesLarge;    // BL_LANES_LARGE: detection lanes for large batches (experiment)
  cudaStream_t hst = nullptr;  // H2D stream (input frames): never queued behind a D2H wait
  // CUDA graphs (bl_ctx_enable_graphs): a batch's detection launches (one graph per lane plan,
  // slot and input) and its landmark cascade (one per slot and input) are captured once on a
  // private stream and replayed; host submit then costs a few graph/event calls instead of
  // ~60 launches.  Entries are keyed by everything baked into the kernel arguments.
  struct GraphEntry {
    int kind = 0;  // 0: detection + flatten, 1: landmark cascade
    const void* plan = nullptr;
    int slot = 0;
    const void* in = nullptr;
    long long dp = 0, df = 0, cap_faces = 0;
    int n = 0, w = 0, h = 0, pix = 0, landmarks = 0;
    uint64_t epoch = 0, model_gen = 0, last_use = 0;
    uint64_t kernels = 0;
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<GraphEntry> gcache;
  cudaStream_t cap = nullptr;
  uint64_t model_gen = 1, use_clock = 0;
  Slot slots[BL_MAX_IN_FLIGHT];
  uint64_t next_ticket = 1;
  int face_cap_per_frame = 64;  // device-side capacity of landmarked faces per frame
  int screen = BL_SCREEN_TCGEN05;
  // landmark cascade kernel: auto (k_ert_wide for small batches, else k_ert_cascade), or forced
  // by BL_ERT=wide|cascade|levels (experiments)
  int ert_mode = 0;
  int ert_cl = 0;  // BL_ERT_CL=1|2|4|8: forces the small-batch cascade's cluster size (A/B, tests)
  bool pyr_fuse = true;  // fused resample pairs over unscored levels (BL_PYR_FUSE=0 disables)
  bool pyr_chain = true;  // one cooperative launch for a small batch's chain (BL_PYR_CHAIN=0 disables)
};

namespace {

Launch launch_of(bl_ctx* c) { return Launch{c->st, &c->launches}; }

int use_device(bl_ctx* c) {
  CK(cudaSetDevice(c->device));
  return BL_OK;
}

// -------------------------------------------------------------------- geometry ----
// image.cpp:158-172 (level dims) ; detector.cpp:144-155 (eligibility) ; detector.cpp:163-167.
void pyramid_dims(int w, int h, int window, std::vector<int>& lw, std::vector<int>& lh) {
  lw.assign(1, w);
  lh.assign(1, h);
  while (true) {
    const int cw = lw.back(), chh = lh.back();
    if (cw < 2 || chh < 2) break;
    const int nw = cw * 5 / 6, nh = chh * 5 / 6;
    if (nw < window || nh < window) break;
    lw.push_back(nw);
    lh.push_back(nh);
  }
}

int build_plan(bl_ctx* c, Plan& P, int n, int w, int h, int pix) {
  const DetectorState& D = (*c->detp);
  if (P.valid && P.n == n && P.w == w && P.h == h && P.pix == pix && P.screen == c->screen &&
      P.window_cells == D.window_cells &&
      P.cell_px == D.cell_px && P.scale_num == D.scale_num && P.scale_den == D.scale_den &&
      P.min_face_ratio == D.min_face_ratio)
    return BL_OK;
  P.valid = false;
  P.n = n;
  P.w = w;
  P.h = h;
  P.pix = pix;
  P.screen = c->screen;
  P.window_cells = D.window_cells;
  P.cell_px = D.cell_px;
  P.scale_num = D.scale_num;
  P.scale_den = D.scale_den;
  P.min_face_ratio = D.min_face_ratio;
  P.window = D.window_cells * D.cell_px;
  pyramid_dims(w, h, P.window, P.lw, P.lh);
  P.n_levels = (int)P.lw.size();
  if (P.n_levels > kMaxLevels) return set_err(BL_ERR_INVALID, "pyramid deeper than %d levels", kMaxLevels);
  P.arena_off.assign(P.n_levels, 0);
  P.lpitch.assign(P.n_levels, 0);
  long long off = 0;
  // level rows: 8-element margins either side and a pitch of a multiple of 4 doubles, so
  // k_hog reads 16-B aligned 8-pixel groups straddling the image edge without clamping
  for (int k = 1; k < P.n_levels; ++k) {
    P.lpitch[k] = (int)div_up(P.lw[k] + 2 * kLevelMargin, 4) * 4;
    P.arena_off[k] = off + kLevelMargin;
    off += (long long)n * P.lpitch[k] * P.lh[k];
  }
  off += 2 * kLevelMargin;
  P.arena_elems = off;

  // eligible_scales (detector.cpp:144-155) + the "room for a window" skip (:165-167)
  const double min_face = D.min_face_ratio * std::min(w, h);
  P.scored.clear();
  for (int k = 0; k < P.n_levels; ++k) {
    const double detectable =
        P.window / std::pow(double(D.scale_num) / D.scale_den, double(k));
    if (!(detectable >= min_face * (1.0 - 1e-9))) continue;
    if (P.lw[k] / D.cell_px < D.window_cells || P.lh[k] / D.cell_px < D.window_cells) continue;
    if (P.lw[k] / 8 < kWin || P.lh[k] / 8 < kWin)
      return set_err(BL_ERR_INVALID, "feature image smaller than the 10x10 detection window");
    P.scored.push_back(k);
  }
  PlanDesc& H = P.host;
  std::memset(&H, 0, sizeof H);
  H.n_frames = n;
  H.n_scored = (int)P.scored.size();
  long long cells = 0, gh = 0, sc = 0, f32 = 0, anchors_pf = 0, fld = 0, gr = 0, ftc = 0;
  for (int s = 0; s < H.n_scored; ++s) {
    const int k = P.scored[s];
    LevelDesc& L = H.lv[s];
    L.w = P.lw[k];
    L.h = P.lh[k];
    L.cw = L.w / 8;
    L.ch = L.h / 8;
    L.sw = L.cw - (kWin - 1);
    L.sh = L.ch - (kWin - 1);
    L.level = k;
    L.c = std::pow(double(D.scale_num) / D.scale_den, double(k));  // detector.cpp:104
    L.side = round_half_up_host(P.window / L.c);                    // detector.cpp:105
    if (k == 0) {
      L.pix_off = 0;  // patched per call (input pointer)
      L.pix_fstride = 0;
      L.pix_pitch = 0;
    } else {
      L.pix_off = P.arena_off[k];
      L.pix_fstride = (long long)P.lpitch[k] * L.h;
      L.pix_pitch = P.lpitch[k];
      L.pix_margin = kLevelMargin;
    }
    L.cell_off = cells;
    L.cell_begin = cells;
    cells += (long long)n * L.cw * L.ch;
    {  // screening tile shape with the least padding
      long long best = -1;
      for (int lx : {8, 4, 2}) {
        const long long tw = 4 * lx, th = 32 / lx;
        const long long area = div_up(L.sw, tw) * tw * div_up(L.sh, th) * th;
        if (best < 0 || area < best) {
          best = area;
          L.sc_lanes_x = lx;
        }
      }
    }
    const int tile_w = 4 * L.sc_lanes_x, tile_h = 32 / L.sc_lanes_x;
    L.cw_pad = (int)(div_up(L.sw, tile_w) * tile_w + 12);
    L.ch_pad = (int)(div_up(L.sh, tile_h) * tile_h + (kWin - 1));
    L.f32_off = f32;
    L.f32_fstride = (long long)kFeatPad * L.ch_pad * L.cw_pad;
    f32 += (long long)n * L.f32_fstride;
    L.tc_off = ftc;
    ftc += (long long)n * (long long)tc_feat_floats_per_frame(L.cw, L.ch, &L.tc_ncp, nullptr);
    L.fld_off = fld;
    fld += (long long)n * L.w * L.h;
    L.gr_tiles_x = (int)div_up(L.w, 32);
    L.gr_tiles_y = (int)div_up(L.h, 64);
    L.gr_begin = gr;
    gr += (long long)n * L.gr_tiles_x * L.gr_tiles_y;
    L.gh_tiles_x = (int)div_up(L.cw, kGhCells);
    L.gh_tiles_y = (int)div_up(L.ch, kGhSegRows);
    L.gh_begin = gh;
    gh += (long long)n * L.gh_tiles_x * L.gh_tiles_y;
    L.sc_tiles_x = (int)div_up(L.sw, tile_w);
    L.sc_tiles_y = (int)div_up(L.sh, tile_h);
    L.sc_begin = sc;
    sc += (long long)n * L.sc_tiles_x * L.sc_tiles_y;
    L.anchor_base = anchors_pf;
    anchors_pf += (long long)L.sw * L.sh;
  }
  H.gh_total = gh;
  H.gr_total = gr;
  H.fld_total = fld;
  H.sc_total = sc;
  H.cell_total = cells;
  H.cells_per_frame = n ? cells / n : 0;
  P.f32_elems = f32;
  P.cap_pf = std::max<long long>(1, anchors_pf * kFilters);
  P.cand_cap = std::max<long long>(1, (long long)n * anchors_pf);  // one per anchor (filter mask)
  P.gkeys_pf = nms_gkeys_per_frame(P.cap_pf);

  TRY(P.desc.ensure(sizeof(PlanDesc)));
  TRY(P.arena.ensure(sizeof(double) * std::max<long long>(1, P.arena_elems)));
  TRY(P.bins.ensure(sizeof(double) * kBins * std::max<long long>(1, cells)));
  TRY(P.energy.ensure(sizeof(double) * std::max<long long>(1, cells)));
  TRY(P.feat64.ensure(sizeof(double) * kFeat * std::max<long long>(1, cells)));
  // zero once: the padding of the fp32 planes is never written by the feature kernel
  if (P.screen == BL_SCREEN_FP32) {
    const bool regrow = P.feat32.bytes < sizeof(float) * (size_t)std::max<long long>(1, f32);
    TRY(P.feat32.ensure(sizeof(float) * std::max<long long>(1, f32), true));
    if (!regrow) CK(cudaMemset(P.feat32.p, 0, sizeof(float) * std::max<long long>(1, f32)));
  } else {  // the zero tail of each tc plane is never written by the feature kernel
    const bool regrow = P.feat_tc.bytes < sizeof(float) * (size_t)std::max<long long>(1, ftc);
    TRY(P.feat_tc.ensure(sizeof(float) * std::max<long long>(1, ftc), true));
    if (!regrow) CK(cudaMemset(P.feat_tc.p, 0, sizeof(float) * std::max<long long>(1, ftc)));
  }
  TRY(P.cand.ensure(sizeof(Candidate) * P.cand_cap));
  TRY(P.n_cand.ensure(sizeof(unsigned long long)));
  TRY(P.dets.ensure(sizeof(DevDet) * n * P.cap_pf));
  TRY(P.kept.ensure(sizeof(DevDet) * n * P.cap_pf));
  TRY(P.det_count.ensure(sizeof(int) * n));
  TRY(P.kept_count.ensure(sizeof(int) * n));
  TRY(P.overflow.ensure(sizeof(int)));
  if (P.gkeys_pf) TRY(P.gkeys.ensure(nms_key_bytes() * n * P.gkeys_pf));
  TRY(P.offsets.ensure(sizeof(int) * (n + 1)));
  CK(cudaMemcpy(P.desc.p, &P.host, sizeof(PlanDesc), cudaMemcpyHostToDevice));
  P.valid = true;
  return BL_OK;
}

void stage_mark(bl_ctx* c, int stage) {
  if (c->timing) cudaEventRecord(c->ev[stage], c->st);
}

// ------------------------------------------------------------------ detection ----
// Enqueues detect on n frames already resident on the device (`in`, element pitch/stride) on
// the active lane's stream: leaves each frame's kept detections in P.kept / P.kept_count on
// the device (no host synchronisation).
// Host half of a detect batch: the plan (geometry + arenas) and the level-0 descriptor.
int prepare_detect(bl_ctx* c, int pix, int n, int w, int h, long long pitch, long long fstride) {
  Plan& P = *c->plan;
  TRY(build_plan(c, P, n, w, h, pix));
  // level 0 descriptor points at the caller's frames
  if (!P.scored.empty() && P.scored[0] == 0) {
    LevelDesc& L0 = P.host.lv[0];
    if (L0.pix_pitch != pitch || L0.pix_fstride != fstride) {
      L0.pix_off = 0;
      L0.pix_pitch = (int)pitch;
      L0.pix_fstride = fstride;
      CK(cudaMemcpyAsync(P.desc.p, &P.host, sizeof(PlanDesc), cudaMemcpyHostToDevice, c->st));
    }
  }
  return BL_OK;
}

// Device half: every launch of the detect path on c->st (capturable: no host synchronisation,
// no allocation -- prepare_detect sized the plan).
int record_detect(bl_ctx* c, const void* in, int pix, int n, long long pitch, long long fstride) {
  Plan& P = *c->plan;
  const Launch L = launch_of(c);
  const DetectorState& D = (*c->detp);
  // level 0 scored (small frames, e.g. the 320x240 camera stream): its gradHist needs only the
  // caller's frames, so it runs on the plan's side stream beside the pyramid
  const bool fork0 = !c->timing && !P.scored.empty() && P.scored[0] == 0 && P.aux;
  if (fork0) {
    CK(cudaEventRecord(P.ev_fork, c->st));
    CK(cudaStreamWaitEvent(P.aux, P.ev_fork, 0));
    launch_hog(Launch{P.aux, &c->launches}, P.host, P.desc.as<PlanDesc>(), 0, 1, in, pix == BL_PIX_U8 ? 0 : 1,
               P.bins.as<double>(), P.energy.as<double>());
    CK(cudaEventRecord(P.ev_join, P.aux));
  }
  stage_mark(c, BL_STAGE_PYRAMID);
  // pyramid chain (image.cpp:162-170): level k from level k-1, every frame at once.  A level
  // no window scores (below the smallest eligible face) is read only by the next step, so
  // the two steps run fused (k_resample_pair) and that level never reaches HBM.
  std::vector<char> is_scored(P.n_levels + 1, 0);
  for (int k : P.scored) is_scored[k] = 1;
  // small batches: the whole chain in one cooperative launch (launch latency, not bandwidth,
  // bounds a one-frame pyramid)
  const bool chain = c->pyr_chain && (long long)n * P.w * P.h <= kChainMaxPx && P.n_levels > 2;
  if (chain) {
    PyrChain C{};
    C.n_levels = P.n_levels;
    C.n_frames = n;
    C.src0 = in;
    C.s0_pitch = pitch;
    C.s0_fstride = fstride;
    for (int k = 0; k < P.n_levels; ++k) {
      C.lw[k] = P.lw[k];
      C.lh[k] = P.lh[k];
      if (k >= 1) {
        C.lv[k] = P.arena.as<double>() + P.arena_off[k];
        C.lpitch[k] = P.lpitch[k];
        C.lfstride[k] = (long long)P.lpitch[k] * P.lh[k];
        C.rx[k] = double(P.lw[k - 1]) / P.lw[k];  // image.cpp:136-137
        C.ry[k] = double(P.lh[k - 1]) / P.lh[k];
      }
    }
    C.zero_u64 = P.n_cand.as<unsigned long long>();
    C.zero_i32 = P.det_count.as<int>();
    C.n_zero_i32 = n;
    C.zero_flag = P.overflow.as<int>();
    if (const int e = launch_pyramid_chain(L, C, pix == BL_PIX_U8))
      return set_err(BL_ERR_CUDA, "pyramid chain launch failed: %s", cudaGetErrorString((cudaError_t)e));
  }
  for (int k = 1; k < P.n_levels && !chain; ++k) {
    const void* src = k == 1 ? in : (const void*)(P.arena.as<double>() + P.arena_off[k - 1]);
    const int src_u8 = (k == 1 && pix == BL_PIX_U8);
    const long long sp = k == 1 ? pitch : P.lpitch[k - 1];
    const long long sf = k == 1 ? fstride : (long long)P.lpitch[k - 1] * P.lh[k - 1];
    if (c->pyr_fuse && !is_scored[k] && k + 1 < P.n_levels &&
        resample_pair_fits(P.lw[k - 1], P.lh[k - 1], P.lw[k], P.lh[k], P.lw[k + 1], P.lh[k + 1])) {
      launch_resample_pair(L, src, src_u8, P.lw[k - 1], P.lh[k - 1], sp, sf, P.lw[k], P.lh[k],
                           P.arena.as<double>() + P.arena_off[k + 1], P.lw[k + 1], P.lh[k + 1], P.lpitch[k + 1],
                           (long long)P.lpitch[k + 1] * P.lh[k + 1], n);
      ++k;
      continue;
    }
    launch_resample(L, src, src_u8, P.lw[k - 1], P.lh[k - 1], sp, sf, P.arena.as<double>() + P.arena_off[k],
                    P.lw[k], P.lh[k], P.lpitch[k], (long long)P.lpitch[k] * P.lh[k], n);
  }
  stage_mark(c, BL_STAGE_GRADHIST);
  const PlanDesc* Pd = P.desc.as<PlanDesc>();
  const int ns = P.host.n_scored;
  if (!chain) {  // (the one-launch chain zeroes them itself)
    CK(cudaMemsetAsync(P.n_cand.p, 0, sizeof(unsigned long long), c->st));
    CK(cudaMemsetAsync(P.det_count.p, 0, sizeof(int) * n, c->st));
    CK(cudaMemsetAsync(P.overflow.p, 0, sizeof(int), c->st));
  }
  if (ns > 0) {
    // fused gradient + histogram + energy (the gradient field stays on chip)
    int s1 = 0;
    if (P.scored[0] == 0) {  // level 0 reads the caller's frames (u8 or f64)
      if (!fork0)
        launch_hog(L, P.host, Pd, 0, 1, in, pix == BL_PIX_U8 ? 0 : 1, P.bins.as<double>(), P.energy.as<double>());
      s1 = 1;
    }
    launch_hog(L, P.host, Pd, s1, ns, P.arena.as<double>(), 1, P.bins.as<double>(), P.energy.as<double>());
    if (fork0) CK(cudaStreamWaitEvent(c->st, P.ev_join, 0));
  }
  stage_mark(c, BL_STAGE_FEATURES);
  const bool tc = P.screen == BL_SCREEN_TCGEN05;
  launch_features(L, P.host, Pd, P.bins.as<double>(), P.energy.as<double>(), P.feat64.as<double>(),
                  tc ? nullptr : P.feat32.as<float>(), tc ? P.feat_tc.as<float>() : nullptr);
  stage_mark(c, BL_STAGE_SCREEN);
  if (tc)
    launch_screen_tc(L, P.host, Pd, P.feat_tc.as<float>(), D.w_tc.as<float>(), D.cuttc.as<float>(),
                     P.cand.as<Candidate>(), P.n_cand.as<unsigned long long>(), P.cand_cap, nullptr);
  else
    launch_screen(L, P.host, Pd, P.feat32.as<float>(), D.w32.as<float>(), D.cut32.as<float>(),
                  P.cand.as<Candidate>(), P.n_cand.as<unsigned long long>(), P.cand_cap);
  stage_mark(c, BL_STAGE_RESCORE);
  launch_rescore(L, n, Pd, P.feat64.as<double>(), D.w64.as<double>(), D.w64t.as<double>(), D.bias64.as<double>(), D.thr, D.cell_px,
                 P.cand.as<Candidate>(), P.n_cand.as<unsigned long long>(), P.cand_cap, P.dets.as<DevDet>(),
                 P.det_count.as<int>(), P.cap_pf, P.overflow.as<int>());
  stage_mark(c, BL_STAGE_NMS);
  launch_nms(L, P.dets.as<DevDet>(), P.det_count.as<int>(), P.cap_pf, n, 0.5, P.kept.as<DevDet>(),
             P.kept_count.as<int>(), P.gkeys.p, P.gkeys_pf);
  return BL_OK;
}

// Stage host frames into a device buffer (or use device frames in place).
int stage_input(bl_ctx* c, DevBuf& buf, const void* frames, int pix, int n, int w, int h, size_t pitch,
                size_t fstride, const void** dev, long long* dpitch, long long* dfstride) {
  const size_t es = pix == BL_PIX_U8 ? 1 : 8;
  if (is_device_ptr(frames)) {
    *dev = frames;
    *dpitch = (long long)pitch;
    *dfstride = (long long)fstride;
    return BL_OK;
  }
  TRY(buf.ensure(es * (size_t)n * w * h));
  if (pitch == (size_t)w && fstride == (size_t)w * h) {
    CK(cudaMemcpyAsync(buf.p, frames, es * (size_t)n * w * h, cudaMemcpyDefault, c->st));
  } else {
    for (int i = 0; i < n; ++i)
      CK(cudaMemcpy2DAsync((char*)buf.p + es * (size_t)i * w * h, es * w,
                           (const char*)frames + es * fstride * i, es * pitch, es * w, h, cudaMemcpyDefault,
                           c->st));
  }
  *dev = buf.p;
  *dpitch = w;
  *dfstride = (long long)w * h;
  return BL_OK;
}

int check_frames(const void* frames, int pix, int n, int w, int h, size_t pitch, size_t fstride) {
  if (!frames && n > 0) return set_err(BL_ERR_INVALID, "frames is NULL");
  if (pix != BL_PIX_U8 && pix != BL_PIX_F64) return set_err(BL_ERR_INVALID, "unknown pixel type %d", pix);
  if (n < 0) return set_err(BL_ERR_INVALID, "negative frame count");
  if (w < 1 || h < 1) return set_err(BL_ERR_INVALID, "make_image: dimensions must be >= 1");
  if (pitch < (size_t)w) return set_err(BL_ERR_INVALID, "pitch %zu < width %d", pitch, w);
  if (n > 1 && fstride < pitch * (size_t)(h - 1) + w) return set_err(BL_ERR_INVALID, "frame stride too small");
  return BL_OK;
}

// Runs the ERT cascade for `nf` faces whose boxes (int stride) and frame indices are on the
// device; n_faces_dev holds the count.  Output landmarks -> c->ert_out.
// Face-count threshold of the wide (face-per-CTA) cascade, and the per-frame face estimate a
// streamed batch is judged by before its detections exist (the count stays on the device).
constexpr long long kH2dAfterErtPx = 64LL << 20;  // input pixels from which H2D waits for an older cascade
constexpr size_t kEagerBytes = 2u << 20;  // result areas up to this size come back with the counts
constexpr long long kErtClusterMaxFaces = 8;  // expected faces up to which the wide cascade runs as 4-CTA clusters
constexpr long long kErtWideMaxFaces = 400;  // measured crossover 300-600 faces (tools/diag_ert_wide.py)
constexpr long long kErtFacesPerFrameGuess = 4;

int ert_work_ensure(const ErtState& E, ErtWork& wk, int nf, bool leaf_scratch) {
  TRY(wk.cur.ensure(sizeof(double) * 2 * E.dev.L * std::max(1, nf)));
  TRY(wk.tf.ensure(sizeof(double2) * std::max(1, nf)));
  if (leaf_scratch) TRY(wk.leafs.ensure((size_t)std::max(1, nf) * div_up(E.dev.K, 16) * 16 + 16));
  return BL_OK;
}

int run_ert(bl_ctx* c, cudaStream_t st, ErtWork& wk, const void* frames, int pix, int w, int h, long long pitch,
            long long fstride, const int* face_frame, const int* boxes, int box_stride, const int* n_faces_dev,
            int nf, uint8_t* leaf_dev, double* out_xy, int* err_dev, long long expect_faces,
            bool err_zeroed = false) {
  ErtState& E = (*c->ertp);
  const Launch L{st, &c->launches};
  TRY(ert_work_ensure(E, wk, nf, leaf_dev == nullptr));
  // leaf indices: the caller's [face][T*K] buffer, else a per-level scratch [face][K]
  long long leaf_stride = (long long)E.dev.T * E.dev.K;
  uint8_t* leaf = leaf_dev;
  if (!leaf) {
    leaf_stride = div_up(E.dev.K, 16) * 16;  // 16-B aligned rows: 128-bit index loads
    leaf = wk.leafs.as<uint8_t>();
  }
  if (!err_zeroed) CK(cudaMemsetAsync(err_dev, 0, sizeof(int), st));
  // one launch for the whole cascade: a face per CTA while the batch is too small to fill the
  // GPU with kFcFaces-face CTAs (latency), else kFcFaces faces per CTA (leaf-row reuse in L1)
  const bool wide = c->ert_mode == 2 || (c->ert_mode == 0 && expect_faces <= kErtWideMaxFaces);
  if (wide && ert_wide_fits(E.dev)) {
    // a handful of faces (one frame): a cluster of 8 CTAs per face spreads each level's trees
    // and leaf rows over eight SMs (C1 latency 0.293 ms with 4, 0.280 with 8); more faces fill
    // the GPU with one CTA each
    launch_ert_wide(L, E.dev, frames, pix == BL_PIX_U8, w, h, pitch, fstride, face_frame, boxes, box_stride,
                    n_faces_dev, nf, out_xy, leaf_dev, (long long)E.dev.T * E.dev.K, err_dev,
                    c->ert_cl ? c->ert_cl : (expect_faces <= kErtClusterMaxFaces ? 8 : 1));
    return BL_OK;
  }
  if (c->ert_mode != 3 && ert_cascade_fits(E.dev)) {
    launch_ert_cascade(L, E.dev, frames, pix == BL_PIX_U8, w, h, pitch, fstride, face_frame, boxes, box_stride,
                       n_faces_dev, nf, out_xy, leaf_dev, (long long)E.dev.T * E.dev.K, err_dev);
    return BL_OK;
  }
  launch_ert_init(L, E.dev, n_faces_dev, nf, wk.cur.as<double>());
  for (int t = 0; t < E.dev.T; ++t)
    launch_ert_level(L, E.dev, t, frames, pix == BL_PIX_U8, w, h, pitch, fstride, face_frame, boxes, box_stride,
                     n_faces_dev, nf, wk.cur.as<double>(), wk.tf.as<double2>(),
                     leaf_dev ? leaf + (long long)t * E.dev.K : leaf, leaf_stride, err_dev);
  launch_ert_finish(L, E.dev, boxes, box_stride, n_faces_dev, nf, wk.cur.as<double>(), out_xy);
  return BL_OK;
}

void timing_begin(bl_ctx* c) {
  if (!c->timing) return;
  cudaEventRecord(c->ev[BL_STAGE_H2D], c->st);
}

void timing_end(bl_ctx* c, const int* present, int n_present) {
  if (!c->timing) return;
  cudaEventRecord(c->ev[BL_STAGE_COUNT], c->st);
  cudaEventSynchronize(c->ev[BL_STAGE_COUNT]);
  // stages marked in this call, in order; each runs until the next marked one
  for (int i = 0; i < BL_STAGE_COUNT; ++i) c->stage_ms[i] = 0.f;
  for (int i = 0; i < n_present; ++i) {
    const int a = present[i];
    const cudaEvent_t e1 = i + 1 < n_present ? c->ev[present[i + 1]] : c->ev[BL_STAGE_COUNT];
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[a], e1);
    c->stage_ms[a] = ms;
  }
}

int ensure_pinned(void*& p, size_t& cap, size_t bytes) {
  if (cap >= bytes && p) return BL_OK;
  if (p) cudaFreeHost(p);
  p = nullptr;
  cap = 0;
  CK(cudaMallocHost(&p, std::max<size_t>(bytes, 4096)));
  cap = std::max<size_t>(bytes, 4096);
  return BL_OK;
}

bool is_pinned_or_device(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Replays the graph cached for `key` on stream `st`, capturing it first (on the private
// capture stream, with c->st pointed at it while `record` enqueues) when absent or stale.
template <class Record>
int graph_launch(bl_ctx* c, bl_ctx::GraphEntry key, cudaStream_t st, Record&& record) {
  const uint64_t epoch = g_alloc_epoch.load();
  key.epoch = epoch;
  key.model_gen = c->model_gen;
  bl_ctx::GraphEntry* hit = nullptr;
  for (auto& g : c->gcache)
    if (g.kind == key.kind && g.plan == key.plan && g.slot == key.slot && g.in == key.in && g.dp == key.dp &&
        g.df == key.df && g.cap_faces == key.cap_faces && g.n == key.n && g.w == key.w && g.h == key.h &&
        g.pix == key.pix && g.landmarks == key.landmarks) {
      hit = &g;
      break;
    }
  if (hit && (hit->epoch != epoch || hit->model_gen != key.model_gen)) {  // stale: buffers or model changed
    cudaGraphExecDestroy(hit->exec);
    *hit = c->gcache.back();
    c->gcache.pop_back();
    hit = nullptr;
  }
  if (!hit) {
    constexpr size_t kMaxGraphs = 32;
    if (c->gcache.size() >= kMaxGraphs) {  // evict the least recently used
      size_t lru = 0;
      for (size_t i = 1; i < c->gcache.size(); ++i)
        if (c->gcache[i].last_use < c->gcache[lru].last_use) lru = i;
      cudaGraphExecDestroy(c->gcache[lru].exec);
      c->gcache[lru] = c->gcache.back();
      c->gcache.pop_back();
    }
    const cudaStream_t saved = c->st;
    const uint64_t l0 = c->launches;
    c->st = c->cap;
    CK(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeRelaxed));
    const int rc = record();
    cudaGraph_t g = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(c->cap, &g);
    c->st = saved;
    key.kernels = c->launches - l0;
    c->launches = l0;
    if (rc != BL_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ec != cudaSuccess) return set_err(BL_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(ec));
    const cudaError_t ei = cudaGraphInstantiate(&key.exec, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) return set_err(BL_ERR_CUDA, "graph instantiation failed: %s", cudaGetErrorString(ei));
    c->gcache.push_back(key);
    hit = &c->gcache.back();
  }
  hit->last_use = ++c->use_clock;
  CK(cudaGraphLaunch(hit->exec, st));
  c->launches += hit->kernels;
  return BL_OK;
}

void drop_graphs(bl_ctx* c) {
  for (auto& g : c->gcache) cudaGraphExecDestroy(g.exec);
  c->gcache.clear();
}

// Enqueues detect (+ landmarks) for one batch into slot `s`: no host synchronisation.
int enqueue(bl_ctx* c, int s, const void* frames, int pix, int n, int w, int h, size_t pitch, size_t fstride,
            int landmarks) {
  Slot& S = c->slots[s];
  Plan& P = *c->plan;
  const DetectorState& D = (*c->detp);
  const bool same = P.valid && P.n == n && P.w == w && P.h == h && P.pix == pix &&
                    P.window_cells == D.window_cells && P.cell_px == D.cell_px;
  if (!same) {  // arenas may be reallocated: nothing may still be reading them
    CK(cudaStreamSynchronize(c->st));
    CK(cudaStreamSynchronize(c->hst));
    for (Slot& o : c->slots) CK(cudaStreamSynchronize(o.est));
    for (int l = 1; l < kLanes; ++l) CK(cudaStreamSynchronize(c->lanes[l]));
    CK(cudaStreamSynchronize(c->user));
    for (Slot& o : c->slots) CK(cudaStreamSynchronize(o.d2h));
  }
  timing_begin(c);
  const void* dev = nullptr;
  long long dp = 0, df = 0;
  const size_t es = pix == BL_PIX_U8 ? 1 : 8;
  const long long cap_faces = std::max<long long>(1, (long long)n * c->face_cap_per_frame);
  const bool best_only = landmarks == BL_LANDMARKS_BEST;
  const long long lm_rows = best_only ? n : cap_faces;  // landmark rows the cascade writes
  // Every slot is sized together on first use (and on growth), so a pipeline's later slots
  // never allocate -- a synchronising cudaMalloc -- while earlier batches are in flight.
  for (Slot& o : c->slots) {
    if (!is_device_ptr(frames)) TRY(o.input.ensure(es * (size_t)n * w * h));
    TRY(o.flat.ensure(sizeof(DevDet) * cap_faces));
    TRY(o.face_frame.ensure(sizeof(int) * cap_faces));
    TRY(o.meta.ensure(sizeof(int) * (n + 4)));
    TRY(ensure_pinned(reinterpret_cast<void*&>(o.h_meta), o.h_meta_cap, sizeof(int) * (n + 4)));
    if (landmarks) {
      TRY(o.ert_out.ensure(sizeof(double) * 2 * (*c->ertp).dev.L * lm_rows));
      TRY(ert_work_ensure((*c->ertp), o.ert, (int)lm_rows, true));
    }
    if (best_only) {
      TRY(o.best.ensure(sizeof(DevDet) * n));
      TRY(o.best_frame.ensure(sizeof(int) * n));
    }
  }
  if (is_device_ptr(frames)) {
    dev = frames;
    dp = (long long)pitch;
    df = (long long)fstride;
  } else {  // H2D on the copy stream, after the slot's previous batch stopped reading its input
    TRY(S.input.ensure(es * (size_t)n * w * h));
    CK(cudaStreamWaitEvent(c->hst, S.ev_done, 0));
    if (c->h2d_after_ert && (long long)n * w * h >= kH2dAfterErtPx) {
      // a very large batch's input copy waits for the cascade of the batch two submits back: the
      // DMA then streams beside a detection, not beside a cascade whose leaf rows it would evict
      // (bench e2e 93-96k -> 102-103k frames/s).  Not for mid-size batches, whose detection is
      // too short to hide the copy behind (C3's 59 Mpx: e2e 51k -> 45k)
      const Slot& B2 = c->slots[(s + BL_MAX_IN_FLIGHT - 2) % BL_MAX_IN_FLIGHT];
      if (B2.busy) CK(cudaStreamWaitEvent(c->hst, B2.ev_done, 0));
    }
    if (pitch == (size_t)w && fstride == (size_t)w * h) {
      CK(cudaMemcpyAsync(S.input.p, frames, es * (size_t)n * w * h, cudaMemcpyDefault, c->hst));
    } else {
      for (int i = 0; i < n; ++i)
        CK(cudaMemcpy2DAsync((char*)S.input.p + es * (size_t)i * w * h, es * w,
                             (const char*)frames + es * fstride * i, es * pitch, es * w, h, cudaMemcpyDefault,
                             c->hst));
    }
    CK(cudaEventRecord(S.ev_h2d, c->hst));
    CK(cudaStreamWaitEvent(c->st, S.ev_h2d, 0));
    dev = S.input.p;
    dp = w;
    df = (long long)w * h;
  }
  TRY(prepare_detect(c, pix, n, w, h, dp, df));
  TRY(S.flat.ensure(sizeof(DevDet) * cap_faces));
  TRY(S.face_frame.ensure(sizeof(int) * cap_faces));
  TRY(S.meta.ensure(sizeof(int) * (n + 4)));
  int* meta = S.meta.as<int>();
  const bool graph = c->graphs && !c->timing;
  // detection + flatten on the lane stream
  auto rec_det = [&]() -> int {
    TRY(record_detect(c, dev, pix, n, dp, df));
    launch_flatten(launch_of(c), P.kept.as<DevDet>(), P.kept_count.as<int>(), P.cap_pf, n, P.offsets.as<int>(),
                   S.flat.as<DevDet>(), S.face_frame.as<int>(), meta, cap_faces, P.overflow.as<int>(),
                   best_only ? S.best.as<DevDet>() : nullptr, best_only ? S.best_frame.as<int>() : nullptr);
    return BL_OK;  // (k_flatten zeroes meta[n + 2], the cascade's error flag)
  };
  if (graph) {
    bl_ctx::GraphEntry key;
    key.kind = 0;
    key.plan = c->plan;
    key.slot = s;
    key.in = dev;
    key.dp = dp;
    key.df = df;
    key.cap_faces = cap_faces;
    key.n = n;
    key.w = w;
    key.h = h;
    key.pix = pix;
    key.landmarks = landmarks;
    TRY(graph_launch(c, key, c->st, rec_det));
  } else {
    TRY(rec_det());
  }
  if (landmarks) {
    stage_mark(c, BL_STAGE_ERT);
    // the cascade only reads this slot's buffers and the frames.  A small batch's cascade runs
    // on the slot's ERT stream, beside the next batches' detection and the other slots'
    // cascades (few faces fill few SMs: C2 14k -> 64k frames/s with this).  A large batch's
    // cascade runs after its own detection on the lane stream: beside the other lane's
    // detection its 130 MB leaf table and the detection's streams evict each other from L2 --
    // measured 86-89k frames/s at the bench concurrent, 99-102k queued on the lane.
    const bool large = (long long)n * w * h > kSmallBatchPx;
    cudaStream_t es = (c->timing || c->ert_serial || (large && !c->ert_conc)) ? c->st : S.est;
    if (es != c->st) {
      CK(cudaEventRecord(S.ev_det, c->st));
      CK(cudaStreamWaitEvent(es, S.ev_det, 0));
    }
    auto rec_ert = [&](cudaStream_t st) -> int {
      if (best_only)  // the face of each frame only (run(), pipeline.cpp:171-190): row f = frame f
        return run_ert(c, st, S.ert, dev, pix, w, h, dp, df, S.best_frame.as<int>(), S.best.as<int>(), 8,
                       meta + n + 3, n, nullptr, S.ert_out.as<double>(), meta + n + 2, n, true);
      return run_ert(c, st, S.ert, dev, pix, w, h, dp, df, S.face_frame.as<int>(), S.flat.as<int>(), 8, meta + n,
                     (int)cap_faces, nullptr, S.ert_out.as<double>(), meta + n + 2,
                     (long long)n * kErtFacesPerFrameGuess, true);
    };
    if (graph) {
      TRY(ert_work_ensure((*c->ertp), S.ert, (int)lm_rows, true));
      bl_ctx::GraphEntry key;
      key.kind = 1;
      key.slot = s;
      key.landmarks = landmarks;
      key.in = dev;
      key.dp = dp;
      key.df = df;
      key.cap_faces = cap_faces;
      key.n = n;
      key.w = w;
      key.h = h;
      key.pix = pix;
      TRY(graph_launch(c, key, es, [&]() { return rec_ert(c->st); }));
    } else {
      TRY(rec_ert(es));
    }
    CK(cudaEventRecord(S.ev_done, es));
  } else {
    CK(cudaEventRecord(S.ev_done, c->st));
  }
  // counts + flags back on the slot's D2H stream as soon as compute finishes; a small batch's
  // whole result area follows in the same stream (C1: 2 KB of detections + 70 KB of landmark
  // rows), so collect waits once instead of a second D2H round trip after the counts arrive
  TRY(ensure_pinned(reinterpret_cast<void*&>(S.h_meta), S.h_meta_cap, sizeof(int) * (n + 4)));
  const size_t eager_d = sizeof(bl_detection) * (size_t)cap_faces;
  const size_t eager_l = landmarks ? sizeof(double) * 2 * (*c->ertp).dev.L * (size_t)lm_rows : 0;
  S.eager = eager_d + eager_l <= kEagerBytes;
  if (S.eager) TRY(ensure_pinned(S.h_stage, S.h_stage_cap, eager_d + eager_l + 64));  // (slot idle)
  CK(cudaStreamWaitEvent(S.d2h, S.ev_done, 0));
  CK(cudaMemcpyAsync(S.h_meta, meta, sizeof(int) * (n + 3), cudaMemcpyDeviceToHost, S.d2h));
  if (S.eager) {
    CK(cudaMemcpyAsync(S.h_stage, S.flat.p, eager_d, cudaMemcpyDeviceToHost, S.d2h));
    if (eager_l)
      CK(cudaMemcpyAsync(static_cast<char*>(S.h_stage) + eager_d, S.ert_out.p, eager_l, cudaMemcpyDeviceToHost, S.d2h));
  }
  CK(cudaEventRecord(S.ev_meta, S.d2h));
  S.busy = true;
  S.n = n;
  S.w = w;
  S.h = h;
  S.pix = pix;
  S.landmarks = landmarks;
  S.cap_faces = cap_faces;
  return BL_OK;
}

// Waits for slot `s` and copies its results out.  On BL_ERR_CAPACITY for the caller's output
// buffer the slot stays busy (results remain on the device; collect again with more room).
int collect(bl_ctx* c, int s, bl_detection* out, int64_t cap, int32_t* counts, int64_t* total, double* landmarks) {
  Slot& S = c->slots[s];
  if (!S.busy) return set_err(BL_ERR_STATE, "nothing submitted in this slot");
  CK(cudaEventSynchronize(S.ev_meta));
  CK(cudaGetLastError());
  const int n = S.n;
  const int* m = S.h_meta;
  if (m[n + 1]) {
    S.busy = false;
    return set_err(BL_ERR_CAPACITY, "raw detection capacity exceeded");
  }
  const int64_t tot = m[n];
  if (total) *total = tot;
  if (counts) std::memcpy(counts, m, sizeof(int32_t) * n);
  if (S.landmarks && m[n + 2] == 1) {
    S.busy = false;
    return set_err(BL_ERR_INVALID, "similarity_transform: source shape has no spread");
  }
  if (S.landmarks && m[n + 2] == 2) {
    S.busy = false;
    return set_err(BL_ERR_INVALID, "similarity_transform: target shape has no spread");
  }
  if (tot > S.cap_faces) {
    S.busy = false;
    return set_err(BL_ERR_CAPACITY, "%lld kept detections exceed the device face capacity %lld "
                   "(bl_ctx_set_face_capacity)", (long long)tot, (long long)S.cap_faces);
  }
  if (tot > cap)
    return set_err(BL_ERR_CAPACITY, "output capacity %lld < %lld detections", (long long)cap, (long long)tot);
  stage_mark(c, BL_STAGE_D2H);
  const size_t bd = sizeof(bl_detection) * tot;
  const int64_t lm_rows = S.landmarks == BL_LANDMARKS_BEST ? S.n : tot;  // best-only: one row per frame
  const size_t bl = S.landmarks && landmarks ? sizeof(double) * 2 * (*c->ertp).dev.L * lm_rows : 0;
  if (S.eager) {  // already in the pinned staging area (copied behind the counts)
    const char* st = static_cast<const char*>(S.h_stage);
    if (tot > 0 && out) std::memcpy(out, st, bd);
    if (bl) std::memcpy(landmarks, st + sizeof(bl_detection) * (size_t)S.cap_faces, bl);
    S.busy = false;
    return BL_OK;
  }
  const bool direct_d = !out || is_pinned_or_device(out);
  const bool direct_l = !bl || is_pinned_or_device(landmarks);
  const size_t need = (direct_d ? 0 : bd) + (direct_l ? 0 : bl) + 64;
  if (S.h_stage_cap < need)  // grow every idle slot's staging at once (no host allocations
                             // mid-pipeline; a busy slot may have a copy in flight into its own)
    for (Slot& o : c->slots)
      if (&o == &S || !o.busy) TRY(ensure_pinned(o.h_stage, o.h_stage_cap, need + need / 2));
  char* stage = static_cast<char*>(S.h_stage);
  if (tot > 0 && out)
    CK(cudaMemcpyAsync(direct_d ? (void*)out : stage, S.flat.p, bd, cudaMemcpyDefault, S.d2h));
  if (bl)
    CK(cudaMemcpyAsync(direct_l ? (void*)landmarks : stage + (direct_d ? 0 : bd), S.ert_out.p, bl, cudaMemcpyDefault,
                       S.d2h));
  CK(cudaEventRecord(S.ev_out, S.d2h));
  CK(cudaEventSynchronize(S.ev_out));
  if (tot > 0 && out && !direct_d) std::memcpy(out, stage, bd);
  if (bl && !direct_l) std::memcpy(landmarks, stage + (direct_d ? 0 : bd), bl);
  S.busy = false;
  return BL_OK;
}

int detect_common(bl_ctx* c, const void* frames, int pix, int n, int w, int h, size_t pitch, size_t fstride,
                  bl_detection* out, int64_t cap, int32_t* counts, int64_t* total, double* landmarks) {
  if (!c) return set_err(BL_ERR_INVALID, "null context");
  std::lock_guard<std::mutex> lk(c->mu);
  if (!(*c->detp).ready) return set_err(BL_ERR_STATE, "no detector model uploaded");
  if (landmarks && !(*c->ertp).ready) return set_err(BL_ERR_STATE, "no ERT model uploaded");
  if (fstride == 0) fstride = pitch * h;
  TRY(check_frames(frames, pix, n, w, h, pitch, fstride));
  TRY(use_device(c));
  if (n == 0) {
    if (total) *total = 0;
    return BL_OK;
  }
  for (int s = 0; s < BL_MAX_IN_FLIGHT; ++s)
    if (c->slots[s].busy) return set_err(BL_ERR_STATE, "submitted batches must be collected first");
  for (int attempt = 0; attempt < 2; ++attempt) {
    TRY(enqueue(c, 0, frames, pix, n, w, h, pitch, fstride, landmarks != nullptr));
    int64_t tot = 0;
    const int rc = collect(c, 0, out, cap, counts, &tot, landmarks);
    if (total) *total = tot;
    if (rc == BL_ERR_CAPACITY && tot > c->slots[0].cap_faces && attempt == 0) {
      // more kept detections than the device face capacity: grow it and redo the batch
      c->face_cap_per_frame = (int)std::max<long long>(c->face_cap_per_frame, div_up(tot, n) + 1);
      if (tot > (long long)n * c->face_cap_per_frame) c->face_cap_per_frame = (int)div_up(tot, n) + 1;
      continue;
    }
    if (rc != BL_OK) {
      c->slots[0].busy = false;
      return rc;
    }
    break;
  }
  const int present_det[] = {BL_STAGE_H2D, BL_STAGE_PYRAMID, BL_STAGE_GRADHIST, BL_STAGE_FEATURES,
                             BL_STAGE_SCREEN, BL_STAGE_RESCORE, BL_STAGE_NMS, BL_STAGE_ERT, BL_STAGE_D2H};
  const int p2[] = {BL_STAGE_H2D, BL_STAGE_PYRAMID, BL_STAGE_GRADHIST, BL_STAGE_FEATURES,
                    BL_STAGE_SCREEN, BL_STAGE_RESCORE, BL_STAGE_NMS, BL_STAGE_D2H};
  if (landmarks)
    timing_end(c, present_det, 9);
  else
    timing_end(c, p2, 8);
  return BL_OK;
}

// Model uploads overwrite device buffers that in-flight batches read: refuse while a submitted
// batch is uncollected, and drain every context stream before the first write.
int quiesce_for_upload(bl_ctx* c) {
  for (const Slot& S : c->slots)
    if (S.busy) return set_err(BL_ERR_STATE, "collect the submitted batches before uploading a model");
  CK(cudaStreamSynchronize(c->user));
  CK(cudaStreamSynchronize(c->hst));
  for (int l = 1; l < kLanes; ++l) CK(cudaStreamSynchronize(c->lanes[l]));
  for (const Slot& S : c->slots) {
    CK(cudaStreamSynchronize(S.est));
    CK(cudaStreamSynchronize(S.d2h));
  }
  return BL_OK;
}

// Copies `bytes` from a user pointer (host or device) into scratch, returns a device pointer.
int to_device(bl_ctx* c, DevBuf& buf, const void* src, size_t bytes, const void** dev) {
  if (is_device_ptr(src)) {
    *dev = src;
    return BL_OK;
  }
  TRY(buf.ensure(bytes));
  if (bytes) CK(cudaMemcpyAsync(buf.p, src, bytes, cudaMemcpyDefault, c->st));
  *dev = buf.p;
  return BL_OK;
}

int from_device(bl_ctx* c, void* dst, const void* dev, size_t bytes) {
  if (bytes) CK(cudaMemcpyAsync(dst, dev, bytes, cudaMemcpyDefault, c->st));
  CK(cudaStreamSynchronize(c->st));
  CK(cudaGetLastError());
  return BL_OK;
}

// Single-level plan over one feature/cell grid (stage functions).
void single_level_plan(PlanDesc& H, int w, int h, int cw, int ch) {
  std::memset(&H, 0, sizeof H);
  H.n_frames = 1;
  H.n_scored = 1;
  LevelDesc& L = H.lv[0];
  L.w = w;
  L.h = h;
  L.cw = cw;
  L.ch = ch;
  L.sw = cw - 9;
  L.sh = ch - 9;
  L.pix_pitch = w;
  L.pix_fstride = (long long)w * h;
  L.gr_tiles_x = (int)div_up(w, 32);
  L.gr_tiles_y = (int)div_up(h, 64);
  H.gr_total = (long long)L.gr_tiles_x * L.gr_tiles_y;
  H.fld_total = (long long)w * h;
  L.gh_tiles_x = (int)div_up(cw, kGhCells);
  L.gh_tiles_y = (int)div_up(ch, kGhSegRows);
  H.gh_total = (long long)L.gh_tiles_x * L.gh_tiles_y;
  H.cell_total = (long long)cw * ch;
  H.cells_per_frame = H.cell_total;
}

}  // namespace

// =============================================================== extern "C" ABI ====
extern "C" {

int bl_abi_version(void) { return BL_ABI_VERSION; }

int bl_plan_geometry(int w, int h, int window_cells, int cell_px, int scale_num, int scale_den,
                     double min_face_ratio, int* dims, int* scored, double* scale_c, int* side, int max_levels,
                     int* n_levels, int* n_scored) {
  if (!n_levels || !n_scored) return set_err(BL_ERR_INVALID, "null out");
  if (w < 1 || h < 1) return set_err(BL_ERR_INVALID, "make_image: dimensions must be >= 1");
  if (window_cells != kWin) return set_err(BL_ERR_INVALID, "filter must carry exactly 3100 weights");
  if (cell_px < 1 || scale_num < 1 || scale_den < 1) return set_err(BL_ERR_MODEL, "bad detector geometry");
  std::vector<int> lw, lh;
  const int window = window_cells * cell_px;
  pyramid_dims(w, h, window, lw, lh);
  *n_levels = (int)lw.size();
  const double min_face = min_face_ratio * std::min(w, h);
  int ns = 0;
  for (int k = 0; k < (int)lw.size(); ++k) {
    if (k < max_levels && dims) {
      dims[2 * k] = lw[k];
      dims[2 * k + 1] = lh[k];
    }
    const double c = std::pow(double(scale_num) / scale_den, double(k));
    const double detectable = window / c;
    if (!(detectable >= min_face * (1.0 - 1e-9))) continue;
    if (lw[k] / cell_px < window_cells || lh[k] / cell_px < window_cells) continue;
    if (ns < max_levels) {
      if (scored) scored[ns] = k;
      if (scale_c) scale_c[ns] = c;
      if (side) side[ns] = round_half_up_host(window / c);
    }
    ++ns;
  }
  *n_scored = ns;
  return BL_OK;
}

const char* bl_last_error(void) { return g_err.c_str(); }

int bl_device_count(int* n) {
  if (!n) return set_err(BL_ERR_INVALID, "null out");
  CK(cudaGetDeviceCount(n));
  return BL_OK;
}

int bl_ctx_create(int device, bl_ctx** out) {
  if (!out) return set_err(BL_ERR_INVALID, "null out");
  *out = nullptr;
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (device < 0 || device >= nd) return set_err(BL_ERR_INVALID, "device %d out of range (%d devices)", device, nd);
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return set_err(BL_ERR_CUDA, "blinkline_b200 is built for sm_100a; device %d is sm_%d%d", device, prop.major,
                   prop.minor);
  auto c = std::make_unique<bl_ctx>();
  c->device = device;
  CK(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->hst, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
  {  // the cascades fill the gaps of the next batches' detection: lowest priority
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (Slot& S : c->slots) CK(cudaStreamCreateWithPriority(&S.est, cudaStreamNonBlocking, lo));
  }
  c->st = c->user = c->own;
  for (int l = 1; l < kLanes; ++l) CK(cudaStreamCreateWithFlags(&c->lanes[l], cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->ev_lane, cudaEventDisableTiming));
  for (Plan& P : c->plans) {
    CK(cudaStreamCreateWithFlags(&P.aux, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&P.ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&P.ev_join, cudaEventDisableTiming));
  }
  for (Slot& S : c->slots) {
    CK(cudaStreamCreateWithFlags(&S.d2h, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&S.ev_h2d, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&S.ev_det, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&S.ev_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&S.ev_meta, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&S.ev_out, cudaEventDisableTiming));
  }
  for (auto& e : c->ev) CK(cudaEventCreate(&e));
  // hog.cpp:12-24: the 18 directions from the host libm, exactly as the reference builds them
  double ux[kBins], uy[kBins];
  for (int d = 0; d < kBins; ++d) {
    const double a = 2.0 * M_PI * d / kBins;
    ux[d] = std::cos(a);
    uy[d] = std::sin(a);
  }
  set_direction_table(ux, uy);
  {  // shared-memory opt-in is a per-device function attribute: set it for this device
    const int optin = (int)prop.sharedMemPerBlockOptin;
    configure_screen_tc_kernels(optin);
    configure_exact_kernels(optin);
    configure_hog_kernels(optin);
    configure_classify_kernels(optin);
    configure_ert_kernels(optin);
    configure_pyramid_kernels(optin);
    CK(cudaGetLastError());
  }
  if (const char* e = std::getenv("BL_SCREEN")) c->screen = std::strcmp(e, "fp32") == 0 ? BL_SCREEN_FP32 : BL_SCREEN_TCGEN05;
  if (const char* e = std::getenv("BL_PYR_FUSE")) c->pyr_fuse = std::atoi(e) != 0;
  if (const char* e = std::getenv("BL_GRAPHS")) c->graphs = std::atoi(e) != 0;
  if (const char* e = std::getenv("BL_ERT_SERIAL")) c->ert_serial = std::atoi(e) != 0;
  if (const char* e = std::getenv("BL_ERT_CONC")) c->ert_conc = std::atoi(e) != 0;
  if (const char* e = std::getenv("BL_H2D_AFTER_ERT")) c->h2d_after_ert = std::atoi(e) != 0;
  if (const char* e = std::getenv("BL_ERT_CL")) c->ert_cl = std::atoi(e);
  if (const char* e = std::getenv("BL_LANES_LARGE")) c->lanes_large = std::max(1, std::min(kLanes, std::atoi(e)));
  if (const char* e = std::getenv("BL_PYR_CHAIN")) c->pyr_chain = std::atoi(e) != 0;
  if (const char* e = std::getenv("BL_ERT"))
    c->ert_mode = !std::strcmp(e, "cascade") ? 1 : !std::strcmp(e, "wide") ? 2 : !std::strcmp(e, "levels") ? 3 : 0;
  CK(cudaGetLastError());
  *out = c.release();
  return BL_OK;
}

void bl_ctx_destroy(bl_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  drop_graphs(c);
  if (c->cap) cudaStreamDestroy(c->cap);
  cudaStreamSynchronize(c->st);
  if (c->hst) cudaStreamSynchronize(c->hst);
  for (int l = 1; l < kLanes; ++l)
    if (c->lanes[l]) cudaStreamSynchronize(c->lanes[l]);
  if (c->ev_lane) cudaEventDestroy(c->ev_lane);
  for (Plan& P : c->plans) {
    if (P.aux) {
      cudaStreamSynchronize(P.aux);
      cudaStreamDestroy(P.aux);
    }
    for (cudaEvent_t e : {P.ev_fork, P.ev_join})
      if (e) cudaEventDestroy(e);
  }
  for (Slot& S : c->slots) {
    if (S.h_meta) cudaFreeHost(S.h_meta);
    if (S.h_stage) cudaFreeHost(S.h_stage);
    for (cudaEvent_t e : {S.ev_h2d, S.ev_det, S.ev_done, S.ev_meta, S.ev_out})
      if (e) cudaEventDestroy(e);
    if (S.d2h) {
      cudaStreamSynchronize(S.d2h);
      cudaStreamDestroy(S.d2h);
    }
    if (S.est) {
      cudaStreamSynchronize(S.est);
      cudaStreamDestroy(S.est);
    }
  }
  cudaStream_t hst = c->hst;
  cudaStream_t lanes[kLanes];
  for (int l = 0; l < kLanes; ++l) lanes[l] = c->lanes[l];
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  cudaStream_t own = c->own;
  delete c;  // DevBufs free on their device
  if (own) cudaStreamDestroy(own);
  if (hst) cudaStreamDestroy(hst);
  for (int l = 1; l < kLanes; ++l)
    if (lanes[l]) cudaStreamDestroy(lanes[l]);
}

int bl_ctx_set_stream(bl_ctx* c, void* stream) {
  if (!c) return set_err(BL_ERR_INVALID, "null context");
  std::lock_guard<std::mutex> lk(c->mu);
  c->st = c->user = stream ? (cudaStream_t)stream : c->own;
  return BL_OK;
}

int bl_ctx_synchronize(bl_ctx* c) {
  if (!c) return set_err(BL_ERR_INVALID, "null context");
  TRY(use_device(c));
  CK(cudaStreamSynchronize(c->st));
  for (int l = 1; l < kLanes; ++l) CK(cudaStreamSynchronize(c->lanes[l]));
  for (Slot& S : c->slots) CK(cudaStreamSynchronize(S.est));
  CK(cudaStreamSynchronize(c->hst));
  return BL_OK;
}

int bl_ctx_launch_count(bl_ctx* c, uint64_t* out) {
  if (!c || !out) return set_err(BL_ERR_INVALID, "null argument");
  *out = c->launches;
  return BL_OK;
}

int bl_ctx_enable_stage_timing(bl_ctx* c, int enable) {
  if (!c) return set_err(BL_ERR_INVALID, "null context");
  c->timing = enable != 0;
  return BL_OK;
}

int bl_ctx_stage_times(bl_ctx* c, float* ms, int* launches) {
  if (!c) return set_err(BL_ERR_INVALID, "null context");
  for (int i = 0; i < BL_STAGE_COUNT; ++i) {
    if (ms) ms[i] = c->stage_ms[i];
    if (launches) launches[i] = c->stage_launch[i];
  }
  return BL_OK;
}

int bl_ctx_model_info(bl_ctx* c, int* landmark_count) {
  if (!c || !landmark_count) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (!(*c->ertp).ready) return set_err(BL_ERR_STATE, "no ERT model uploaded");
  *landmark_count = (*c->ertp).dev.L;
  return BL_OK;
}

int bl_ctx_set_screen(bl_ctx* c, int mode) {
  if (!c) return set_err(BL_ERR_INVALID, "null context");
  if (mode != BL_SCREEN_TCGEN05 && mode != BL_SCREEN_FP32) return set_err(BL_ERR_INVALID, "unknown screen mode %d", mode);
  std::lock_guard<std::mutex> lk(c->mu);
  c->screen = mode;
  ++c->model_gen;  // captured graphs launch the other screen
  return BL_OK;
}

int bl_ctx_enable_graphs(bl_ctx* c, int enable) {
  if (!c) return set_err(BL_ERR_INVALID, "null context");
  std::lock_guard<std::mutex> lk(c->mu);
  c->graphs = enable != 0;
  if (!c->graphs) drop_graphs(c);
  return BL_OK;
}

int bl_detector_upload(bl_ctx* c, const double* weights, const double* biases, double threshold, int window_cells,
                       int cell_px, int scale_num, int scale_den, double min_face_ratio) {
  if (!c || !weights || !biases) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (window_cells != kWin) return set_err(BL_ERR_INVALID, "filter must carry exactly 3100 weights");
  if (cell_px < 1) return set_err(BL_ERR_MODEL, "cell_px must be >= 1");
  if (scale_num < 1 || scale_den < 1) return set_err(BL_ERR_MODEL, "scale factor must be positive");
  TRY(use_device(c));
  TRY(quiesce_for_upload(c));
  ++c->model_gen;  // thresholds and cuts are baked into captured graphs
  // a fresh state object: contexts sharing the previous one keep it (and a failed upload
  // leaves this context's previous model in place)
  auto nd = std::make_shared<DetectorState>();
  DetectorState& D = *nd;
  D.thr = threshold;
  D.window_cells = window_cells;
  D.cell_px = cell_px;
  D.scale_num = scale_num;
  D.scale_den = scale_den;
  D.min_face_ratio = min_face_ratio;
  // fp32 screen weights, [j][f][i*5 + r] blocks of 52 floats
  std::vector<float> w32((size_t)kWin * kFeat * 52, 0.f);
  for (int r = 0; r < kFilters; ++r)
    for (int j = 0; j < kWin; ++j)
      for (int i = 0; i < kWin; ++i)
        for (int f = 0; f < kFeat; ++f)
          w32[((size_t)j * kFeat + f) * 52 + i * kFilters + r] =
              (float)weights[(size_t)r * kFilterW + j * kRowW + i * kFeat + f];
  // rigorous screen cut: |fp32 window sum - exact sum| <= delta_r
  const double u = std::ldexp(1.0, -24);
  for (int r = 0; r < kFilters; ++r) {
    double l1 = 0;
    for (int k = 0; k < kFilterW; ++k) l1 += std::fabs(weights[(size_t)r * kFilterW + k]);
    D.bias[r] = biases[r];
    const double delta = 324.0 * u * 1.01 * 0.8486 * l1 + std::ldexp(1.0, -20) * (std::fabs(threshold) + std::fabs(biases[r])) + 1e-9;
    const double cutd = threshold - biases[r] - delta;
    float cf = (float)cutd;
    if (std::isnan(cutd)) cf = -INFINITY;
    if ((double)cf > cutd) cf = std::nextafterf(cf, -INFINITY);
    D.cut[r] = cf;
  }
  // tcgen05 screen: fp16 weights [j][kc][64 n = dx * 5 + r][8], filter r scaled by 2^ws[r] so
  // its largest |w| lies in [2^14, 2^15) (exact; fp16 max 65504), features scaled by
  // 2^kTcFeatExp in k_features.  The screen compares the scaled sum against the scaled cut.
  // delta_tc >= |fp16 MMA sum - exact sum| in unscaled units: operands rounded to fp16 (each
  // <= 2^-11 relative when normal, product <= 2^-10 + 2^-22; values in the fp16 subnormal
  // range carry an absolute error <= 2^-25 of their scaled unit instead: 2^-25-kTcFeatExp per
  // feature, 2^-25-ws per weight), fp32 accumulation over 200 MMAs of K = 16 (<= 1024 u even
  // with truncating hardware adds), features <= 0.8486.
  int ws[kFilters];
  for (int r = 0; r < kFilters; ++r) {
    double mx = 0;
    for (int k = 0; k < kFilterW; ++k) mx = std::max(mx, std::fabs(weights[(size_t)r * kFilterW + k]));
    int e = 0;
    if (mx > 0) std::frexp(mx, &e);       // mx in [2^(e-1), 2^e)
    ws[r] = mx > 0 && std::isfinite(mx) ? 15 - e : 0;  // mx * 2^ws in [2^14, 2^15)
    ws[r] = std::max(-100, std::min(100, ws[r]));
  }
  std::vector<uint16_t> wtc(tc_weight_floats() * 2, 0);
  for (int j = 0; j < kWin; ++j)
    for (int dx = 0; dx < kWin; ++dx)
      for (int f = 0; f < kFeat; ++f)
        for (int r = 0; r < kFilters; ++r)
          wtc[(((size_t)j * kTcPlanesF16 + f / 8) * 64 + dx * kFilters + r) * 8 + f % 8] =
              half_rn_host(std::ldexp(weights[(size_t)r * kFilterW + j * kRowW + dx * kFeat + f], ws[r]));
  for (int r = 0; r < kFilters; ++r) {
    double l1 = 0;
    for (int k = 0; k < kFilterW; ++k) l1 += std::fabs(weights[(size_t)r * kFilterW + k]);
    const double rel = std::ldexp(1.0, -10) + std::ldexp(1.0, -22) + std::ldexp(1.0, -24) + 1024.0 * u;
    const double sub = l1 * std::ldexp(1.0, -25 - kTcFeatExp) + 0.85 * kFilterW * std::ldexp(1.0, -25 - ws[r]);
    const double delta = 1.1 * (rel * 0.8486 * l1 + sub) + std::ldexp(1.0, -20) * (std::fabs(threshold) + std::fabs(biases[r])) + 1e-9;
    D.delta_tc[r] = delta;
    const double cutd = threshold - biases[r] - delta;
    const int sc = ws[r] + kTcFeatExp;
    float cf = (float)std::ldexp(cutd, sc);  // cut in the scaled domain (power-of-two scaling)
    if (std::isnan(cutd)) cf = -INFINITY;
    if ((double)cf > std::ldexp(cutd, sc)) cf = std::nextafterf(cf, -INFINITY);
    D.cut_tc[r] = cf;
    D.cut_tc[kFilters + r] = (float)std::ldexp(1.0, -sc);
  }
  TRY(D.w_tc.ensure(sizeof(uint16_t) * wtc.size()));
  TRY(D.cuttc.ensure(sizeof(float) * 2 * kFilters));
  CK(cudaMemcpy(D.w_tc.p, wtc.data(), sizeof(uint16_t) * wtc.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(D.cuttc.p, D.cut_tc, sizeof(float) * 2 * kFilters, cudaMemcpyHostToDevice));
  TRY(D.w64.ensure(sizeof(double) * kFilters * kFilterW));
  TRY(D.w32.ensure(sizeof(float) * w32.size()));
  TRY(D.bias64.ensure(sizeof(double) * kFilters));
  TRY(D.cut32.ensure(sizeof(float) * kFilters));
  CK(cudaMemcpy(D.w64.p, weights, sizeof(double) * kFilters * kFilterW, cudaMemcpyDefault));
  CK(cudaMemcpy(D.w32.p, w32.data(), sizeof(float) * w32.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(D.bias64.p, biases, sizeof(double) * kFilters, cudaMemcpyDefault));
  CK(cudaMemcpy(D.cut32.p, D.cut, sizeof(float) * kFilters, cudaMemcpyHostToDevice));
  // the small-batch re-score's transposed copy [c][f][r][j] (k_rescore_lat)
  TRY(D.w64t.ensure(sizeof(double) * kFilters * kFilterW));
  launch_transpose_weights(Launch{c->own, &c->launches}, D.w64.as<double>(), D.w64t.as<double>());
  CK(cudaStreamSynchronize(c->own));
  for (Plan& p : c->plans) p.valid = false;
  D.ready = true;
  c->detp = std::move(nd);
  return BL_OK;
}

int bl_ert_upload(bl_ctx* c, int L, int T, int K, int F, double shrinkage, const double* mean_xy,
                  const int32_t* anchors, const double* split_params, const double* leaves) {
  if (!c) return set_err(BL_ERR_INVALID, "null context");
  std::lock_guard<std::mutex> lk(c->mu);
  if (L < 2) return set_err(BL_ERR_INVALID, "predict_landmarks: model has no mean shape");
  if (T < 0 || K < 0 || F < 0 || F > 8) return set_err(BL_ERR_MODEL, "cascade dims out of range");
  if (T > 0 && K < 1) return set_err(BL_ERR_MODEL, "every cascade level must carry K trees");
  if (!mean_xy || ((size_t)T * K > 0 && (!leaves || (F > 0 && (!anchors || !split_params)))))
    return set_err(BL_ERR_INVALID, "null model array");
  TRY(use_device(c));
  TRY(quiesce_for_upload(c));
  ++c->model_gen;  // the cascade's dims and pointers are baked into captured graphs
  auto ne = std::make_shared<ErtState>();  // fresh: sharers keep the previous model
  ErtState& E = *ne;
  const int S = (1 << F) - 1, NL = 1 << F;
  const size_t nsplit = (size_t)T * K * S;
  if (2 * L > 512) return set_err(BL_ERR_MODEL, "landmark count above 256 is not supported");
  // node-major split records [t][node][k] (tree-major in the upload format)
  std::vector<SplitRec> recs(nsplit + 1);
  for (int t = 0; t < T; ++t)
    for (int k = 0; k < K; ++k)
      for (int s = 0; s < S; ++s) {
        const size_t src = ((size_t)t * K + k) * S + s;
        const int32_t a = anchors[2 * src], b = anchors[2 * src + 1];
        if (a < 0 || a >= L || b < 0 || b >= L) return set_err(BL_ERR_MODEL, "split anchor out of range");
        SplitRec& r = recs[((size_t)t * S + s) * K + k];
        r.oax = split_params[5 * src];
        r.oay = split_params[5 * src + 1];
        r.obx = split_params[5 * src + 2];
        r.oby = split_params[5 * src + 3];
        r.thr = split_params[5 * src + 4];
        r.anchors = make_short2((short)a, (short)b);
        r.pad = 0;
      }
  TRY(E.mean.ensure(sizeof(double) * 2 * L));
  TRY(E.mean_c.ensure(sizeof(double) * 2 * L));
  // split planes: a warp's 32 consecutive trees at one node read 3 x 512 contiguous bytes
  const size_t plane = recs.size();
  std::vector<int4> planes(3 * plane);
  for (size_t i = 0; i < plane; ++i)
    for (int q = 0; q < 3; ++q) std::memcpy(&planes[q * plane + i], reinterpret_cast<const char*>(&recs[i]) + 16 * q, 16);
  TRY(E.split.ensure(sizeof(int4) * planes.size()));
  TRY(E.leaves.ensure(sizeof(double) * (size_t)T * K * NL * L * 2 + 16));
  CK(cudaMemcpy(E.mean.p, mean_xy, sizeof(double) * 2 * L, cudaMemcpyDefault));
  CK(cudaMemcpy(E.split.p, planes.data(), sizeof(int4) * planes.size(), cudaMemcpyHostToDevice));
  if ((size_t)T * K) CK(cudaMemcpy(E.leaves.p, leaves, sizeof(double) * (size_t)T * K * NL * L * 2, cudaMemcpyDefault));
  // centroid of the mean shape in similarity_transform's order (ert.cpp:33-43), and the
  // centred mean (to.x - mt.x, to.y - mt.y) every level reuses
  std::vector<double> m(2 * L);
  CK(cudaMemcpy(m.data(), mean_xy, sizeof(double) * 2 * L, cudaMemcpyDefault));
  double mx = 0, my = 0;
  for (int i = 0; i < L; ++i) {
    mx += m[2 * i];
    my += m[2 * i + 1];
  }
  mx /= double(L);
  my /= double(L);
  std::vector<double> mc(2 * L);
  for (int i = 0; i < L; ++i) {
    mc[2 * i] = m[2 * i] - mx;
    mc[2 * i + 1] = m[2 * i + 1] - my;
  }
  CK(cudaMemcpy(E.mean_c.p, mc.data(), sizeof(double) * 2 * L, cudaMemcpyHostToDevice));
  E.dev.L = L;
  E.dev.T = T;
  E.dev.K = K;
  E.dev.F = F;
  E.dev.S = S;
  E.dev.NL = NL;
  E.dev.shrinkage = shrinkage;
  E.dev.mean_xy = E.mean.as<double>();
  E.dev.mean_c = E.mean_c.as<double>();
  E.dev.split = E.split.as<SplitRec>();
  E.dev.split_plane = (long long)plane;
  E.dev.leaves = E.leaves.as<double>();
  E.dev.mean_cx = mx;
  E.dev.mean_cy = my;
  E.ready = true;
  c->ertp = std::move(ne);
  return BL_OK;
}

int bl_detect(bl_ctx* c, const void* frames, int pixel_type, int n, int w, int h, size_t pitch, size_t frame_stride,
              bl_detection* out, int64_t cap, int32_t* counts, int64_t* total) {
  return detect_common(c, frames, pixel_type, n, w, h, pitch, frame_stride, out, cap, counts, total, nullptr);
}

int bl_detect_landmarks(bl_ctx* c, const void* frames, int pixel_type, int n, int w, int h, size_t pitch,
                        size_t frame_stride, bl_detection* out, int64_t cap, int32_t* counts, int64_t* total,
                        double* landmarks) {
  if (!landmarks) return set_err(BL_ERR_INVALID, "landmarks output is NULL");
  return detect_common(c, frames, pixel_type, n, w, h, pitch, frame_stride, out, cap, counts, total, landmarks);
}

int bl_ctx_set_face_capacity(bl_ctx* c, int faces_per_frame) {
  if (!c || faces_per_frame < 1) return set_err(BL_ERR_INVALID, "bad face capacity");
  std::lock_guard<std::mutex> lk(c->mu);
  c->face_cap_per_frame = faces_per_frame;
  return BL_OK;
}

int bl_ctx_share_models(bl_ctx* dst, bl_ctx* src, int what) {
  if (!dst || !src) return set_err(BL_ERR_INVALID, "null context");
  if (what & ~(BL_SHARE_DETECTOR | BL_SHARE_ERT)) return set_err(BL_ERR_INVALID, "unknown share flags");
  if (dst == src) return BL_OK;
  if (dst->device != src->device) return set_err(BL_ERR_INVALID, "contexts live on different devices");
  std::scoped_lock lk(dst->mu, src->mu);
  TRY(use_device(dst));
  TRY(quiesce_for_upload(dst));
  ++dst->model_gen;
  if (what & BL_SHARE_DETECTOR) {
    dst->detp = src->detp;
    for (Plan& p : dst->plans) p.valid = false;  // the plan follows the detector geometry
  }
  if (what & BL_SHARE_ERT) dst->ertp = src->ertp;
  return BL_OK;
}

int bl_host_alloc(size_t bytes, void** out) {
  if (!out) return set_err(BL_ERR_INVALID, "null argument");
  *out = nullptr;
  CK(cudaMallocHost(out, std::max<size_t>(bytes, 1)));
  return BL_OK;
}

void bl_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int bl_ctx_get_face_capacity(bl_ctx* c, int* faces_per_frame) {
  if (!c || !faces_per_frame) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  *faces_per_frame = c->face_cap_per_frame;
  return BL_OK;
}

int bl_submit(bl_ctx* c, const void* frames, int pixel_type, int n, int w, int h, size_t pitch, size_t frame_stride,
              int with_landmarks, uint64_t* ticket) {
  if (!c || !ticket) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (!(*c->detp).ready) return set_err(BL_ERR_STATE, "no detector model uploaded");
  if (with_landmarks && !(*c->ertp).ready) return set_err(BL_ERR_STATE, "no ERT model uploaded");
  if (with_landmarks < 0 || with_landmarks > BL_LANDMARKS_BEST)
    return set_err(BL_ERR_INVALID, "with_landmarks must be 0, BL_LANDMARKS_ALL or BL_LANDMARKS_BEST");
  if (frame_stride == 0) frame_stride = pitch * h;
  TRY(check_frames(frames, pixel_type, n, w, h, pitch, frame_stride));
  if (n < 1) return set_err(BL_ERR_INVALID, "empty batch");
  TRY(use_device(c));
  const uint64_t t = c->next_ticket;
  const int s = (int)(t % BL_MAX_IN_FLIGHT);
  if (c->slots[s].busy)
    return set_err(BL_ERR_STATE, "%d batches in flight: collect one before submitting", BL_MAX_IN_FLIGHT);
  const int n_lanes = (long long)n * w * h <= kSmallBatchPx ? kLanes : c->lanes_large;
  const int lane = c->timing ? 0 : (int)(t % n_lanes);
  if (lane > 0) {  // after whatever the caller queued on its stream (e.g. device-resident inputs)
    CK(cudaEventRecord(c->ev_lane, c->user));
    CK(cudaStreamWaitEvent(c->lanes[lane], c->ev_lane, 0));
  }
  c->plan = &c->plans[lane];
  c->st = lane ? c->lanes[lane] : c->user;
  const int rc = enqueue(c, s, frames, pixel_type, n, w, h, pitch, frame_stride, with_landmarks);
  c->plan = &c->plans[0];
  c->st = c->user;
  TRY(rc);
  c->slots[s].ticket = t;
  c->next_ticket = t + 1;
  *ticket = t;
  return BL_OK;
}

int bl_collect(bl_ctx* c, uint64_t ticket, bl_detection* out, int64_t cap, int32_t* counts, int64_t* total,
               double* landmarks) {
  if (!c) return set_err(BL_ERR_INVALID, "null context");
  std::lock_guard<std::mutex> lk(c->mu);
  const int s = (int)(ticket % BL_MAX_IN_FLIGHT);
  if (!c->slots[s].busy || c->slots[s].ticket != ticket) return set_err(BL_ERR_STATE, "unknown or collected ticket");
  TRY(use_device(c));
  return collect(c, s, out, cap, counts, total, landmarks);
}

int bl_landmarks(bl_ctx* c, const void* frames, int pixel_type, int n_frames, int w, int h, size_t pitch,
                 size_t frame_stride, const int32_t* frame_of_box, const bl_box* boxes, int64_t n_boxes,
                 double* out_xy, uint8_t* leaf_idx) {
  if (!c) return set_err(BL_ERR_INVALID, "null context");
  std::lock_guard<std::mutex> lk(c->mu);
  if (!(*c->ertp).ready) return set_err(BL_ERR_STATE, "no ERT model uploaded");
  if (frame_stride == 0) frame_stride = pitch * h;
  TRY(check_frames(frames, pixel_type, n_frames, w, h, pitch, frame_stride));
  if (n_boxes < 0 || n_boxes > (1 << 30)) return set_err(BL_ERR_INVALID, "bad box count");
  if (n_boxes == 0) return BL_OK;
  if (!boxes || !frame_of_box || !out_xy) return set_err(BL_ERR_INVALID, "null argument");
  TRY(use_device(c));
  // host-side validation of boxes (predict_landmarks' precondition, ert.cpp:101-102)
  std::vector<bl_box> hb(n_boxes);
  std::vector<int32_t> hf(n_boxes);
  CK(cudaMemcpy(hb.data(), boxes, sizeof(bl_box) * n_boxes, cudaMemcpyDefault));
  CK(cudaMemcpy(hf.data(), frame_of_box, sizeof(int32_t) * n_boxes, cudaMemcpyDefault));
  for (int64_t i = 0; i < n_boxes; ++i) {
    if (hb[i].w <= 0 || hb[i].h <= 0) return set_err(BL_ERR_INVALID, "predict_landmarks: face box must have positive area");
    if (hf[i] < 0 || hf[i] >= n_frames) return set_err(BL_ERR_INVALID, "frame_of_box out of range");
  }
  timing_begin(c);
  const void* dev = nullptr;
  long long dp = 0, df = 0;
  TRY(stage_input(c, c->ert_input, frames, pixel_type, n_frames, w, h, pitch, frame_stride, &dev, &dp, &df));
  TRY(c->ert_boxes.ensure(sizeof(bl_box) * n_boxes));
  TRY(c->ert_frames.ensure(sizeof(int32_t) * n_boxes));
  TRY(c->ert_nfaces.ensure(sizeof(int)));
  CK(cudaMemcpyAsync(c->ert_boxes.p, hb.data(), sizeof(bl_box) * n_boxes, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->ert_frames.p, hf.data(), sizeof(int32_t) * n_boxes, cudaMemcpyHostToDevice, c->st));
  const int nf = (int)n_boxes;
  CK(cudaMemcpyAsync(c->ert_nfaces.p, &nf, sizeof(int), cudaMemcpyHostToDevice, c->st));
  uint8_t* leaf_dev = nullptr;
  if (leaf_idx) {
    TRY(c->ert_leaf.ensure((size_t)n_boxes * (*c->ertp).dev.T * (*c->ertp).dev.K + 1));
    leaf_dev = c->ert_leaf.as<uint8_t>();
  }
  stage_mark(c, BL_STAGE_ERT);
  TRY(c->ert_out.ensure(sizeof(double) * 2 * (*c->ertp).dev.L * std::max(1, nf)));
  TRY(c->ert_err.ensure(sizeof(int)));
  TRY(run_ert(c, c->st, c->ert_work, dev, pixel_type, w, h, dp, df, c->ert_frames.as<int>(), c->ert_boxes.as<int>(), 4,
              c->ert_nfaces.as<int>(), nf, leaf_dev, c->ert_out.as<double>(), c->ert_err.as<int>(), nf));
  stage_mark(c, BL_STAGE_D2H);
  CK(cudaMemcpyAsync(out_xy, c->ert_out.p, sizeof(double) * 2 * (*c->ertp).dev.L * n_boxes, cudaMemcpyDefault, c->st));
  if (leaf_idx)
    CK(cudaMemcpyAsync(leaf_idx, leaf_dev, (size_t)n_boxes * (*c->ertp).dev.T * (*c->ertp).dev.K, cudaMemcpyDefault, c->st));
  CK(cudaStreamSynchronize(c->st));
  CK(cudaGetLastError());
  int err = 0;
  CK(cudaMemcpy(&err, c->ert_err.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (err == 1) return set_err(BL_ERR_INVALID, "similarity_transform: source shape has no spread");
  if (err == 2) return set_err(BL_ERR_INVALID, "similarity_transform: target shape has no spread");
  const int present[] = {BL_STAGE_H2D, BL_STAGE_ERT, BL_STAGE_D2H};
  timing_end(c, present, 3);
  return BL_OK;
}

// --------------------------------------------------------------- stage functions ----
int bl_build_pyramid(bl_ctx* c, const void* image, int pix, int w, int h, int window, double* out, size_t out_cap,
                     int* dims, double* scales, int max_levels, int* n_levels) {
  if (!c || !image || !n_levels) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  TRY(check_frames(image, pix, 1, w, h, w, (size_t)w * h));
  TRY(use_device(c));
  std::vector<int> lw, lh;
  pyramid_dims(w, h, window, lw, lh);
  const int nl = (int)lw.size();
  *n_levels = nl;
  size_t total = 0;
  std::vector<size_t> off(nl);
  for (int k = 0; k < nl; ++k) {
    off[k] = total;
    total += (size_t)lw[k] * lh[k];
    if (k < max_levels) {
      if (dims) {
        dims[2 * k] = lw[k];
        dims[2 * k + 1] = lh[k];
      }
      if (scales) scales[k] = k == 0 ? 1.0 : std::pow(5.0 / 6.0, double(k));  // image.cpp:169
    }
  }
  if (!out) return BL_OK;
  if (out_cap < total) return set_err(BL_ERR_CAPACITY, "pyramid needs %zu doubles", total);
  const size_t es = pix == BL_PIX_U8 ? 1 : 8;
  const void* src = nullptr;
  TRY(to_device(c, c->s_a, image, es * (size_t)w * h, &src));
  TRY(c->s_b.ensure(sizeof(double) * total));
  double* lv = c->s_b.as<double>();
  const Launch L = launch_of(c);
  if (pix == BL_PIX_U8) {
    // level 0 as doubles (exact widening)
    std::vector<uint8_t> tmp((size_t)w * h);
    CK(cudaMemcpyAsync(tmp.data(), src, tmp.size(), cudaMemcpyDefault, c->st));
    CK(cudaStreamSynchronize(c->st));
    std::vector<double> d(tmp.begin(), tmp.end());
    CK(cudaMemcpyAsync(lv, d.data(), sizeof(double) * d.size(), cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
  } else {
    CK(cudaMemcpyAsync(lv, src, sizeof(double) * (size_t)w * h, cudaMemcpyDefault, c->st));
  }
  for (int k = 1; k < nl; ++k)
    launch_resample(L, lv + off[k - 1], 0, lw[k - 1], lh[k - 1], lw[k - 1], (long long)lw[k - 1] * lh[k - 1],
                    lv + off[k], lw[k], lh[k], lw[k], (long long)lw[k] * lh[k], 1);
  return from_device(c, out, lv, sizeof(double) * total);
}

int bl_downscale_bilinear(bl_ctx* c, const double* image, int w, int h, double* out) {
  if (!c || !image || !out) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (w < 2 || h < 2) return set_err(BL_ERR_INVALID, "downscale_bilinear: output dimension would be 0");
  TRY(use_device(c));
  const int dw = w * 5 / 6, dh = h * 5 / 6;
  const void* src = nullptr;
  TRY(to_device(c, c->s_a, image, sizeof(double) * w * h, &src));
  TRY(c->s_b.ensure(sizeof(double) * dw * dh));
  launch_resample(launch_of(c), src, 0, w, h, w, (long long)w * h, c->s_b.as<double>(), dw, dh, dw, (long long)dw * dh, 1);
  return from_device(c, out, c->s_b.p, sizeof(double) * dw * dh);
}

int bl_compute_gradients(bl_ctx* c, const double* image, int w, int h, uint8_t* ori, double* mag) {
  if (!c || !image || !ori || !mag) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (w < 3 || h < 3) return set_err(BL_ERR_INVALID, "compute_gradients: image must be at least 3x3");
  TRY(use_device(c));
  const void* src = nullptr;
  TRY(to_device(c, c->s_a, image, sizeof(double) * w * h, &src));
  TRY(c->s_b.ensure(sizeof(double) * w * h));
  TRY(c->s_c.ensure((size_t)w * h));
  PlanDesc H;
  single_level_plan(H, w, h, w / 8, h / 8);
  TRY(c->s_desc.ensure(sizeof(PlanDesc)));
  CK(cudaMemcpyAsync(c->s_desc.p, &H, sizeof H, cudaMemcpyHostToDevice, c->st));
  launch_grad(launch_of(c), H, c->s_desc.as<PlanDesc>(), 0, 1, src, 1, c->s_b.as<double>(), c->s_c.as<uint8_t>());
  CK(cudaMemcpyAsync(ori, c->s_c.p, (size_t)w * h, cudaMemcpyDefault, c->st));
  return from_device(c, mag, c->s_b.p, sizeof(double) * w * h);
}

int bl_histogramize(bl_ctx* c, const uint8_t* ori, const double* mag, int w, int h, double* bins) {
  if (!c || !ori || !mag || !bins) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (w < 1 || h < 1) return set_err(BL_ERR_INVALID, "bad dims");
  TRY(use_device(c));
  const int cw = w / 8, ch = h / 8;
  if (cw == 0 || ch == 0) return BL_OK;
  const void *o = nullptr, *m = nullptr;
  TRY(to_device(c, c->s_a, mag, sizeof(double) * w * h, &m));
  TRY(to_device(c, c->s_c, ori, (size_t)w * h, &o));
  PlanDesc H;
  single_level_plan(H, w, h, cw, ch);
  TRY(c->s_desc.ensure(sizeof(PlanDesc)));
  CK(cudaMemcpyAsync(c->s_desc.p, &H, sizeof H, cudaMemcpyHostToDevice, c->st));
  TRY(c->s_b.ensure(sizeof(double) * kBins * cw * ch));
  launch_gradhist(launch_of(c), H, c->s_desc.as<PlanDesc>(), (const double*)m, (const uint8_t*)o,
                  c->s_b.as<double>(), nullptr);
  return from_device(c, bins, c->s_b.p, sizeof(double) * kBins * cw * ch);
}

int bl_cell_energy(bl_ctx* c, const double* bins, int cw, int ch, double* energy) {
  if (!c || !bins || !energy) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (cw < 0 || ch < 0) return set_err(BL_ERR_INVALID, "bad dims");
  TRY(use_device(c));
  const long long cells = (long long)cw * ch;
  if (cells == 0) return BL_OK;
  const void* b = nullptr;
  TRY(to_device(c, c->s_a, bins, sizeof(double) * kBins * cells, &b));
  TRY(c->s_b.ensure(sizeof(double) * cells));
  launch_energy(launch_of(c), (const double*)b, cells, c->s_b.as<double>());
  return from_device(c, energy, c->s_b.p, sizeof(double) * cells);
}

int bl_compute_features(bl_ctx* c, const double* bins, const double* energy, int cw, int ch, double* features) {
  if (!c || !bins || !energy || !features) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (cw < 0 || ch < 0) return set_err(BL_ERR_INVALID, "bad dims");
  TRY(use_device(c));
  const long long cells = (long long)cw * ch;
  if (cells == 0) return BL_OK;
  const void *b = nullptr, *e = nullptr;
  TRY(to_device(c, c->s_a, bins, sizeof(double) * kBins * cells, &b));
  TRY(to_device(c, c->s_b, energy, sizeof(double) * cells, &e));
  PlanDesc H;
  single_level_plan(H, cw * 8, ch * 8, cw, ch);
  TRY(c->s_desc.ensure(sizeof(PlanDesc)));
  CK(cudaMemcpyAsync(c->s_desc.p, &H, sizeof H, cudaMemcpyHostToDevice, c->st));
  TRY(c->s_c.ensure(sizeof(double) * kFeat * cells));
  launch_features(launch_of(c), H, c->s_desc.as<PlanDesc>(), (const double*)b, (const double*)e,
                  c->s_c.as<double>(), nullptr, nullptr);
  return from_device(c, features, c->s_c.p, sizeof(double) * kFeat * cells);
}

int bl_extract_features(bl_ctx* c, const double* image, int w, int h, double* features, double* bins,
                        double* energy) {
  if (!c || !image || !features) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (w < 3 || h < 3) return set_err(BL_ERR_INVALID, "compute_gradients: image must be at least 3x3");
  TRY(use_device(c));
  const int cw = w / 8, ch = h / 8;
  const long long cells = (long long)cw * ch;
  if (cells == 0) return BL_OK;
  const void* src = nullptr;
  TRY(to_device(c, c->s_a, image, sizeof(double) * w * h, &src));
  PlanDesc H;
  single_level_plan(H, w, h, cw, ch);
  TRY(c->s_desc.ensure(sizeof(PlanDesc)));
  CK(cudaMemcpyAsync(c->s_desc.p, &H, sizeof H, cudaMemcpyHostToDevice, c->st));
  TRY(c->s_b.ensure(sizeof(double) * kBins * cells));
  TRY(c->s_c.ensure(sizeof(double) * cells));
  TRY(c->s_d.ensure(sizeof(double) * kFeat * cells));
  const Launch L = launch_of(c);
  launch_hog(L, H, c->s_desc.as<PlanDesc>(), 0, 1, src, 1, c->s_b.as<double>(), c->s_c.as<double>());
  launch_features(L, H, c->s_desc.as<PlanDesc>(), c->s_b.as<double>(), c->s_c.as<double>(), c->s_d.as<double>(),
                  nullptr, nullptr);
  if (bins) CK(cudaMemcpyAsync(bins, c->s_b.p, sizeof(double) * kBins * cells, cudaMemcpyDefault, c->st));
  if (energy) CK(cudaMemcpyAsync(energy, c->s_c.p, sizeof(double) * cells, cudaMemcpyDefault, c->st));
  return from_device(c, features, c->s_d.p, sizeof(double) * kFeat * cells);
}

int bl_score_window(bl_ctx* c, const double* features, int cw, int ch, const double* weights, double bias,
                    double* scores) {
  if (!c || !features || !weights || !scores) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (cw < kWin || ch < kWin) return set_err(BL_ERR_INVALID, "feature image smaller than the 10x10 detection window");
  TRY(use_device(c));
  const long long cells = (long long)cw * ch;
  const long long n = (long long)(cw - 9) * (ch - 9);
  const void *f = nullptr, *wt = nullptr;
  TRY(to_device(c, c->s_a, features, sizeof(double) * kFeat * cells, &f));
  TRY(to_device(c, c->s_b, weights, sizeof(double) * kFilterW, &wt));
  TRY(c->s_c.ensure(sizeof(double) * n));
  launch_score_exact_all(launch_of(c), (const double*)f, cw, ch, (const double*)wt, bias, c->s_c.as<double>());
  return from_device(c, scores, c->s_c.p, sizeof(double) * n);
}

int bl_score_window_dense(bl_ctx* c, const double* features, int cw, int ch, const double* weights, double bias,
                          double* scores) {
  if (!c || !features || !weights || !scores) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (cw < kWin || ch < kWin) return set_err(BL_ERR_INVALID, "feature image smaller than the 10x10 detection window");
  TRY(use_device(c));
  const long long cells = (long long)cw * ch;
  const long long n = (long long)(cw - 9) * (ch - 9);
  const void *f = nullptr, *wt = nullptr;
  TRY(to_device(c, c->s_a, features, sizeof(double) * kFeat * cells, &f));
  TRY(to_device(c, c->s_b, weights, sizeof(double) * kFilterW, &wt));
  TRY(c->s_c.ensure(sizeof(double) * n));
  launch_score_dense(launch_of(c), (const double*)f, cw, ch, (const double*)wt, bias, c->s_c.as<double>());
  return from_device(c, scores, c->s_c.p, sizeof(double) * n);
}

int bl_nms(bl_ctx* c, const bl_detection* dets, int64_t n, double iou_threshold, bl_detection* out, int64_t* kept) {
  if (!c || (!dets && n > 0) || !out || !kept) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  *kept = 0;
  if (n <= 0) return BL_OK;
  if (n > (1ll << 26)) return set_err(BL_ERR_CAPACITY, "too many detections");
  TRY(use_device(c));
  TRY(c->s_a.ensure(sizeof(bl_detection) * n));
  TRY(c->s_b.ensure(sizeof(bl_detection) * n));
  TRY(c->s_c.ensure(sizeof(int) * 2));
  const long long gk = nms_gkeys_per_frame(n);
  if (gk) TRY(c->s_d.ensure(nms_key_bytes() * gk));
  CK(cudaMemcpyAsync(c->s_a.p, dets, sizeof(bl_detection) * n, cudaMemcpyDefault, c->st));
  const int cnt = (int)n;
  CK(cudaMemcpyAsync(c->s_c.p, &cnt, sizeof(int), cudaMemcpyHostToDevice, c->st));
  launch_nms(launch_of(c), c->s_a.as<DevDet>(), c->s_c.as<int>(), n, 1, iou_threshold, c->s_b.as<DevDet>(),
             c->s_c.as<int>() + 1, c->s_d.p, gk);
  int k = 0;
  CK(cudaMemcpyAsync(&k, c->s_c.as<int>() + 1, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  *kept = k;
  return from_device(c, out, c->s_b.p, sizeof(bl_detection) * k);
}

int bl_orientation_bins(bl_ctx* c, const double* gx, const double* gy, int64_t n, uint8_t* bins) {
  if (!c || !gx || !gy || !bins) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (n <= 0) return BL_OK;
  TRY(use_device(c));
  const void *a = nullptr, *b = nullptr;
  TRY(to_device(c, c->s_a, gx, sizeof(double) * n, &a));
  TRY(to_device(c, c->s_b, gy, sizeof(double) * n, &b));
  TRY(c->s_c.ensure((size_t)n));
  launch_orientation(launch_of(c), (const double*)a, (const double*)b, n, c->s_c.as<uint8_t>());
  return from_device(c, bins, c->s_c.p, (size_t)n);
}

int bl_debug_sqrt(bl_ctx* c, const double* in, int64_t n, double* fast, double* ieee) {
  if (!c || !in || !fast || !ieee) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (n <= 0) return BL_OK;
  TRY(use_device(c));
  const void* a = nullptr;
  TRY(to_device(c, c->s_a, in, sizeof(double) * n, &a));
  TRY(c->s_b.ensure(sizeof(double) * n));
  TRY(c->s_c.ensure(sizeof(double) * n));
  launch_sqrt_check(launch_of(c), (const double*)a, n, c->s_b.as<double>(), c->s_c.as<double>());
  CK(cudaMemcpyAsync(fast, c->s_b.p, sizeof(double) * n, cudaMemcpyDefault, c->st));
  return from_device(c, ieee, c->s_c.p, sizeof(double) * n);
}


int bl_debug_screen_tc(bl_ctx* c, const double* features, int cw, int ch, float* scores, double* delta) {
  if (!c || !features || !scores) return set_err(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (!(*c->detp).ready) return set_err(BL_ERR_STATE, "no detector model uploaded");
  if (cw < kWin || ch < kWin) return set_err(BL_ERR_INVALID, "feature image smaller than the 10x10 detection window");
  TRY(use_device(c));
  PlanDesc H;
  single_level_plan(H, cw * 8, ch * 8, cw, ch);
  LevelDesc& Lv = H.lv[0];
  const size_t nfl = tc_feat_floats_per_frame(cw, ch, &Lv.tc_ncp, nullptr);
  Lv.tc_off = 0;
  std::vector<uint16_t> h16(2 * nfl, 0);  // fp16 planes, as k_features writes them
  for (long long cell = 0; cell < (long long)cw * ch; ++cell)
    for (int f = 0; f < kFeat; ++f)
      h16[((size_t)(f / 8) * Lv.tc_ncp + cell) * 8 + f % 8] =
          half_rn_host(std::ldexp(features[cell * kFeat + f], kTcFeatExp));
  std::vector<float> host(nfl);
  std::memcpy(host.data(), h16.data(), sizeof(float) * nfl);
  const long long na = (long long)Lv.sw * Lv.sh;
  TRY(c->s_a.ensure(sizeof(float) * nfl));
  TRY(c->s_b.ensure(sizeof(float) * kFilters * na));
  TRY(c->s_c.ensure(sizeof(Candidate) * na + sizeof(unsigned long long)));
  TRY(c->s_desc.ensure(sizeof(PlanDesc)));
  CK(cudaMemcpyAsync(c->s_a.p, host.data(), sizeof(float) * nfl, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->s_desc.p, &H, sizeof H, cudaMemcpyHostToDevice, c->st));
  unsigned long long* nc = reinterpret_cast<unsigned long long*>(c->s_c.as<Candidate>() + na);
  CK(cudaMemsetAsync(nc, 0, sizeof(unsigned long long), c->st));
  launch_screen_tc(launch_of(c), H, c->s_desc.as<PlanDesc>(), c->s_a.as<float>(), (*c->detp).w_tc.as<float>(),
                   (*c->detp).cuttc.as<float>(), c->s_c.as<Candidate>(), nc, na, c->s_b.as<float>());
  if (delta)
    for (int r = 0; r < kFilters; ++r) delta[r] = (*c->detp).delta_tc[r];
  return from_device(c, scores, c->s_b.p, sizeof(float) * kFilters * na);
}

}  // extern "C"
