// Multi-device frame sharding (the reference's frame-parallel worker pool,
// pipeline.cpp:230-324, moved from CPU threads to GPUs).  Frames are independent, so a batch
// is split into contiguous per-device shards (the same rule as sharding.shard_range: sizes
// differ by at most one, lower ranks take the extra frame), each device runs the whole
// detect + landmark path on its shard with its own model replica, driven by its own host
// worker thread through the pipelined bl_submit / bl_collect pair, and the results are
// concatenated in frame order -- the order restoration pipeline.cpp:302-303 does.  No
// collective touches the data path: the only cross-device step is the host-side gather.
//
// Host C++ on top of the C-ABI only (no CUDA types): every device call is a bl_* call on the
// worker's own context.
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/blinkline_b200.h"

namespace blb {
void set_last_error(const char* msg);
}

namespace {

int fail(int code, const std::string& msg) {
  blb::set_last_error(msg.c_str());
  return code;
}

// One device: its context and a persistent host thread that runs jobs on it.
struct Worker {
  int device = 0;
  bl_ctx* ctx = nullptr;
  std::thread th;
  std::mutex mu;
  std::condition_variable cv;
  std::function<int()> job;
  bool has_job = false, done = false, quit = false;
  int rc = BL_OK;
  std::string err;
  double ms = 0;
  // the shard's results
  std::vector<bl_detection> dets;
  std::vector<int32_t> counts;
  std::vector<double> landmarks;

  void loop() {
    std::unique_lock<std::mutex> lk(mu);
    while (true) {
      cv.wait(lk, [&] { return has_job || quit; });
      if (quit) return;
      std::function<int()> f = std::move(job);
      has_job = false;
      lk.unlock();
      const auto t0 = std::chrono::steady_clock::now();
      const int r = f();
      const double dt = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      std::string e = r == BL_OK ? std::string() : std::string(bl_last_error());
      lk.lock();
      rc = r;
      err = e;
      ms = dt;
      done = true;
      cv.notify_all();
    }
  }
  void post(std::function<int()> f) {
    std::lock_guard<std::mutex> lk(mu);
    job = std::move(f);
    has_job = true;
    done = false;
    cv.notify_all();
  }
  int wait() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return done; });
    return rc;
  }
};

// Contiguous [begin, end) of shard r of n frames over `world` devices (sharding.shard_range).
void shard_range(long long n, int r, int world, long long* b, long long* e) {
  const long long base = n / world, extra = n % world;
  *b = r * base + std::min<long long>(r, extra);
  *e = *b + base + (r < extra ? 1 : 0);
}

}  // namespace

struct bl_multi {
  std::vector<std::unique_ptr<Worker>> w;
  long long px_per_submit = 160LL << 20;  // ~512 VGA frames, ~80 1080p frames per submitted batch
  std::mutex call_mu;
};

namespace {

// Detect (+ landmarks) over frames [b, e) on worker W: batches of `chunk` frames, up to
// BL_MAX_IN_FLIGHT in flight, results appended in frame order.
int run_shard(Worker& W, const char* frames, int pix, long long b, long long e, int w, int h, size_t pitch,
              size_t fstride, int with_landmarks, int L, long long chunk) {
  const size_t es = pix == BL_PIX_U8 ? 1 : 8;
  W.dets.clear();
  W.counts.assign((size_t)(e - b), 0);
  W.landmarks.clear();
  struct Pending {
    uint64_t ticket;
    long long first, n;
  };
  std::vector<Pending> q;
  long long next = b;
  auto submit_one = [&]() -> int {
    const long long n = std::min(chunk, e - next);
    uint64_t t = 0;
    if (int rc = bl_submit(W.ctx, frames + es * fstride * next, pix, (int)n, w, h, pitch, fstride, with_landmarks, &t))
      return rc;
    q.push_back({t, next, n});
    next += n;
    return BL_OK;
  };
  int fc = 0;
  if (int rc = bl_ctx_get_face_capacity(W.ctx, &fc)) return rc;
  int rc = BL_OK;
  while (rc == BL_OK && next < e && (int)q.size() < BL_MAX_IN_FLIGHT) rc = submit_one();
  std::vector<bl_detection> out;
  std::vector<double> lm;
  while (!q.empty()) {
    const Pending p = q.front();
    q.erase(q.begin());
    // room for the batch's whole device face capacity: a short output buffer never happens, so
    // BL_ERR_CAPACITY means the device capacity itself was exceeded (bl_ctx_set_face_capacity)
    const int64_t cap = std::max<int64_t>(1, p.n * (int64_t)fc);
    if ((int64_t)out.size() < cap) out.resize((size_t)cap);
    if (with_landmarks && (int64_t)lm.size() < cap * L * 2) lm.resize((size_t)(cap * L * 2));
    int64_t total = 0;
    if (rc == BL_OK) {
      rc = bl_collect(W.ctx, p.ticket, out.data(), cap, W.counts.data() + (p.first - b), &total,
                      with_landmarks ? lm.data() : nullptr);
      if (rc == BL_OK) {
        W.dets.insert(W.dets.end(), out.begin(), out.begin() + total);
        if (with_landmarks) W.landmarks.insert(W.landmarks.end(), lm.begin(), lm.begin() + total * L * 2);
        if (next < e) rc = submit_one();
      }
    } else {  // an earlier batch failed: drain the rest so the context stays usable
      std::vector<int32_t> scratch((size_t)p.n);
      const std::string keep = bl_last_error();
      bl_collect(W.ctx, p.ticket, out.data(), cap, scratch.data(), &total, with_landmarks ? lm.data() : nullptr);
      blb::set_last_error(keep.c_str());
    }
  }
  return rc;
}

}  // namespace

extern "C" {

int bl_multi_create(const int* devices, int n_devices, bl_multi** out) {
  if (!out || !devices || n_devices < 1) return fail(BL_ERR_INVALID, "bl_multi_create: need at least one device");
  *out = nullptr;
  auto m = std::make_unique<bl_multi>();
  for (int i = 0; i < n_devices; ++i) {
    auto W = std::make_unique<Worker>();
    W->device = devices[i];
    if (int rc = bl_ctx_create(devices[i], &W->ctx)) {
      for (auto& o : m->w) {
        {
          std::lock_guard<std::mutex> lk(o->mu);
          o->quit = true;
          o->cv.notify_all();
        }
        o->th.join();
        bl_ctx_destroy(o->ctx);
      }
      return rc;
    }
    Worker* wp = W.get();
    W->th = std::thread([wp] { wp->loop(); });
    m->w.push_back(std::move(W));
  }
  *out = m.release();
  return BL_OK;
}

void bl_multi_destroy(bl_multi* m) {
  if (!m) return;
  for (auto& W : m->w) {
    {
      std::lock_guard<std::mutex> lk(W->mu);
      W->quit = true;
      W->cv.notify_all();
    }
    W->th.join();
    bl_ctx_destroy(W->ctx);
  }
  delete m;
}

int bl_multi_size(bl_multi* m, int* n_devices) {
  if (!m || !n_devices) return fail(BL_ERR_INVALID, "null argument");
  *n_devices = (int)m->w.size();
  return BL_OK;
}

int bl_multi_context(bl_multi* m, int i, bl_ctx** ctx) {
  if (!m || !ctx) return fail(BL_ERR_INVALID, "null argument");
  if (i < 0 || i >= (int)m->w.size()) return fail(BL_ERR_INVALID, "device slot out of range");
  *ctx = m->w[i]->ctx;
  return BL_OK;
}

int bl_multi_set_batch_pixels(bl_multi* m, int64_t pixels_per_submit) {
  if (!m || pixels_per_submit < 1) return fail(BL_ERR_INVALID, "bad batch size");
  std::lock_guard<std::mutex> lk(m->call_mu);
  m->px_per_submit = pixels_per_submit;
  return BL_OK;
}

int bl_multi_detector_upload(bl_multi* m, const double* weights, const double* biases, double threshold,
                             int window_cells, int cell_px, int scale_num, int scale_den, double min_face_ratio) {
  if (!m) return fail(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(m->call_mu);
  for (auto& W : m->w)
    if (int rc = bl_detector_upload(W->ctx, weights, biases, threshold, window_cells, cell_px, scale_num, scale_den,
                                    min_face_ratio))
      return rc;
  return BL_OK;
}

int bl_multi_ert_upload(bl_multi* m, int L, int T, int K, int F, double shrinkage, const double* mean_xy,
                        const int32_t* anchors, const double* split_params, const double* leaves) {
  if (!m) return fail(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(m->call_mu);
  for (auto& W : m->w)
    if (int rc = bl_ert_upload(W->ctx, L, T, K, F, shrinkage, mean_xy, anchors, split_params, leaves)) return rc;
  return BL_OK;
}

int bl_multi_detect_landmarks(bl_multi* m, const void* frames, int pixel_type, int n, int w, int h, size_t pitch,
                              size_t frame_stride, bl_detection* out, int64_t cap, int32_t* counts, int64_t* total,
                              double* landmarks, double* device_ms) {
  if (!m) return fail(BL_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(m->call_mu);
  if (total) *total = 0;
  if (n < 0) return fail(BL_ERR_INVALID, "negative frame count");
  if (n == 0) return BL_OK;
  if (!frames) return fail(BL_ERR_INVALID, "frames is NULL");
  if (pixel_type != BL_PIX_U8 && pixel_type != BL_PIX_F64) return fail(BL_ERR_INVALID, "unknown pixel type");
  if (w < 1 || h < 1) return fail(BL_ERR_INVALID, "make_image: dimensions must be >= 1");
  if (pitch < (size_t)w) return fail(BL_ERR_INVALID, "pitch < width");
  if (frame_stride == 0) frame_stride = pitch * h;
  int L = 0;
  const int with_lm = landmarks != nullptr;
  if (with_lm)
    if (int rc = bl_ctx_model_info(m->w[0]->ctx, &L)) return rc;
  const int world = (int)m->w.size();
  const long long chunk = std::max<long long>(1, m->px_per_submit / ((long long)w * h));
  for (int r = 0; r < world; ++r) {
    long long b = 0, e = 0;
    shard_range(n, r, world, &b, &e);
    Worker* W = m->w[r].get();
    W->post([=]() -> int {
      if (e <= b) {
        W->dets.clear();
        W->counts.clear();
        W->landmarks.clear();
        return BL_OK;
      }
      return run_shard(*W, static_cast<const char*>(frames), pixel_type, b, e, w, h, pitch, frame_stride, with_lm, L,
                       chunk);
    });
  }
  int first_rc = BL_OK;
  std::string first_err;
  for (int r = 0; r < world; ++r) {
    const int rc = m->w[r]->wait();
    if (device_ms) device_ms[r] = m->w[r]->ms;
    if (rc && first_rc == BL_OK) {
      first_rc = rc;
      first_err = "device " + std::to_string(m->w[r]->device) + ": " + m->w[r]->err;
    }
  }
  if (first_rc) return fail(first_rc, first_err);
  // gather in frame order: shards are contiguous and ascending
  int64_t tot = 0;
  for (auto& W : m->w) tot += (int64_t)W->dets.size();
  if (total) *total = tot;
  if (tot > cap) return fail(BL_ERR_CAPACITY, "output capacity " + std::to_string(cap) + " < " + std::to_string(tot) +
                                                   " detections");
  int64_t off = 0, fo = 0;
  for (auto& W : m->w) {
    if (counts && !W->counts.empty()) std::memcpy(counts + fo, W->counts.data(), sizeof(int32_t) * W->counts.size());
    fo += (int64_t)W->counts.size();
    if (out && !W->dets.empty()) std::memcpy(out + off, W->dets.data(), sizeof(bl_detection) * W->dets.size());
    if (with_lm && !W->landmarks.empty())
      std::memcpy(landmarks + off * L * 2, W->landmarks.data(), sizeof(double) * W->landmarks.size());
    off += (int64_t)W->dets.size();
  }
  return BL_OK;
}

}  // extern "C"
