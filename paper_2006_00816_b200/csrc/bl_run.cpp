// The GPU-backed frame-sequence runtime: the reference's
// ingest() / run() (pipeline.hpp:24-60, pipeline.cpp:36-66, 150-190, 358-404) with the
// detect and landmark stages on the device, batched, and the decode of the next batch
// overlapped with the device work of the current one; plus the EAR / blink-trace fold
// (blink.hpp:16-70, blink.cpp:13-135) on the results, on the host (O(frames) scalars).
//
// Results are the reference's, frame for frame: detections bit-identical (the device path),
// the face of a frame is its first post-NMS detection (NMS order: best first,
// pipeline.cpp:167), landmarks are predicted for that face only (pipeline.cpp:184), EARs and
// the trace follow blink.cpp's definitions (linear-interpolation quantile baseline,
// closure = clamp(1 - ear / baseline, 0, 1)).  Sequential (batch 1) and pipelined runs give
// identical results, like the reference's modes (acceptance C8).
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <string>
#include <thread>
#include <vector>

#include "../../include/blinkline_b200.h"

namespace blb {
void set_last_error(const char* msg);
}

namespace {

namespace fs = std::filesystem;
using Clock = std::chrono::steady_clock;

int fail(int code, const std::string& msg) {
  blb::set_last_error(msg.c_str());
  return code;
}

double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

std::string frame_name(size_t i) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "frame_%06zu.pgm", i);
  return buf;
}

// ingest (pipeline.cpp:358-394): frame_%06d.pgm numbered from 0 without gaps, equal dims.
int ingest(const char* dir, std::vector<std::string>& paths, int& w, int& h) {
  const std::string d(dir);
  std::error_code ec;
  if (!fs::is_directory(d, ec)) return fail(BL_ERR_IO, d + ": not a directory");
  size_t max_index = 0;
  bool any = false;
  for (const auto& e : fs::directory_iterator(d, ec)) {
    if (!e.is_regular_file()) continue;
    const std::string name = e.path().filename().string();
    size_t idx = 0;
    if (std::sscanf(name.c_str(), "frame_%zu.pgm", &idx) == 1 && name == frame_name(idx)) {
      any = true;
      max_index = std::max(max_index, idx);
    }
  }
  if (!any) return fail(BL_ERR_IO, d + ": no frame_%06d.pgm files found");
  paths.clear();
  for (size_t i = 0; i <= max_index; ++i) {
    const fs::path p = fs::path(d) / frame_name(i);
    if (!fs::exists(p)) return fail(BL_ERR_IO, d + ": gap in frame numbering, missing " + frame_name(i));
    paths.push_back(p.string());
  }
  for (size_t i = 0; i < paths.size(); ++i) {
    int fw = 0, fh = 0;
    if (int rc = bl_read_pgm(paths[i].c_str(), &fw, &fh, nullptr, 0)) return rc;  // header only
    if (i == 0) {
      w = fw;
      h = fh;
    } else if (fw != w || fh != h) {
      return fail(BL_ERR_IO, paths[i] + ": dimension change mid-sequence (" + std::to_string(fw) + "x" +
                                 std::to_string(fh) + " vs " + std::to_string(w) + "x" + std::to_string(h) + ")");
    }
  }
  return BL_OK;
}

// blink.cpp:15, 40-45: EAR = (|p2-p6| + |p3-p5|) / (2 |p1-p4|) with std::hypot distances.
double dist(const double* a, const double* b) { return std::hypot(a[0] - b[0], a[1] - b[1]); }

int eye_ear(const double* lm, const int* eye, double& ear) {
  const double* p[6];
  for (int i = 0; i < 6; ++i) p[i] = lm + 2 * eye[i];
  const double horiz = dist(p[0], p[3]);
  if (horiz <= 1e-9) return fail(BL_ERR_INVALID, "eye_aspect_ratio: degenerate eye, corner span ~ 0");
  ear = (dist(p[1], p[5]) + dist(p[2], p[4])) / (2.0 * horiz);
  return BL_OK;
}

// blink.cpp:17-26: linear interpolation over the sorted values.
double quantile(std::vector<double> v, double q) {
  std::sort(v.begin(), v.end());
  if (v.size() == 1) return v[0];
  const double pos = q * double(v.size() - 1);
  const size_t lo = size_t(pos);
  if (lo + 1 >= v.size()) return v.back();
  const double frac = pos - double(lo);
  return v[lo] + frac * (v[lo + 1] - v[lo]);
}

double closure_of(double ear, double baseline) {  // blink.cpp:28-31
  if (baseline <= 0.0) return 1.0;
  return std::clamp(1.0 - ear / baseline, 0.0, 1.0);
}

}  // namespace

extern "C" {

int bl_ingest(const char* frames_dir, int* n_frames, int* w, int* h) {
  if (!frames_dir || !n_frames || !w || !h) return fail(BL_ERR_INVALID, "null argument");
  std::vector<std::string> paths;
  if (int rc = ingest(frames_dir, paths, *w, *h)) return rc;
  *n_frames = (int)paths.size();
  return BL_OK;
}

int bl_run(bl_ctx* ctx, const char* frames_dir, double fps, int batch_size, bl_frame_result* frames,
           int64_t frames_cap, bl_detection* dets, int64_t det_cap, int64_t* det_total, double* landmarks,
           double* baselines) {
  if (!ctx || !frames_dir || !frames || !dets || !det_total || !landmarks) return fail(BL_ERR_INVALID, "null argument");
  if (batch_size < 1) return fail(BL_ERR_INVALID, "batch_size must be >= 1");
  int L = 0;
  if (int rc = bl_ctx_model_info(ctx, &L)) return rc;
  if (L != 68)  // eye_indices (ert.cpp:340-347), called by run_stats before any frame
    return fail(BL_ERR_INVALID, "eye_indices: no eye mapping for L=" + std::to_string(L) +
                                    "; only the 68-landmark convention is built in");
  static const int kLeft[6] = {36, 37, 38, 39, 40, 41}, kRight[6] = {42, 43, 44, 45, 46, 47};
  std::vector<std::string> paths;
  int w = 0, h = 0;
  if (int rc = ingest(frames_dir, paths, w, h)) return rc;
  const int64_t n = (int64_t)paths.size();
  if (n > frames_cap) return fail(BL_ERR_CAPACITY, "frame result buffer holds " + std::to_string(frames_cap) +
                                                       " < " + std::to_string(n) + " frames");
  const size_t fpx = (size_t)w * h;
  const int B = (int)std::min<int64_t>(batch_size, n);
  const int64_t n_batches = (n + B - 1) / B;

  // Decode ring: kDecoders persistent decoder threads (batch b on thread b % kDecoders) parse
  // PGMs straight to u8 into pinned buffer b % kRing while the device works on up to
  // BL_MAX_IN_FLIGHT earlier batches (one upload per batch; detection and the best face's
  // landmarks run in the same device pass).
  const int kDecoders = (int)std::max<unsigned>(1u, std::min<unsigned>(4u, std::thread::hardware_concurrency() / 2));
  const int kRing = BL_MAX_IN_FLIGHT + kDecoders;
  struct RingBuf {
    uint8_t* p = nullptr;
    int64_t batch = -1;  // batch decoded into it (ready), -1: free
    int rc = BL_OK;
    std::string err;
  };
  std::vector<RingBuf> ring(kRing);
  for (RingBuf& r : ring)
    if (int rc = bl_host_alloc(fpx * B, reinterpret_cast<void**>(&r.p))) {
      for (RingBuf& q : ring) bl_host_free(q.p);
      return rc;
    }
  std::vector<double> dec_ms(n, 0.0);
  std::mutex mu;
  std::condition_variable cv;
  bool stop = false;
  auto decode_loop = [&](int who) {
    for (int64_t b = who; b < n_batches; b += kDecoders) {
      RingBuf& r = ring[b % kRing];
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return stop || r.batch < 0; });
        if (stop) return;
      }
      const int64_t b0 = b * B;
      const int nb = (int)std::min<int64_t>(B, n - b0);
      int rc = BL_OK;
      for (int i = 0; i < nb && rc == BL_OK; ++i) {
        const auto t0 = Clock::now();
        int fw = 0, fh = 0;
        rc = bl_read_pgm(paths[b0 + i].c_str(), &fw, &fh, r.p + fpx * i, fpx);
        dec_ms[b0 + i] = ms_since(t0);
      }
      std::lock_guard<std::mutex> lk(mu);
      r.rc = rc;
      if (rc) r.err = bl_last_error();
      r.batch = b;
      cv.notify_all();
      if (rc) return;
    }
  };
  std::vector<std::thread> decoders;
  for (int d = 0; d < kDecoders; ++d) decoders.emplace_back(decode_loop, d);
  auto finish = [&](int rc) {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
      cv.notify_all();
    }
    for (std::thread& t : decoders) t.join();
    for (RingBuf& r : ring) bl_host_free(r.p);
    return rc;
  };

  struct Pending {
    uint64_t ticket;
    int64_t b;
    Clock::time_point t0;
  };
  std::vector<Pending> q;
  std::vector<int32_t> counts(B);
  std::vector<double> xy((size_t)B * 2 * L);
  int64_t total = 0;
  // results of batch p, in frame order (detect_frame + landmark_frame, pipeline.cpp:159-190)
  auto collect_one = [&](const Pending& p) -> int {
    const int64_t b0 = p.b * B;
    const int nb = (int)std::min<int64_t>(B, n - b0);
    int64_t got = 0;
    int rc = bl_collect(ctx, p.ticket, dets + total, det_cap - total, counts.data(), &got, xy.data());
    const double batch_ms = ms_since(p.t0);
    {
      std::lock_guard<std::mutex> lk(mu);
      ring[p.b % kRing].batch = -1;  // the decoder may refill it
      cv.notify_all();
    }
    if (rc) return rc;
    int64_t off = total;
    for (int i = 0; i < nb && rc == BL_OK; ++i) {
      bl_frame_result& fr = frames[b0 + i];
      std::memset(&fr, 0, sizeof fr);
      fr.frame_index = (int32_t)(b0 + i);
      fr.n_detections = counts[i];
      fr.t = double(b0 + i) / fps;
      fr.decode_ms = dec_ms[b0 + i];
      fr.detect_ms = batch_ms / nb;  // submit -> results, detection + landmarks in one device pass
      fr.landmark_ms = 0.0;
      if (counts[i] > 0) {  // the face = the first (best) detection, pipeline.cpp:167
        fr.face_found = 1;
        fr.face = dets[off];
        const double* pxy = xy.data() + (size_t)i * 2 * L;
        std::memcpy(landmarks + (b0 + i) * 2 * (int64_t)L, pxy, sizeof(double) * 2 * L);
        rc = eye_ear(pxy, kLeft, fr.ear_left);
        if (rc == BL_OK) rc = eye_ear(pxy, kRight, fr.ear_right);
      }
      off += counts[i];
    }
    total = off;
    return rc;
  };
  int rc = BL_OK;
  for (int64_t b = 0; b < n_batches && rc == BL_OK; ++b) {
    RingBuf& r = ring[b % kRing];
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return r.batch == b; });
      if (r.rc) {
        blb::set_last_error(r.err.c_str());
        rc = r.rc;
        break;
      }
    }
    if ((int)q.size() == BL_MAX_IN_FLIGHT) {
      rc = collect_one(q.front());
      q.erase(q.begin());
      if (rc) break;
    }
    const int nb = (int)std::min<int64_t>(B, n - b * B);
    uint64_t t = 0;
    const auto t0 = Clock::now();
    rc = bl_submit(ctx, r.p, BL_PIX_U8, nb, w, h, (size_t)w, fpx, BL_LANDMARKS_BEST, &t);
    if (rc == BL_OK) q.push_back({t, b, t0});
  }
  while (!q.empty()) {  // drain (after an error: collect and discard, keeping the first error)
    if (rc == BL_OK) {
      rc = collect_one(q.front());
    } else {
      const std::string keep = bl_last_error();
      int64_t got = 0;
      bl_collect(ctx, q.front().ticket, dets + total, det_cap - total, counts.data(), &got, xy.data());
      blb::set_last_error(keep.c_str());
    }
    q.erase(q.begin());
  }
  rc = finish(rc);
  if (rc) return rc;
  *det_total = total;
  // build_trace (blink.cpp:47-93): per-eye baseline quantile over frames with a face
  if (fps <= 0.0) return fail(BL_ERR_INVALID, "build_trace: fps must be positive");
  std::vector<double> lefts, rights;
  for (int64_t i = 0; i < n; ++i)
    if (frames[i].face_found) {
      lefts.push_back(frames[i].ear_left);
      rights.push_back(frames[i].ear_right);
    }
  if (lefts.empty())
    return fail(BL_ERR_INVALID, "build_trace: no frames with a detected face, cannot establish an EAR baseline");
  const double bl_l = quantile(lefts, 0.95), bl_r = quantile(rights, 0.95);
  for (int64_t i = 0; i < n; ++i)
    if (frames[i].face_found) {
      frames[i].closure_left = closure_of(frames[i].ear_left, bl_l);
      frames[i].closure_right = closure_of(frames[i].ear_right, bl_r);
    }
  if (baselines) {
    baselines[0] = bl_l;
    baselines[1] = bl_r;
  }
  return BL_OK;
}

}  // extern "C"
