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
  std::vector<uint8_t> buf[2] = {std::vector<uint8_t>(fpx * B), std::vector<uint8_t>(fpx * B)};
  std::vector<double> dec_ms(n, 0.0);

  // decode batch b into buf[b & 1] (the next batch decodes on a helper thread while the
  // device works on the current one)
  auto decode = [&](int64_t b0, int nb, std::vector<uint8_t>& dst) -> int {
    for (int i = 0; i < nb; ++i) {
      const auto t0 = Clock::now();
      int fw = 0, fh = 0;
      if (int rc = bl_read_pgm(paths[b0 + i].c_str(), &fw, &fh, dst.data() + fpx * i, fpx)) return rc;
      dec_ms[b0 + i] = ms_since(t0);
    }
    return BL_OK;
  };
  int rc = decode(0, B, buf[0]);
  if (rc) return rc;
  int64_t total = 0;
  std::vector<int32_t> counts(B), face_frame;
  std::vector<bl_box> boxes;
  std::vector<double> xy;
  for (int64_t b0 = 0, bi = 0; b0 < n; b0 += B, ++bi) {
    const int nb = (int)std::min<int64_t>(B, n - b0);
    std::vector<uint8_t>& cur = buf[bi & 1];
    const int64_t nb_next = std::min<int64_t>(B, n - (b0 + nb));
    int rc_next = BL_OK;
    std::thread next;
    if (nb_next > 0) next = std::thread([&] { rc_next = decode(b0 + nb, (int)nb_next, buf[(bi + 1) & 1]); });
    // detect (detect_frame, pipeline.cpp:159-169) for the batch, straight into the output
    const auto td = Clock::now();
    int64_t got = 0;
    rc = bl_detect(ctx, cur.data(), BL_PIX_U8, nb, w, h, (size_t)w, fpx, dets + total, det_cap - total, counts.data(),
                   &got);
    const double det_ms = ms_since(td);
    // the face of each frame = its first detection; landmarks for the faces (pipeline.cpp:171-190)
    face_frame.clear();
    boxes.clear();
    int64_t off = total;
    for (int i = 0; rc == BL_OK && i < nb; ++i) {
      bl_frame_result& fr = frames[b0 + i];
      std::memset(&fr, 0, sizeof fr);
      fr.frame_index = (int32_t)(b0 + i);
      fr.n_detections = counts[i];
      fr.t = double(b0 + i) / fps;
      fr.decode_ms = dec_ms[b0 + i];
      fr.detect_ms = det_ms / nb;
      if (counts[i] > 0) {
        fr.face_found = 1;
        fr.face = dets[off];
        face_frame.push_back(i);
        boxes.push_back(dets[off].box);
      }
      off += counts[i];
    }
    const auto tl = Clock::now();
    if (rc == BL_OK && !boxes.empty()) {
      xy.resize(boxes.size() * 2 * L);
      rc = bl_landmarks(ctx, cur.data(), BL_PIX_U8, nb, w, h, (size_t)w, fpx, face_frame.data(), boxes.data(),
                        (int64_t)boxes.size(), xy.data(), nullptr);
    }
    const double lm_ms = ms_since(tl);
    for (size_t k = 0; rc == BL_OK && k < boxes.size(); ++k) {
      bl_frame_result& fr = frames[b0 + face_frame[k]];
      const double* p = xy.data() + k * 2 * L;
      std::memcpy(landmarks + (b0 + face_frame[k]) * 2 * (int64_t)L, p, sizeof(double) * 2 * L);
      rc = eye_ear(p, kLeft, fr.ear_left);
      if (rc == BL_OK) rc = eye_ear(p, kRight, fr.ear_right);
    }
    for (int i = 0; i < nb; ++i) frames[b0 + i].landmark_ms = lm_ms / nb;
    if (next.joinable()) next.join();
    if (rc) return rc;
    if (rc_next) return rc_next;
    total = off;
  }
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
