// Host-side adapters of the hot path's data formats, behind the
// C-ABI: PGM frames (image.hpp:23-28, image.cpp:67-127) and the "hog-v1" / "ert-v1" model
// files (detector.hpp:99-100, detector.cpp:291-351; ert.hpp:128-129, ert.cpp:358-469).
//
// Frames are parsed straight into u8 (the reference widens them to double, image.cpp:98-110;
// every PGM sample is an integer <= 255, so u8 is exact) ready for a pinned upload; models
// are parsed into the flat arrays bl_detector_upload / bl_ert_upload take.  Error behaviour
// follows the reference: unreadable files -> BL_ERR_IO (io_error), PGM syntax errors ->
// BL_ERR_IO with the reference's message and byte offset, malformed or wrong-version models
// -> BL_ERR_MODEL (model_error).  JSON goes through nlohmann/json, the library the
// reference uses, so files round-trip between the two implementations bit-for-bit.
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/blinkline_b200.h"
#include "json.hpp"

namespace blb {
void set_last_error(const char* msg);
}

namespace {

int fail(int code, const std::string& msg) {
  blb::set_last_error(msg.c_str());
  return code;
}

// --------------------------------------------------------------------------- PGM ----
struct PgmError {
  std::string msg;
};

// Reads the fully buffered file; on malformed input throws PgmError("<what> at byte <pos>").
struct PgmReader {
  const std::string& data;
  size_t pos = 0;

  [[noreturn]] void bad(const std::string& what) const { throw PgmError{what + " at byte " + std::to_string(pos)}; }
  bool at_end() const { return pos >= data.size(); }
  void skip_ws_comments() {
    while (!at_end()) {
      const unsigned char ch = (unsigned char)data[pos];
      if (ch == '#') {
        while (!at_end() && data[pos] != '\n') ++pos;
      } else if (std::isspace(ch)) {
        ++pos;
      } else {
        return;
      }
    }
  }
  long number(const char* what) {
    skip_ws_comments();
    if (at_end()) bad(std::string("truncated header, missing ") + what);
    if (!std::isdigit((unsigned char)data[pos])) bad(std::string("malformed header, expected ") + what);
    long v = 0;
    for (; !at_end() && std::isdigit((unsigned char)data[pos]); ++pos) {
      v = v * 10 + (data[pos] - '0');
      if (v > 1000000000L) bad(std::string("malformed header, ") + what + " out of range");
    }
    return v;
  }
};

int read_file(const char* path, std::string& out) {
  std::ifstream in(path, std::ios::binary);
  if (!in) return fail(BL_ERR_IO, std::string(path) + ": cannot open file");
  std::ostringstream buf;
  buf << in.rdbuf();
  out = buf.str();
  return BL_OK;
}

// ------------------------------------------------------------------------ models ----
using json = nlohmann::json;

int parse_json(const char* path, const char* version, json& j) {
  std::ifstream in(path);
  if (!in) return fail(BL_ERR_IO, std::string(path) + ": cannot open file");
  try {
    in >> j;
  } catch (const json::exception& e) {
    return fail(BL_ERR_MODEL, std::string(path) + ": invalid JSON (" + e.what() + ")");
  }
  if (!j.contains("version") || !j["version"].is_string() || j["version"] != version)
    return fail(BL_ERR_MODEL, std::string(path) + ": unsupported model version, expected \"" + version + "\"");
  return BL_OK;
}

int write_json(const char* path, const json& j) {
  std::ofstream out(path);
  if (!out) return fail(BL_ERR_IO, std::string(path) + ": cannot open file for writing");
  out << j.dump();
  if (!out) return fail(BL_ERR_IO, std::string(path) + ": write failed");
  return BL_OK;
}

}  // namespace

// A parsed ert-v1 file in the upload layout of bl_ert_upload.
struct bl_ert_file {
  int L = 0, T = 0, K = 0, F = 0;
  double shrinkage = 0.1;
  std::vector<double> mean_xy, split_params, leaves;
  std::vector<int32_t> anchors;
};

// Fast path for a well-formed binary PGM: the header parsed from the first 4 KB, the pixel
// bytes read straight into the caller's buffer (no whole-file copy; header-only calls read
// 4 KB).  Anything unusual -- P2, a header past 4 KB, truncation, a sample above maxval --
// returns handled = false and the full parser below decides, with the reference's messages.
int read_pgm_fast(const char* path, int* w, int* h, uint8_t* pixels, size_t cap, bool& handled) {
  handled = false;
  FILE* f = std::fopen(path, "rb");
  if (!f) return BL_OK;
  char head[4096];
  const size_t got = std::fread(head, 1, sizeof head, f);
  const std::string hs(head, got);
  PgmReader rd{hs};
  long pw = 0, ph = 0, maxval = 0;
  try {
    if (got < 2 || hs[0] != 'P' || hs[1] != '5') throw PgmError{};
    rd.pos = 2;
    pw = rd.number("width");
    ph = rd.number("height");
    maxval = rd.number("maxval");
    if (pw < 1 || ph < 1 || maxval < 1 || maxval > 255) throw PgmError{};
    if (rd.at_end() || !std::isspace((unsigned char)hs[rd.pos])) throw PgmError{};
  } catch (const PgmError&) {
    std::fclose(f);
    return BL_OK;
  }
  const size_t n = (size_t)pw * (size_t)ph;
  if (pixels && cap < n) {
    std::fclose(f);
    return BL_OK;  // the full parser reports the capacity error
  }
  if (pixels) {
    if (std::fseek(f, (long)(rd.pos + 1), SEEK_SET) != 0 || std::fread(pixels, 1, n, f) != n) {
      std::fclose(f);
      return BL_OK;
    }
    if (maxval < 255)
      for (size_t i = 0; i < n; ++i)
        if (pixels[i] > maxval) {
          std::fclose(f);
          return BL_OK;
        }
  }
  std::fclose(f);
  *w = (int)pw;
  *h = (int)ph;
  handled = true;
  return BL_OK;
}

extern "C" {

int bl_read_pgm(const char* path, int* w, int* h, uint8_t* pixels, size_t cap) {
  if (!path || !w || !h) return fail(BL_ERR_INVALID, "null argument");
  bool handled = false;
  if (int rc = read_pgm_fast(path, w, h, pixels, cap, handled)) return rc;
  if (handled) return BL_OK;
  std::string data;
  if (int rc = read_file(path, data)) return rc;
  PgmReader rd{data};
  try {
    if (data.size() < 2 || data[0] != 'P' || (data[1] != '5' && data[1] != '2'))
      rd.bad("malformed header, expected P5 or P2 magic");
    const bool binary = data[1] == '5';
    rd.pos = 2;
    const long pw = rd.number("width");
    const long ph = rd.number("height");
    if (pw < 1 || ph < 1) rd.bad("malformed header, dimensions must be >= 1");
    const long maxval = rd.number("maxval");
    if (maxval < 1) rd.bad("malformed header, maxval must be >= 1");
    if (maxval > 255) rd.bad("unsupported maxval " + std::to_string(maxval) + " (limit 255)");
    const size_t n = (size_t)pw * (size_t)ph;
    *w = (int)pw;
    *h = (int)ph;
    if (!pixels) {  // dimensions only (header parsed)
      if (binary) {
        if (rd.at_end() || !std::isspace((unsigned char)data[rd.pos]))
          rd.bad("malformed header, expected single whitespace after maxval");
      }
      return BL_OK;
    }
    if (cap < n) return fail(BL_ERR_CAPACITY, "pixel buffer holds " + std::to_string(cap) + " < " + std::to_string(n));
    if (binary) {
      if (rd.at_end() || !std::isspace((unsigned char)data[rd.pos]))
        rd.bad("malformed header, expected single whitespace after maxval");
      ++rd.pos;
      if (data.size() - rd.pos < n) {
        rd.pos = data.size();
        rd.bad("truncated pixel data, expected " + std::to_string(n) + " bytes");
      }
      for (size_t i = 0; i < n; ++i, ++rd.pos) {
        const unsigned char b = (unsigned char)data[rd.pos];
        if (b > maxval) rd.bad("pixel value exceeds maxval");
        pixels[i] = b;
      }
    } else {
      for (size_t i = 0; i < n; ++i) {
        rd.skip_ws_comments();
        if (rd.at_end()) rd.bad("truncated pixel data, expected " + std::to_string(n) + " samples");
        const long v = rd.number("pixel value");
        if (v > maxval) rd.bad("pixel value exceeds maxval");
        pixels[i] = (uint8_t)v;
      }
    }
  } catch (const PgmError& e) {
    return fail(BL_ERR_IO, std::string(path) + ": " + e.msg);
  }
  return BL_OK;
}

int bl_write_pgm(const char* path, const double* pixels, int w, int h) {
  if (!path || !pixels) return fail(BL_ERR_INVALID, "null argument");
  if (w < 1 || h < 1) return fail(BL_ERR_INVALID, "make_image: dimensions must be >= 1");
  std::ofstream out(path, std::ios::binary);
  if (!out) return fail(BL_ERR_IO, std::string(path) + ": cannot open file for writing");
  out << "P5\n" << w << " " << h << "\n255\n";
  std::string bytes((size_t)w * h, '\0');
  for (size_t i = 0; i < bytes.size(); ++i) {  // clamp to [0, 255], round half away from zero
    const double v = pixels[i] < 0.0 ? 0.0 : (pixels[i] > 255.0 ? 255.0 : pixels[i]);
    bytes[i] = (char)(unsigned char)std::llround(v);
  }
  out.write(bytes.data(), (std::streamsize)bytes.size());
  if (!out) return fail(BL_ERR_IO, std::string(path) + ": write failed");
  return BL_OK;
}

int bl_read_detector_json(const char* path, double* weights, double* biases, double* threshold, int* window_cells,
                          int* cell_px, int* scale_num, int* scale_den, double* min_face_ratio) {
  if (!path || !window_cells) return fail(BL_ERR_INVALID, "null argument");
  json j;
  if (int rc = parse_json(path, "hog-v1", j)) return rc;
  try {
    const int wc = j.at("window_cells").get<int>();
    *window_cells = wc;
    if (cell_px) *cell_px = j.at("cell_px").get<int>();
    if (scale_num) *scale_num = j.at("scale_factor_num").get<int>();
    if (scale_den) *scale_den = j.at("scale_factor_den").get<int>();
    if (min_face_ratio) *min_face_ratio = j.at("min_face_ratio").get<double>();
    if (threshold) *threshold = j.at("threshold").get<double>();
    const json& filters = j.at("filters");
    if (!filters.is_array() || filters.size() != 5) return fail(BL_ERR_MODEL, std::string(path) + ": expected exactly 5 filters");
    const size_t expected = (size_t)wc * wc * 31;
    for (size_t i = 0; i < 5; ++i) {
      const json& wj = filters[i].at("weights");
      if (!wj.is_array() || wj.size() != expected)
        return fail(BL_ERR_MODEL, std::string(path) + ": filter " + std::to_string(i) + " carries " +
                                      std::to_string(wj.is_array() ? wj.size() : 0) + " weights, expected " +
                                      std::to_string(expected));
      if (weights)
        for (size_t k = 0; k < expected; ++k) weights[i * expected + k] = wj[k].get<double>();
      if (biases) biases[i] = filters[i].at("bias").get<double>();
    }
  } catch (const json::exception& e) {
    return fail(BL_ERR_MODEL, std::string(path) + ": malformed model file (" + e.what() + ")");
  }
  return BL_OK;
}

int bl_write_detector_json(const char* path, const double* weights, const double* biases, double threshold,
                           int window_cells, int cell_px, int scale_num, int scale_den, double min_face_ratio) {
  if (!path || !weights || !biases) return fail(BL_ERR_INVALID, "null argument");
  if (window_cells < 1) return fail(BL_ERR_MODEL, "window_cells must be >= 1");
  const size_t per = (size_t)window_cells * window_cells * 31;
  json j;
  j["version"] = "hog-v1";
  j["window_cells"] = window_cells;
  j["cell_px"] = cell_px;
  j["scale_factor_num"] = scale_num;
  j["scale_factor_den"] = scale_den;
  j["min_face_ratio"] = min_face_ratio;
  j["threshold"] = threshold;
  json filters = json::array();
  for (int r = 0; r < 5; ++r)
    filters.push_back({{"weights", std::vector<double>(weights + r * per, weights + (r + 1) * per)}, {"bias", biases[r]}});
  j["filters"] = std::move(filters);
  return write_json(path, j);
}

int bl_ert_file_open(const char* path, bl_ert_file** out, int* L, int* T, int* K, int* F, double* shrinkage) {
  if (!path || !out) return fail(BL_ERR_INVALID, "null argument");
  *out = nullptr;
  json j;
  if (int rc = parse_json(path, "ert-v1", j)) return rc;
  auto m = std::make_unique<bl_ert_file>();
  const std::string p(path);
  try {
    m->L = j.at("L").get<int>();
    m->T = j.at("T").get<int>();
    m->K = j.at("K").get<int>();
    m->F = j.at("F").get<int>();
    m->shrinkage = j.at("shrinkage").get<double>();
    if (m->L < 0 || m->T < 0 || m->K < 0 || m->F < 0 || m->F > 16) return fail(BL_ERR_MODEL, p + ": cascade dims out of range");
    const json& mean = j.at("mean_shape");
    if ((int)mean.size() != m->L) return fail(BL_ERR_MODEL, p + ": mean_shape must carry L points");
    for (const json& pt : mean) {
      m->mean_xy.push_back(pt.at(0).get<double>());
      m->mean_xy.push_back(pt.at(1).get<double>());
    }
    const json& cascade = j.at("cascade");
    if ((int)cascade.size() != m->T) return fail(BL_ERR_MODEL, p + ": cascade must carry T levels");
    const size_t S = ((size_t)1 << m->F) - 1, NL = (size_t)1 << m->F;
    const size_t trees = (size_t)m->T * m->K;
    m->anchors.reserve(trees * S * 2);
    m->split_params.reserve(trees * S * 5);
    m->leaves.reserve(trees * NL * m->L * 2);
    for (const json& level : cascade) {
      if ((int)level.size() != m->K) return fail(BL_ERR_MODEL, p + ": every cascade level must carry K trees");
      for (const json& tj : level) {
        const json& splits = tj.at("splits");
        const json& leaves = tj.at("leaves");
        if (splits.size() != S || leaves.size() != NL)
          return fail(BL_ERR_MODEL, p + ": tree split/leaf counts do not match depth F");
        for (const json& sj : splits) {
          const int a = sj.at("a").get<int>(), b = sj.at("b").get<int>();
          if (a < 0 || a >= m->L || b < 0 || b >= m->L) return fail(BL_ERR_MODEL, p + ": split anchor out of range");
          m->anchors.push_back(a);
          m->anchors.push_back(b);
          for (const char* key : {"ox_a", "oy_a", "ox_b", "oy_b", "thr"}) m->split_params.push_back(sj.at(key).get<double>());
        }
        for (const json& lj : leaves) {
          if ((int)lj.size() != m->L) return fail(BL_ERR_MODEL, p + ": leaf delta must carry L points");
          for (const json& pt : lj) {
            m->leaves.push_back(pt.at(0).get<double>());
            m->leaves.push_back(pt.at(1).get<double>());
          }
        }
      }
    }
  } catch (const json::exception& e) {
    return fail(BL_ERR_MODEL, p + ": malformed model file (" + e.what() + ")");
  }
  if (L) *L = m->L;
  if (T) *T = m->T;
  if (K) *K = m->K;
  if (F) *F = m->F;
  if (shrinkage) *shrinkage = m->shrinkage;
  *out = m.release();
  return BL_OK;
}

int bl_ert_file_copy(const bl_ert_file* m, double* mean_xy, int32_t* anchors, double* split_params, double* leaves) {
  if (!m) return fail(BL_ERR_INVALID, "null model file");
  if (mean_xy) std::memcpy(mean_xy, m->mean_xy.data(), sizeof(double) * m->mean_xy.size());
  if (anchors) std::memcpy(anchors, m->anchors.data(), sizeof(int32_t) * m->anchors.size());
  if (split_params) std::memcpy(split_params, m->split_params.data(), sizeof(double) * m->split_params.size());
  if (leaves) std::memcpy(leaves, m->leaves.data(), sizeof(double) * m->leaves.size());
  return BL_OK;
}

int bl_ert_file_upload(const bl_ert_file* m, bl_ctx* ctx) {
  if (!m || !ctx) return fail(BL_ERR_INVALID, "null argument");
  return bl_ert_upload(ctx, m->L, m->T, m->K, m->F, m->shrinkage, m->mean_xy.data(), m->anchors.data(),
                       m->split_params.data(), m->leaves.data());
}

void bl_ert_file_close(bl_ert_file* m) { delete m; }

int bl_write_ert_json(const char* path, int L, int T, int K, int F, double shrinkage, const double* mean_xy,
                      const int32_t* anchors, const double* split_params, const double* leaves) {
  if (!path || !mean_xy || ((size_t)T * K > 0 && (!leaves || (F > 0 && (!anchors || !split_params)))))
    return fail(BL_ERR_INVALID, "null argument");
  if (L < 0 || T < 0 || K < 0 || F < 0 || F > 16) return fail(BL_ERR_MODEL, "cascade dims out of range");
  const size_t S = ((size_t)1 << F) - 1, NL = (size_t)1 << F;
  json j;
  j["version"] = "ert-v1";
  j["L"] = L;
  j["T"] = T;
  j["K"] = K;
  j["F"] = (T > 0 && K > 0) ? F : 0;  // the reference records depth 0 for an empty cascade
  j["shrinkage"] = shrinkage;
  json mean = json::array();
  for (int i = 0; i < L; ++i) mean.push_back({mean_xy[2 * i], mean_xy[2 * i + 1]});
  j["mean_shape"] = std::move(mean);
  json cascade = json::array();
  for (int t = 0; t < T; ++t) {
    json level = json::array();
    for (int k = 0; k < K; ++k) {
      const size_t tree = (size_t)t * K + k;
      json splits = json::array();
      for (size_t s = 0; s < S; ++s) {
        const size_t i = tree * S + s;
        splits.push_back({{"a", anchors[2 * i]},
                          {"b", anchors[2 * i + 1]},
                          {"ox_a", split_params[5 * i]},
                          {"oy_a", split_params[5 * i + 1]},
                          {"ox_b", split_params[5 * i + 2]},
                          {"oy_b", split_params[5 * i + 3]},
                          {"thr", split_params[5 * i + 4]}});
      }
      json lv = json::array();
      for (size_t q = 0; q < NL; ++q) {
        json pts = json::array();
        const double* d = leaves + ((tree * NL + q) * L) * 2;
        for (int i = 0; i < L; ++i) pts.push_back({d[2 * i], d[2 * i + 1]});
        lv.push_back(std::move(pts));
      }
      level.push_back({{"splits", std::move(splits)}, {"leaves", std::move(lv)}});
    }
    cascade.push_back(std::move(level));
  }
  j["cascade"] = std::move(cascade);
  return write_json(path, j);
}

}  // extern "C"
