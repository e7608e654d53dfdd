// rvk_gpu -- the reference CLI's `estimate` command (tools/rvk_main.cpp:104-158)
// on the B200 path, SURVEY.md 8(f) rows 1 and 4.
//
//   rvk_gpu estimate FRAMES.csv -o ESTIMATES.csv [--mode parallel|sequential|gpu|lsq-only]
//           [--seed S] [--eps E] [--min-pts M] [--max-trials T]
//           [--threshold-scale K] [--workers W (accepted, ignored)]
//
// Frame CSV v1 in (header "frame_id,x,y,z,doppler,azimuth", frames grouped by
// frame_id in first-appearance order, the reference's row checks and
// line-numbered messages: src/frame_io.cpp:86-139), estimate CSV out
// (shortest round-trip doubles, heading in degrees or "nan":
// src/frame_io.cpp:158-180). Per frame: rvk_estimate_frame (dbscan ->
// extract_clusters -> gather -> run_ransac -> estimate_all on the device), or
// for --mode lsq-only the all-true masks (src/ransac.cpp:244-256) through
// rvk_estimate_all. A failing frame is reported on stderr and skipped
// (tools/rvk_main.cpp:146-148). Exit codes: 0 ok, 2 usage / input, 3 runtime.
//
// Host side: the frame file is parsed by all hardware threads (the body is
// split at line boundaries, each thread runs from_chars over its chunk; the
// first malformed line in file order is reported, exactly as the sequential
// reader would), then grouped into frames in first-appearance order; frames
// then run on three host threads, each with its own device context and
// stream, so consecutive frames overlap on the device; rows are written in
// frame order.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <limits>
#include <numbers>
#include <sstream>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

#include "rvk_gpu.h"

namespace {

constexpr int kExitUsage = 2;
constexpr int kExitRuntime = 3;
constexpr const char* kFrameHeader = "frame_id,x,y,z,doppler,azimuth";
constexpr const char* kEstimateHeader = "frame_id,cluster_id,v_x,v_y,heading_deg,inlier_count";

struct FrameSoA {
  int64_t frame_id = 0;
  std::vector<double> x, y, z, doppler, azimuth;
};

struct InputError {
  std::string what;
};

bool parse_double(std::string_view t, double& v) {
  const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}
bool parse_int(std::string_view t, int64_t& v) {
  const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}

// Rows of one chunk of the body, in file order.
struct Rows {
  std::vector<int64_t> fid;
  std::vector<double> v;        // 5 per row: x, y, z, doppler, azimuth
  std::size_t lines = 0;        // lines consumed (the chunk's own)
  std::size_t bad_line = 0;     // 1-based within the chunk, 0 = none
  std::string bad_what;
};

// One chunk [b, e) of the body (whole lines): the row checks of read_frames
// (src/frame_io.cpp:100-132), stopping at the chunk's first malformed row.
void parse_chunk(std::string_view text, std::size_t b, std::size_t e, Rows& out) {
  std::size_t pos = b;
  while (pos < e) {
    std::size_t nl = text.find('\n', pos);
    if (nl == std::string_view::npos || nl > e) nl = e;
    const std::string_view line = text.substr(pos, nl - pos);
    pos = nl + 1;
    ++out.lines;
    auto bad = [&](const std::string& what) {
      out.bad_line = out.lines;
      out.bad_what = what;
    };
    std::string_view f[7];
    int nf = 0;
    std::size_t s = 0;
    for (;;) {
      const std::size_t c = line.find(',', s);
      if (nf < 7) f[nf] = line.substr(s, c == std::string_view::npos ? std::string_view::npos : c - s);
      ++nf;
      if (c == std::string_view::npos) break;
      s = c + 1;
    }
    if (nf != 6) return bad("expected 6 fields");
    int64_t fid = 0;
    if (!parse_int(f[0], fid)) return bad("bad frame_id '" + std::string(f[0]) + "'");
    double v[5];
    static const char* names[5] = {"x", "y", "z", "doppler", "azimuth"};
    for (int k = 0; k < 5; ++k)
      if (!parse_double(f[k + 1], v[k]) || !std::isfinite(v[k]))
        return bad(std::string("bad ") + names[k] + " '" + std::string(f[k + 1]) + "'");
    if (!(v[4] > -std::numbers::pi && v[4] <= std::numbers::pi))
      return bad("azimuth outside (-pi, pi]");
    out.fid.push_back(fid);
    out.v.insert(out.v.end(), v, v + 5);
  }
}

// read_frames (src/frame_io.cpp:86-139), parsed by `threads` threads.
std::vector<FrameSoA> read_frames(const std::string& path, unsigned threads) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw InputError{"cannot open for reading: " + path};
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string text_s = ss.str();
  const std::string_view text(text_s);
  if (text.empty()) throw InputError{"empty frame file: " + path};
  std::size_t hdr_end = text.find('\n');
  if (hdr_end == std::string_view::npos) hdr_end = text.size();
  const std::string_view header = text.substr(0, hdr_end);
  if (header != kFrameHeader)
    throw InputError{"expected header '" + std::string(kFrameHeader) + "', got '" +
                     std::string(header) + "'"};
  // body [b0, end): chunks of whole lines (the reader's lines end at '\n'; a
  // final line without one is a line too)
  const std::size_t b0 = std::min(hdr_end + 1, text.size());
  std::size_t end = text.size();
  const std::size_t body = end - b0;
  threads = std::max(1u, std::min<unsigned>(threads, static_cast<unsigned>(body / (1 << 16) + 1)));
  std::vector<std::size_t> cut{b0};
  for (unsigned t = 1; t < threads; ++t) {
    std::size_t c = b0 + body * t / threads;
    c = text.find('\n', std::max(c, cut.back()));
    c = c == std::string_view::npos ? end : c + 1;
    cut.push_back(std::max(c, cut.back()));
  }
  cut.push_back(end);
  std::vector<Rows> rows(threads);
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < threads; ++t)
    pool.emplace_back(parse_chunk, text, cut[t], cut[t + 1], std::ref(rows[t]));
  parse_chunk(text, cut[0], cut[1], rows[0]);
  for (auto& th : pool) th.join();
  // the first malformed row in file order
  std::size_t line_base = 1;  // the header
  for (const Rows& r : rows) {
    if (r.bad_line)
      throw InputError{"malformed row at line " + std::to_string(line_base + r.bad_line) + ": " +
                       r.bad_what};
    line_base += r.lines;
  }
  // group by frame_id, frames in first-appearance order, rows in file order
  std::vector<FrameSoA> frames;
  std::unordered_map<int64_t, std::size_t> slot;
  for (const Rows& r : rows)
    for (std::size_t k = 0; k < r.fid.size(); ++k) {
      auto [it, inserted] = slot.try_emplace(r.fid[k], frames.size());
      if (inserted) {
        frames.emplace_back();
        frames.back().frame_id = r.fid[k];
      }
      FrameSoA& fr = frames[it->second];
      const double* v = &r.v[5 * k];
      fr.x.push_back(v[0]);
      fr.y.push_back(v[1]);
      fr.z.push_back(v[2]);
      fr.doppler.push_back(v[3]);
      fr.azimuth.push_back(v[4]);
    }
  return frames;
}

void append_double(std::string& out, double v) {
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v);
  out.append(buf, r.ptr);
}
void append_int(std::string& out, int64_t v) {
  char buf[32];
  const auto r = std::to_chars(buf, buf + sizeof buf, v);
  out.append(buf, r.ptr);
}

// write_estimates (src/frame_io.cpp:158-180)
void append_estimate(std::string& out, const rvk_estimate& e) {
  append_int(out, e.frame_id);
  out.push_back(',');
  append_int(out, e.cluster_id);
  out.push_back(',');
  append_double(out, e.v_x);
  out.push_back(',');
  append_double(out, e.v_y);
  out.push_back(',');
  append_double(out, e.has_heading ? e.heading * (180.0 / std::numbers::pi)
                                    : std::numeric_limits<double>::quiet_NaN());
  out.push_back(',');
  append_int(out, e.inlier_count);
  out.push_back('\n');
}

int usage(const char* msg) {
  std::cerr << "error: " << msg << "\n"
            << "usage: rvk_gpu estimate FRAMES.csv -o ESTIMATES.csv [--mode parallel|sequential|gpu|lsq-only] "
               "[--seed S] [--eps E] [--min-pts M] [--max-trials T] [--threshold-scale K] "
               "[--workers W]\n";
  return kExitUsage;
}

// One frame; returns false (message in `err`) on a per-frame error.
bool estimate_one(const FrameSoA& f, const std::string& mode, const rvk_clustering_params& cp,
                  const rvk_ransac_params& rp, std::vector<rvk_estimate>& out, std::string& err) {
  const int64_t n = static_cast<int64_t>(f.x.size());
  std::vector<int32_t> labels(static_cast<std::size_t>(n)), pi(static_cast<std::size_t>(n) + 1);
  std::vector<int64_t> off(static_cast<std::size_t>(n) + 2);
  int32_t m = 0;
  if (mode == "gpu") {
    const std::size_t cap = static_cast<std::size_t>(n) / 3 + 1;  // kMinClusterSize
    std::vector<int32_t> cnt(cap), tr(cap);
    std::vector<uint8_t> mask(static_cast<std::size_t>(n) + 1);
    std::vector<rvk_estimate> est(cap);
    const int st = rvk_estimate_frame(f.frame_id, n, f.x.data(), f.y.data(), f.z.data(),
                                      f.doppler.data(), f.azimuth.data(), &cp, 3, &rp,
                                      labels.data(), &m, off.data(), pi.data(), cnt.data(),
                                      tr.data(), mask.data(), est.data());
    if (st != RVK_OK) {
      err = rvk_last_error();
      return false;
    }
    out.insert(out.end(), est.begin(), est.begin() + m);
    return true;
  }
  // lsq-only: dbscan + extract, all-true masks, estimate_all
  int st = rvk_dbscan(n, f.x.data(), f.y.data(), f.z.data(), &cp, labels.data());
  if (st == RVK_OK) st = rvk_extract_clusters(n, labels.data(), 3, &m, off.data(), pi.data());
  if (st != RVK_OK) {
    err = rvk_last_error();
    return false;
  }
  if (m == 0) return true;
  const std::size_t P = static_cast<std::size_t>(off[m]);
  std::vector<double> az(P), dop(P);
  for (std::size_t k = 0; k < P; ++k) {
    az[k] = f.azimuth[static_cast<std::size_t>(pi[k])];
    dop[k] = f.doppler[static_cast<std::size_t>(pi[k])];
  }
  std::vector<uint8_t> ones(P, 1);
  std::vector<int32_t> ids(static_cast<std::size_t>(m));
  for (int32_t c = 0; c < m; ++c) ids[static_cast<std::size_t>(c)] = c;
  std::vector<rvk_estimate> est(static_cast<std::size_t>(m));
  st = rvk_estimate_all(f.frame_id, m, off.data(), az.data(), dop.data(), ids.data(), ones.data(),
                        0, est.data());
  if (st != RVK_OK) {
    err = rvk_last_error();
    return false;
  }
  out.insert(out.end(), est.begin(), est.end());
  return true;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::strcmp(argv[1], "estimate") != 0) return usage("expected the estimate command");
  std::string frames_path, out_path, mode = "gpu";
  rvk_clustering_params cp{2.0, 3, RVK_FEATURES_XY};     // clustering.hpp:13-17
  rvk_ransac_params rp{256, 0, 1.0, 0};                  // ransac.hpp:19-23
  int64_t workers = 0;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&](const char* name) -> std::string {
      if (i + 1 >= argc) throw InputError{std::string("missing value for ") + name};
      return argv[++i];
    };
    try {
      if (a == "-o" || a == "--output") out_path = val("--output");
      else if (a == "--mode") mode = val("--mode");
      else if (a == "--seed") rp.rng_seed = std::stoull(val("--seed"));
      else if (a == "--eps") cp.eps = std::stod(val("--eps"));
      else if (a == "--min-pts") cp.min_pts = std::stoi(val("--min-pts"));
      else if (a == "--max-trials") rp.max_trials = std::stoi(val("--max-trials"));
      else if (a == "--threshold-scale") rp.threshold_scale = std::stod(val("--threshold-scale"));
      else if (a == "--workers") workers = std::stoll(val("--workers"));
      else if (!a.empty() && a[0] == '-') return usage(("unknown option " + a).c_str());
      else if (frames_path.empty()) frames_path = a;
      else return usage("more than one frames file");
    } catch (const InputError& e) {
      return usage(e.what.c_str());
    } catch (const std::exception&) {
      return usage(("bad value for " + a).c_str());
    }
  }
  if (frames_path.empty() || out_path.empty()) return usage("frames file and -o are required");
  // tools/rvk_main.cpp:106-114
  // the reference's modes (tools/rvk_main.cpp: parallel is its default,
  // sequential its 1-core baseline) are accepted as aliases of the device
  // path: their results are defined to be identical (ransac.hpp:124-125)
  if (mode == "parallel" || mode == "sequential") mode = "gpu";
  if (mode != "gpu" && mode != "lsq-only") {
    std::cerr << "error: mode must be parallel, sequential, gpu or lsq-only\n";
    return kExitUsage;
  }
  if (!(cp.eps > 0.0) || cp.min_pts < 1 || rp.max_trials < 1 || !(rp.threshold_scale > 0.0) ||
      workers < 0) {
    std::cerr << "error: invalid estimation parameters\n";
    return kExitUsage;
  }
  std::vector<FrameSoA> frames;
  try {
    frames = read_frames(frames_path, std::max(1u, std::thread::hardware_concurrency()));
  } catch (const InputError& e) {
    std::cerr << "error: " << e.what << '\n';
    return kExitUsage;
  }
  // Frames are dealt round-robin to kFrameWorkers host threads; each thread
  // has its own device context and stream (rvk_gpu.h: one per thread and
  // device), so frame k+1's copies and clustering overlap frame k's RANSAC on
  // the device. Results, errors and output rows stay in frame order.
  constexpr std::size_t kFrameWorkers = 3;
  const std::size_t nf = frames.size();
  std::vector<std::vector<rvk_estimate>> results(nf);
  std::vector<std::string> errors(nf);
  std::vector<char> ok(nf, 0);
  std::vector<std::thread> workers_t;
  const std::size_t nw = std::min(kFrameWorkers, std::max<std::size_t>(nf, 1));
  for (std::size_t w = 0; w < nw; ++w)
    workers_t.emplace_back([&, w] {
      for (std::size_t k = w; k < nf; k += nw)
        ok[k] = estimate_one(frames[k], mode, cp, rp, results[k], errors[k]) ? 1 : 0;
    });
  for (auto& t : workers_t) t.join();
  std::string text(kEstimateHeader);
  text.push_back('\n');
  for (std::size_t k = 0; k < nf; ++k) {
    if (!ok[k]) std::cerr << "frame " << frames[k].frame_id << ": " << errors[k] << '\n';
    for (const rvk_estimate& e : results[k]) append_estimate(text, e);
  }
  std::ofstream out(out_path, std::ios::binary | std::ios::trunc);
  if (!out) {
    std::cerr << "error: cannot open for writing: " << out_path << '\n';
    return kExitRuntime;
  }
  out.write(text.data(), static_cast<std::streamsize>(text.size()));
  if (!out) {
    std::cerr << "error: write failed: " << out_path << '\n';
    return kExitRuntime;
  }
  return 0;
}
