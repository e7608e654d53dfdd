// Host side of the C-ABI (include/rvk_gpu.h): validation with the
// reference's order and messages, per-thread device context (stream +
// grow-only workspace + pinned staging), host<->device marshalling, and the
// kernel pipeline prep -> score -> select(+refit).
//
// There is no CPU fallback anywhere: if CUDA is unavailable every entry
// point returns RVK_ECUDA with the CUDA error string.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/rvk_gpu.h"
#include "rvk_kernels.cuh"

namespace rvk_gpu {

namespace {

thread_local std::string g_error;
thread_local int32_t g_error_cluster = -1;
thread_local int64_t g_launches = 0;

constexpr int kMinClusterSize = 3;  // include/rvk/types.hpp:20

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_error = buf;
  return status;
}

struct CudaError {
  cudaError_t e;
  const char* what;
};

#define RVK_CUDA(call)                                     \
  do {                                                     \
    const cudaError_t rvk_e_ = (call);                     \
    if (rvk_e_ != cudaSuccess) throw CudaError{rvk_e_, #call}; \
  } while (0)

// Grow-only device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <class T>
  T* get(size_t count) {
    const size_t bytes = std::max<size_t>(count * sizeof(T), 256);
    if (bytes > cap) {
      // headroom: frames of a stream vary in size, and every regrow is a
      // device-synchronizing cudaFree/cudaMalloc
      const size_t want = std::max(bytes + bytes / 4, cap * 2);
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      RVK_CUDA(cudaMalloc(&p, want));
      // zeroed once per (re)allocation: the alignment padding between the
      // arrays of a block is then defined when the block is copied whole.
      // The memset runs on the legacy stream, which does not order against
      // our non-blocking streams: wait for it before any kernel can write.
      RVK_CUDA(cudaMemset(p, 0, want));
      RVK_CUDA(cudaStreamSynchronize(nullptr));
      cap = want;
    }
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Grow-only pinned host buffer (staging for H2D/D2H).
struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      cap = 0;
      const size_t want = std::max<size_t>(bytes + bytes / 4, 1 << 20);
      RVK_CUDA(cudaHostAlloc(&p, want, cudaHostAllocDefault));
      std::memset(p, 0, want);  // padding between staged arrays is copied too
      cap = want;
    }
    return p;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

// Device scratch of one stream's in-flight pipeline.
struct Workspace {
  DevBuf xy64, xy32, thr, norm, upper, hyp, tiles, tile_count, aux;
  DevBuf big;
  void release() {
    for (DevBuf* b : {&xy64, &xy32, &thr, &norm, &upper, &hyp, &tiles, &tile_count, &aux, &big})
      b->release();
  }
};

struct Context {
  int device = -1;
  cudaStream_t stream = nullptr;
  DevBuf db, frame, labels;  // clustering scratch, frame points, labels
  HostBuf stage_frame;
  DevBuf in;       // offsets | az | dop | ids | keys | order (one H2D)
  DevBuf out;      // count | trial | est | mask (one D2H)
  HostBuf stage_in, stage_out;
  // Scratch per stream, so calls on different streams (device API) may be
  // in flight concurrently; the host API uses `stream`.
  std::unordered_map<cudaStream_t, Workspace> ws;
  Workspace& workspace(cudaStream_t s) { return ws[s]; }
  // chunked host pipeline: one copy stream streams every chunk's H2D back
  // to back; two compute streams take the chunks alternately as they land
  cudaStream_t copy = nullptr;
  cudaStream_t pipe[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> landed;  // per chunk: its H2D is done
  cudaEvent_t joined = nullptr;     // the second compute stream's work is done
  Context() = default;
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  // Runs at thread exit; errors are ignored (the runtime may already be
  // shutting down when the main thread's contexts go).
  ~Context() {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return;
    if (cur != device) cudaSetDevice(device);
    for (DevBuf* b : {&db, &frame, &labels, &in, &out}) b->release();
    for (HostBuf* b : {&stage_frame, &stage_in, &stage_out}) b->release();
    for (auto& kv : ws) kv.second.release();
    for (cudaEvent_t e : landed) cudaEventDestroy(e);
    if (joined) cudaEventDestroy(joined);
    for (cudaStream_t st : {stream, copy, pipe[0], pipe[1]})
      if (st) cudaStreamDestroy(st);
    if (cur != device) cudaSetDevice(cur);
  }
  void ensure_pipe(int chunks) {
    if (!copy) {
      RVK_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
      RVK_CUDA(cudaStreamCreateWithFlags(&pipe[0], cudaStreamNonBlocking));
      RVK_CUDA(cudaStreamCreateWithFlags(&pipe[1], cudaStreamNonBlocking));
      RVK_CUDA(cudaEventCreateWithFlags(&joined, cudaEventDisableTiming));
    }
    while (static_cast<int>(landed.size()) < chunks + 1) {
      cudaEvent_t e;
      RVK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      landed.push_back(e);
    }
  }
};

// One context per (thread, device), created on the thread's first call on
// that device and freed when the thread exits (thread_local map of owning
// pointers): a thread that alternates devices keeps one context per device
// instead of leaking a fresh one at every switch.
Context& context() {
  thread_local std::unordered_map<int, std::unique_ptr<Context>> ctxs;
  int dev = 0;
  RVK_CUDA(cudaGetDevice(&dev));
  std::unique_ptr<Context>& slot = ctxs[dev];
  if (!slot) {
    auto c = std::make_unique<Context>();
    c->device = dev;
    RVK_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    slot = std::move(c);
  }
  return *slot;
}

// Restores the calling thread's current device on scope exit (entry points
// that switch to an object's device must not leave it switched).
struct DeviceGuard {
  int saved = -1;
  explicit DeviceGuard(int dev) {
    RVK_CUDA(cudaGetDevice(&saved));
    if (saved != dev) RVK_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != saved) cudaSetDevice(saved);
  }
};

size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }
size_t packed_bytes(int64_t P) { return static_cast<size_t>((P + 7) / 8); }

// Validation in the reference's order (src/ransac.cpp:140-154).
int validate_params(const rvk_ransac_params* p, const char* who) {
  if (p == nullptr) return fail(RVK_EINVAL, "%s: params must not be null", who);
  if (p->max_trials < 1) return fail(RVK_EINVAL, "%s: max_trials must be at least 1", who);
  if (!(p->threshold_scale > 0.0))
    return fail(RVK_EINVAL, "%s: threshold_scale must be positive", who);
  return RVK_OK;
}

int validate_offsets(int32_t n_clusters, const int64_t* offsets, int min_size, const char* who) {
  if (n_clusters < 0) return fail(RVK_EINVAL, "%s: negative cluster count", who);
  if (n_clusters > 0 && offsets == nullptr) return fail(RVK_EINVAL, "%s: offsets is null", who);
  if (n_clusters > 0 && offsets[0] != 0) return fail(RVK_EINVAL, "%s: offsets[0] must be 0", who);
  for (int32_t c = 0; c < n_clusters; ++c) {
    const int64_t n = offsets[c + 1] - offsets[c];
    if (n < 0) return fail(RVK_EINVAL, "%s: offsets must be non-decreasing", who);
    if (n > (int64_t{1} << 30)) return fail(RVK_EINVAL, "%s: cluster %d too large", who, c);
    if (n < min_size) {
      g_error_cluster = c;
      return fail(RVK_ECLUSTER_TOO_SMALL, "%s: cluster %d has %lld points, need %d", who, c,
                  static_cast<long long>(n), min_size);
    }
  }
  return RVK_OK;
}

// Largest cluster of a host CSR (lets the pipeline skip the CTA path's
// launches when the fused kernel takes every cluster).
int64_t max_cluster_size(int32_t n_clusters, const int64_t* offsets) {
  int64_t m = 0;
  for (int32_t c = 0; c < n_clusters; ++c) m = std::max(m, offsets[c + 1] - offsets[c]);
  return m;
}

// Largest clusters first, so the scoring grid's tail is short (LPT).
void lpt_order(int32_t n_clusters, const int64_t* offsets, int32_t* order) {
  std::iota(order, order + n_clusters, 0);
  std::stable_sort(order, order + n_clusters, [&](int32_t a, int32_t b) {
    return offsets[a + 1] - offsets[a] > offsets[b + 1] - offsets[b];
  });
}

// Persistent host workers for rvk_ransac_estimate_multi: part 0 runs on the
// caller, part i > 0 on worker i, which keeps its thread_local per-device
// contexts (streams, pinned and device buffers) across calls. One multi call
// at a time per process; the pool is never torn down (workers park on a
// condition variable at exit).
class MultiPool {
 public:
  void run(int n, const std::function<void(int)>& f) {
    std::lock_guard<std::mutex> call(call_m_);
    while (static_cast<int>(w_.size()) < n - 1) w_.emplace_back(new Worker(static_cast<int>(w_.size()) + 1));
    for (int i = 0; i < n - 1; ++i) w_[i]->post(&f);
    f(0);
    for (int i = 0; i < n - 1; ++i) w_[i]->wait();
  }

 private:
  struct Worker {
    explicit Worker(int idx) : idx(idx), t([this] { loop(); }) { t.detach(); }
    void post(const std::function<void(int)>* f) {
      std::lock_guard<std::mutex> g(m);
      job = f;
      cv.notify_all();
    }
    void wait() {
      std::unique_lock<std::mutex> g(m);
      cv.wait(g, [this] { return job == nullptr; });
    }
    void loop() {
      for (;;) {
        const std::function<void(int)>* f;
        {
          std::unique_lock<std::mutex> g(m);
          cv.wait(g, [this] { return job != nullptr; });
          f = job;
        }
        (*f)(idx);
        std::lock_guard<std::mutex> g(m);
        job = nullptr;
        cv.notify_all();
      }
    }
    const int idx;
    std::mutex m;
    std::condition_variable cv;
    const std::function<void(int)>* job = nullptr;
    std::thread t;
  };
  std::mutex call_m_;
  std::vector<Worker*> w_;
};

MultiPool& multi_pool() {
  static MultiPool* p = new MultiPool;  // intentionally leaked, see above
  return *p;
}

template <class F>
int guarded(F&& f) {
  g_error.clear();
  g_error_cluster = -1;
  try {
    return f();
  } catch (const CudaError& e) {
    return fail(RVK_ECUDA, "CUDA error %s (%s) in %s", cudaGetErrorName(e.e),
                cudaGetErrorString(e.e), e.what);
  } catch (const std::bad_alloc&) {
    return fail(RVK_ENOMEM, "host allocation failed");
  }
}

// Stages the host frame into one pinned buffer, copies it with one H2D and
// returns the device view (offsets, az, dop, ids, keys, order).
struct Staged {
  FrameDev f;
  int64_t* d_offsets;
};

FrameDev stage_frame(Context& ctx, int64_t frame_id, int32_t n_clusters, const int64_t* offsets,
                     const double* az, const double* dop, const int32_t* ids,
                     const int32_t* keys, bool want_order, const uint8_t* mask_in,
                     uint8_t** d_mask_in) {
  const int64_t P = offsets[n_clusters];
  const size_t o_off = 0;
  const size_t o_az = align_up(o_off + sizeof(int64_t) * (n_clusters + 1));
  const size_t o_dop = align_up(o_az + sizeof(double) * P);
  const size_t o_ids = align_up(o_dop + sizeof(double) * P);
  const size_t o_keys = align_up(o_ids + sizeof(int32_t) * n_clusters);
  const size_t o_ord = align_up(o_keys + sizeof(int32_t) * n_clusters);
  const size_t o_mask = align_up(o_ord + sizeof(int32_t) * n_clusters);
  const size_t total = align_up(o_mask + (mask_in ? P : 0));
  char* h = static_cast<char*>(ctx.stage_in.get(total));
  char* d = ctx.in.get<char>(total);
  std::memcpy(h + o_off, offsets, sizeof(int64_t) * (n_clusters + 1));
  std::memcpy(h + o_az, az, sizeof(double) * P);
  std::memcpy(h + o_dop, dop, sizeof(double) * P);
  if (ids) std::memcpy(h + o_ids, ids, sizeof(int32_t) * n_clusters);
  if (keys) std::memcpy(h + o_keys, keys, sizeof(int32_t) * n_clusters);
  if (want_order) lpt_order(n_clusters, offsets, reinterpret_cast<int32_t*>(h + o_ord));
  if (mask_in) std::memcpy(h + o_mask, mask_in, P);
  RVK_CUDA(cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, ctx.stream));
  FrameDev f;
  f.n_clusters = n_clusters;
  f.n_points = P;
  f.offsets = reinterpret_cast<const int64_t*>(d + o_off);
  f.azimuth = reinterpret_cast<const double*>(d + o_az);
  f.doppler = reinterpret_cast<const double*>(d + o_dop);
  f.cluster_ids = ids ? reinterpret_cast<const int32_t*>(d + o_ids) : nullptr;
  f.keys = keys ? reinterpret_cast<const int32_t*>(d + o_keys) : nullptr;
  f.order = want_order ? reinterpret_cast<const int32_t*>(d + o_ord) : nullptr;
  f.frame_id = frame_id;
  if (d_mask_in) *d_mask_in = reinterpret_cast<uint8_t*>(d + o_mask);
  return f;
}

Scratch scratch(Workspace& w, int32_t n_clusters, int64_t P, int32_t T) {
  Scratch s;
  ScoreGeom g = score_geom(std::max(T, 1));
  const size_t C = static_cast<size_t>(n_clusters);
  s.xy64 = w.xy64.get<double2>(P);
  s.xy32 = w.xy32.get<float2>(P + 2 * C + 10);
  s.stat = w.thr.get<double4>(C);
  s.norm = w.norm.get<double>(4 * C);
  s.upper = w.upper.get<int32_t>(C * g.Tg * 8);
  s.hyp = w.hyp.get<float>(C * g.Tg * 32);
  s.ppt = score_ppt(g, P, n_clusters);
  set_ppt(g, s.ppt);
  s.tile_cap = tile_capacity(g, P, n_clusters);
  s.tiles = w.tiles.get<int4>(static_cast<size_t>(kTileBuckets) * s.tile_cap);
  s.tile_count = w.tile_count.get<int32_t>(kTileBuckets + 1);
  s.big_ctl = w.big.get<int32_t>(C + 8);
  s.big_list = s.big_ctl + 8;
  return s;
}

void check_launch() { RVK_CUDA(cudaGetLastError()); }

// Output block: count[C] | trial[C] | est[C] | mask[P] | mask bits[ceil(P/8)],
// one D2H.
struct OutLayout {
  size_t o_cnt, o_tr, o_est, o_mask, o_bits, total;
  OutLayout(int32_t C, int64_t P) {
    o_cnt = 0;
    o_tr = align_up(sizeof(int32_t) * C);
    o_est = align_up(o_tr + sizeof(int32_t) * C);
    o_mask = align_up(o_est + sizeof(rvk_estimate) * C);
    o_bits = align_up(o_mask + P);
    total = align_up(o_bits + packed_bytes(P));
  }
};

// ---- optional stage timing (rvk_profile_enable / rvk_profile_read) ----
struct StageRec {
  int stage;
  cudaEvent_t a, b;
};
struct Profile {
  bool on = false;
  std::vector<StageRec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t ev() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    RVK_CUDA(cudaEventCreate(&e));
    return e;
  }
};
thread_local Profile g_prof;

template <class F>
void stage(int id, cudaStream_t st, F&& launch) {
  if (!g_prof.on) {
    launch();
    return;
  }
  StageRec r{id, g_prof.ev(), g_prof.ev()};
  RVK_CUDA(cudaEventRecord(r.a, st));
  launch();
  RVK_CUDA(cudaEventRecord(r.b, st));
  g_prof.recs.push_back(r);
}

// prep+hyps -> score -> select(+refit): the whole device pipeline of one call.
// Stage ids (rvk_profile_read): 0 = prep + hypothesis setup + tile plan,
// 1 = a fused warp-per-cluster kernel (the whole path for single small
// frames, or prep + score for batches of small clusters), 2 = score,
// 3 = select + refit. On the fused paths stages 0/2 take only the clusters
// the fused kernel listed (none when the host knows they all fit).
void run_pipeline(const FrameDev& f, const rvk_ransac_params& p, const Scratch& s,
                  const Outputs& o, cudaStream_t st) {
  if (fused_path(f, p)) stage(1, st, [&] { launch_fused(f, p, s, o, st); });
  if (prep_score_path(f, p)) stage(1, st, [&] { launch_prep_score(f, p, s, st); });
  stage(0, st, [&] { launch_prep_hyps(f, p, s, st); });
  stage(2, st, [&] { launch_score(f, p, s, st); });
  stage(3, st, [&] { launch_select(f, p, s, o, st); });
  check_launch();
}

bool is_pinned(const void* p) {
  if (p == nullptr) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // clear: pageable pointers may report an error on old drivers
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Host API: the frame is split into up to kPipeMax cluster-aligned chunks of
// >= kPipeChunk points. A copy stream issues every chunk's H2D back to back
// (PCIe runs at full rate for the whole call); chunk i's kernels (prep+hyps
// -> score -> select) and its D2H run on compute stream i % 2 once its bytes
// have landed, so copies and kernels of different chunks overlap. Pinned caller buffers are copied directly (no host
// staging memcpy); pageable ones go through the context's pinned staging.
// RNG keys stay frame-positional, so the result does not depend on the
// chunking.
constexpr int64_t kPipeChunk = 1 << 18;
constexpr int kPipeMax = 4;

// Tunables (environment, read once): RVK_PIPE_CHUNK = minimum points per
// chunk, RVK_PIPE_MAX = maximum number of chunks.
int64_t env_or(const char* name, int64_t dflt) {
  const char* v = std::getenv(name);
  if (v == nullptr || *v == 0) return dflt;
  const long long x = std::atoll(v);
  return x > 0 ? x : dflt;
}
int64_t pipe_chunk() {
  static const int64_t v = env_or("RVK_PIPE_CHUNK", kPipeChunk);
  return v;
}
bool trace_on() {
  static const bool v = env_or("RVK_TRACE", 0) != 0;
  return v;
}
int pipe_max() {
  static const int v = static_cast<int>(env_or("RVK_PIPE_MAX", kPipeMax));
  return v;
}

int ransac_estimate_host(int64_t frame_id, int32_t n_clusters, const int64_t* offsets,
                         const double* az, const double* dop, const int32_t* ids,
                         const rvk_ransac_params* params, const int32_t* keys,
                         int32_t* inlier_count, int32_t* winning_trial, uint8_t* mask,
                         rvk_estimate* out, bool refit, bool packed = false) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  int st = validate_params(params, "run_ransac");
  if (st != RVK_OK) return st;
  st = validate_offsets(n_clusters, offsets, kMinClusterSize, "run_ransac");
  if (st != RVK_OK) return st;
  if (n_clusters == 0) return RVK_OK;
  if ((az == nullptr || dop == nullptr) && offsets[n_clusters] > 0)
    return fail(RVK_EINVAL, "run_ransac: null point arrays");
  Context& ctx = context();
  const int64_t P = offsets[n_clusters];

  // chunk boundaries (cluster-aligned)
  int K = static_cast<int>(std::min<int64_t>(pipe_max(), std::max<int64_t>(1, P / pipe_chunk())));
  std::vector<int32_t> cut(1, 0);
  for (int i = 1; i < K; ++i) {
    const int64_t target = P * i / K;
    int32_t c = cut.back();
    while (c < n_clusters && offsets[c] < target) ++c;
    if (c > cut.back() && c < n_clusters) cut.push_back(c);
  }
  cut.push_back(n_clusters);
  K = static_cast<int>(cut.size()) - 1;
  ctx.ensure_pipe(K);

  const bool pin_in = is_pinned(az) && is_pinned(dop);
  const bool pin_mask = is_pinned(mask);
  const size_t mask_bytes = packed ? packed_bytes(P) : static_cast<size_t>(P);
  const int64_t max_n = max_cluster_size(n_clusters, offsets);
  const auto t1 = clk::now();

  // device input block: [offsets (rebased per chunk) | keys | ids] + az | dop
  const size_t o_keys = align_up(sizeof(int64_t) * (n_clusters + K));
  const size_t o_ids = align_up(o_keys + sizeof(int32_t) * n_clusters);
  const size_t o_az = align_up(o_ids + sizeof(int32_t) * n_clusters);
  const size_t o_dop = align_up(o_az + sizeof(double) * P);
  const size_t in_total = align_up(o_dop + sizeof(double) * P);
  const size_t small = o_az;
  char* h = static_cast<char*>(ctx.stage_in.get(pin_in ? small : in_total));
  char* d = ctx.in.get<char>(in_total);
  int64_t* h_off = reinterpret_cast<int64_t*>(h);
  int32_t* h_keys = reinterpret_cast<int32_t*>(h + o_keys);
  int32_t* h_ids = reinterpret_cast<int32_t*>(h + o_ids);
  for (int i = 0; i < K; ++i)  // chunk i's offsets start at slot cut[i] + i
    for (int32_t c = cut[i]; c <= cut[i + 1]; ++c) h_off[c + i] = offsets[c] - offsets[cut[i]];
  // RNG keys and cluster ids default to the frame-positional index: chunk
  // kernels see chunk-local indices, so both are always passed explicitly.
  for (int32_t c = 0; c < n_clusters; ++c) h_keys[c] = keys ? keys[c] : c;
  for (int32_t c = 0; c < n_clusters; ++c) h_ids[c] = ids ? ids[c] : c;
  if (!pin_in) {
    std::memcpy(h + o_az, az, sizeof(double) * P);
    std::memcpy(h + o_dop, dop, sizeof(double) * P);
  }
  const double* src_az = pin_in ? az : reinterpret_cast<const double*>(h + o_az);
  const double* src_dop = pin_in ? dop : reinterpret_cast<const double*>(h + o_dop);

  const OutLayout L(n_clusters, P);
  char* dout = ctx.out.get<char>(L.total);
  char* hout = static_cast<char*>(ctx.stage_out.get(L.total));
  // all H2D on the copy stream, in chunk order, back to back (RVK_COPY_STREAM=0:
  // each chunk's H2D on its compute stream instead)
  const bool copy_stream = env_or("RVK_COPY_STREAM", 1) != 0;
  cudaStream_t cs = copy_stream ? ctx.copy : ctx.pipe[0];
  RVK_CUDA(cudaMemcpyAsync(d, h, small, cudaMemcpyHostToDevice, cs));  // small arrays
  RVK_CUDA(cudaEventRecord(ctx.landed[K], cs));
  for (int i = 0; copy_stream && i < K; ++i) {
    const int64_t p0 = offsets[cut[i]], np = offsets[cut[i + 1]] - p0;
    RVK_CUDA(cudaMemcpyAsync(d + o_az + sizeof(double) * p0, src_az + p0, sizeof(double) * np,
                             cudaMemcpyHostToDevice, ctx.copy));
    RVK_CUDA(cudaMemcpyAsync(d + o_dop + sizeof(double) * p0, src_dop + p0, sizeof(double) * np,
                             cudaMemcpyHostToDevice, ctx.copy));
    RVK_CUDA(cudaEventRecord(ctx.landed[i], ctx.copy));
  }
  for (int i = 0; i < K; ++i) {
    cudaStream_t sc = ctx.pipe[i & 1];
    if (copy_stream) {
      RVK_CUDA(cudaStreamWaitEvent(sc, ctx.landed[i], 0));
    } else {
      if (sc != cs) RVK_CUDA(cudaStreamWaitEvent(sc, ctx.landed[K], 0));
      const int64_t q0 = offsets[cut[i]], nq = offsets[cut[i + 1]] - q0;
      RVK_CUDA(cudaMemcpyAsync(d + o_az + sizeof(double) * q0, src_az + q0, sizeof(double) * nq,
                               cudaMemcpyHostToDevice, sc));
      RVK_CUDA(cudaMemcpyAsync(d + o_dop + sizeof(double) * q0, src_dop + q0,
                               sizeof(double) * nq, cudaMemcpyHostToDevice, sc));
    }
    const int32_t c0 = cut[i], nc = cut[i + 1] - cut[i];
    const int64_t p0 = offsets[c0], np = offsets[cut[i + 1]] - p0;
    char* daz = d + o_az + sizeof(double) * p0;
    char* ddop = d + o_dop + sizeof(double) * p0;
    FrameDev f;
    f.n_clusters = nc;
    f.n_points = np;
    f.offsets = reinterpret_cast<const int64_t*>(d) + c0 + i;
    f.azimuth = reinterpret_cast<const double*>(daz);
    f.doppler = reinterpret_cast<const double*>(ddop);
    f.keys = reinterpret_cast<const int32_t*>(d + o_keys) + c0;
    f.cluster_ids = reinterpret_cast<const int32_t*>(d + o_ids) + c0;
    f.frame_id = frame_id;
    f.max_cluster = max_n;
    Scratch s = scratch(ctx.workspace(sc), nc, np, params->max_trials);
    Outputs o;
    o.inlier_count = reinterpret_cast<int32_t*>(dout + L.o_cnt) + c0;
    o.winning_trial = reinterpret_cast<int32_t*>(dout + L.o_tr) + c0;
    o.est = refit ? reinterpret_cast<rvk_estimate*>(dout + L.o_est) + c0 : nullptr;
    o.mask = reinterpret_cast<uint8_t*>(dout + L.o_mask) + p0;
    run_pipeline(f, *params, s, o, sc);
    // per-chunk results back (a packed mask once every chunk is done, below:
    // chunk boundaries are not byte-aligned in the bit array)
    if (mask && !packed) {
      uint8_t* dst = pin_mask ? mask + p0 : reinterpret_cast<uint8_t*>(hout + L.o_mask) + p0;
      RVK_CUDA(cudaMemcpyAsync(dst, o.mask, np, cudaMemcpyDeviceToHost, sc));
    }
    if (inlier_count)
      RVK_CUDA(cudaMemcpyAsync(reinterpret_cast<int32_t*>(hout + L.o_cnt) + c0, o.inlier_count,
                               sizeof(int32_t) * nc, cudaMemcpyDeviceToHost, sc));
    if (winning_trial)
      RVK_CUDA(cudaMemcpyAsync(reinterpret_cast<int32_t*>(hout + L.o_tr) + c0, o.winning_trial,
                               sizeof(int32_t) * nc, cudaMemcpyDeviceToHost, sc));
    if (out && refit)
      RVK_CUDA(cudaMemcpyAsync(reinterpret_cast<rvk_estimate*>(hout + L.o_est) + c0, o.est,
                               sizeof(rvk_estimate) * nc, cudaMemcpyDeviceToHost, sc));
  }
  if (mask && packed) {  // 1 bit per point: join the chunks, pack, one D2H
    RVK_CUDA(cudaEventRecord(ctx.joined, ctx.pipe[1]));
    RVK_CUDA(cudaStreamWaitEvent(ctx.pipe[0], ctx.joined, 0));
    uint8_t* dbits = reinterpret_cast<uint8_t*>(dout + L.o_bits);
    launch_pack_mask(reinterpret_cast<const uint8_t*>(dout + L.o_mask), P, dbits, ctx.pipe[0]);
    check_launch();
    uint8_t* dst = pin_mask ? mask : reinterpret_cast<uint8_t*>(hout + L.o_bits);
    RVK_CUDA(cudaMemcpyAsync(dst, dbits, mask_bytes, cudaMemcpyDeviceToHost, ctx.pipe[0]));
  }
  const auto t2 = clk::now();
  RVK_CUDA(cudaStreamSynchronize(ctx.pipe[0]));
  RVK_CUDA(cudaStreamSynchronize(ctx.pipe[1]));
  const auto t3 = clk::now();
  if (inlier_count) std::memcpy(inlier_count, hout + L.o_cnt, sizeof(int32_t) * n_clusters);
  if (winning_trial) std::memcpy(winning_trial, hout + L.o_tr, sizeof(int32_t) * n_clusters);
  if (mask && !pin_mask)
    std::memcpy(mask, hout + (packed ? L.o_bits : L.o_mask), mask_bytes);
  if (out && refit) std::memcpy(out, hout + L.o_est, sizeof(rvk_estimate) * n_clusters);
  if (trace_on()) {
    const auto t4 = clk::now();
    auto us = [](clk::time_point a, clk::time_point b) {
      return std::chrono::duration<double, std::micro>(b - a).count();
    };
    std::fprintf(stderr,
                 "[rvk trace] P=%lld C=%d chunks=%d pinned_in=%d pinned_mask=%d validate=%.1fus "
                 "enqueue=%.1fus wait=%.1fus copy_out=%.1fus total=%.1fus\n",
                 static_cast<long long>(P), n_clusters, K, pin_in, pin_mask, us(t0, t1),
                 us(t1, t2), us(t2, t3), us(t3, t4), us(t0, t4));
  }
  return RVK_OK;
}

// ---- clustering + the whole frame path ----
int validate_clustering(const rvk_clustering_params* p) {
  if (p == nullptr) return fail(RVK_EINVAL, "dbscan: params must not be null");
  if (!(p->eps > 0.0)) return fail(RVK_EINVAL, "dbscan: eps must be positive");
  if (p->min_pts < 1) return fail(RVK_EINVAL, "dbscan: min_pts must be at least 1");
  if (p->features != RVK_FEATURES_XY && p->features != RVK_FEATURES_XYZ)
    return fail(RVK_EINVAL, "dbscan: unknown feature space");
  return RVK_OK;
}

// Frame points (x | y | [z] | [doppler | azimuth]) to the device, one H2D.
struct FramePts {
  double *x, *y, *z, *dop, *az;
};
FramePts upload_points(Context& ctx, int64_t n, const double* x, const double* y, const double* z,
                       const double* dop, const double* az) {
  const size_t bytes = sizeof(double) * static_cast<size_t>(n);
  const int cols = 2 + (z ? 1 : 0) + (dop ? 1 : 0) + (az ? 1 : 0);
  char* h = static_cast<char*>(ctx.stage_frame.get(bytes * cols));
  double* d = ctx.frame.get<double>(static_cast<size_t>(n) * cols);
  FramePts f{};
  int col = 0;
  auto put = [&](const double* src, double** dst) {
    if (src == nullptr) return;
    std::memcpy(h + bytes * col, src, bytes);
    *dst = d + static_cast<size_t>(n) * col;
    ++col;
  };
  put(x, &f.x);
  put(y, &f.y);
  put(z, &f.z);
  put(dop, &f.dop);
  put(az, &f.az);
  RVK_CUDA(cudaMemcpyAsync(d, h, bytes * cols, cudaMemcpyHostToDevice, ctx.stream));
  return f;
}

// ---- pipelined frame stream (rvk_stream_*) ----
//
// Slot k % depth holds frame k: its own device input/output blocks, scratch
// and pinned staging. Frame k's H2D runs on the copy stream; its kernels and
// D2H on compute stream k % 2 once its bytes have landed. A slot is reused
// only after its previous frame completed (host wait on its `done` event),
// so no device buffer is ever overwritten while in use.
struct StreamSlot {
  DevBuf in, out;
  HostBuf small_in, big_in, stage_out;
  Workspace ws;
  cudaEvent_t landed = nullptr, done = nullptr;
  int64_t ticket = -1;  // frame in the slot (-1: none pending)
  int32_t C = 0;
  int64_t P = 0;
  OutLayout L{0, 0};
  int32_t* cnt = nullptr;
  int32_t* tr = nullptr;
  uint8_t* mask = nullptr;
  rvk_estimate* est = nullptr;
  bool pin_mask = false;
  bool packed = false;  // mask delivered as bits (ceil(P/8) bytes)
};

struct FrameStream {
  int device = 0;
  rvk_ransac_params params{};
  int depth = 3;
  cudaStream_t copy = nullptr;
  cudaStream_t compute[2] = {nullptr, nullptr};
  std::vector<StreamSlot> slots;
  int64_t next = 0;

  // Delivers slot s's outputs to the caller's arrays (waits for its D2H).
  void complete(StreamSlot& s) {
    if (s.ticket < 0) return;
    RVK_CUDA(cudaEventSynchronize(s.done));
    const char* h = static_cast<const char*>(s.stage_out.p);
    if (s.cnt) std::memcpy(s.cnt, h + s.L.o_cnt, sizeof(int32_t) * s.C);
    if (s.tr) std::memcpy(s.tr, h + s.L.o_tr, sizeof(int32_t) * s.C);
    if (s.est) std::memcpy(s.est, h + s.L.o_est, sizeof(rvk_estimate) * s.C);
    if (s.mask && !s.pin_mask) {
      if (s.packed) std::memcpy(s.mask, h + s.L.o_bits, packed_bytes(s.P));
      else std::memcpy(s.mask, h + s.L.o_mask, s.P);
    }
    s.ticket = -1;
  }

  int submit(int64_t frame_id, int32_t n_clusters, const int64_t* offsets, const double* az,
             const double* dop, const int32_t* ids, const int32_t* keys, int32_t* cnt,
             int32_t* tr, uint8_t* mask, rvk_estimate* est, int64_t* ticket,
             bool packed = false) {
    int st = validate_offsets(n_clusters, offsets, kMinClusterSize, "run_ransac");
    if (st != RVK_OK) return st;
    const int64_t P = n_clusters ? offsets[n_clusters] : 0;
    if ((az == nullptr || dop == nullptr) && P > 0)
      return fail(RVK_EINVAL, "run_ransac: null point arrays");
    DeviceGuard guard(device);
    const int64_t k = next;
    StreamSlot& s = slots[k % depth];
    const auto tw = std::chrono::steady_clock::now();
    complete(s);  // frees the slot (the frame submitted `depth` calls ago)
    if (trace_on())
      std::fprintf(stderr, "[rvk stream] ticket %lld waited %.1fus for slot %lld\n",
                   static_cast<long long>(k),
                   std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tw)
                       .count(),
                   static_cast<long long>(k % depth));
    if (ticket) *ticket = k;
    ++next;
    if (n_clusters == 0) return RVK_OK;
    cudaStream_t sc = compute[k & 1];

    // small arrays: offsets | keys | ids, always through pinned staging
    const size_t o_keys = align_up(sizeof(int64_t) * (n_clusters + 1));
    const size_t o_ids = align_up(o_keys + sizeof(int32_t) * n_clusters);
    const size_t small = align_up(o_ids + sizeof(int32_t) * n_clusters);
    const size_t o_az = small;
    const size_t o_dop = align_up(o_az + sizeof(double) * P);
    const size_t in_total = align_up(o_dop + sizeof(double) * P);
    char* h = static_cast<char*>(s.small_in.get(small));
    char* d = s.in.get<char>(in_total);
    std::memcpy(h, offsets, sizeof(int64_t) * (n_clusters + 1));
    int32_t* h_keys = reinterpret_cast<int32_t*>(h + o_keys);
    int32_t* h_ids = reinterpret_cast<int32_t*>(h + o_ids);
    for (int32_t c = 0; c < n_clusters; ++c) h_keys[c] = keys ? keys[c] : c;
    for (int32_t c = 0; c < n_clusters; ++c) h_ids[c] = ids ? ids[c] : c;
    const bool pin_in = is_pinned(az) && is_pinned(dop);
    RVK_CUDA(cudaMemcpyAsync(d, h, small, cudaMemcpyHostToDevice, copy));
    if (pin_in) {
      RVK_CUDA(cudaMemcpyAsync(d + o_az, az, sizeof(double) * P, cudaMemcpyHostToDevice, copy));
      RVK_CUDA(cudaMemcpyAsync(d + o_dop, dop, sizeof(double) * P, cudaMemcpyHostToDevice, copy));
    } else {
      char* hb = static_cast<char*>(s.big_in.get(in_total - o_az));
      std::memcpy(hb, az, sizeof(double) * P);
      std::memcpy(hb + (o_dop - o_az), dop, sizeof(double) * P);
      RVK_CUDA(cudaMemcpyAsync(d + o_az, hb, in_total - o_az, cudaMemcpyHostToDevice, copy));
    }
    RVK_CUDA(cudaEventRecord(s.landed, copy));
    RVK_CUDA(cudaStreamWaitEvent(sc, s.landed, 0));

    FrameDev f;
    f.n_clusters = n_clusters;
    f.n_points = P;
    f.offsets = reinterpret_cast<const int64_t*>(d);
    f.azimuth = reinterpret_cast<const double*>(d + o_az);
    f.doppler = reinterpret_cast<const double*>(d + o_dop);
    f.keys = reinterpret_cast<const int32_t*>(d + o_keys);
    f.cluster_ids = reinterpret_cast<const int32_t*>(d + o_ids);
    f.frame_id = frame_id;
    f.max_cluster = max_cluster_size(n_clusters, offsets);
    s.L = OutLayout(n_clusters, P);
    char* dout = s.out.get<char>(s.L.total);
    char* hout = static_cast<char*>(s.stage_out.get(s.L.total));
    Scratch scr = scratch(s.ws, n_clusters, P, params.max_trials);
    Outputs o;
    o.inlier_count = reinterpret_cast<int32_t*>(dout + s.L.o_cnt);
    o.winning_trial = reinterpret_cast<int32_t*>(dout + s.L.o_tr);
    o.est = reinterpret_cast<rvk_estimate*>(dout + s.L.o_est);
    o.mask = reinterpret_cast<uint8_t*>(dout + s.L.o_mask);
    run_pipeline(f, params, scr, o, sc);
    s.pin_mask = is_pinned(mask);
    // counts | trials | estimates in one D2H, the mask straight to the caller
    // when it is pinned
    if (cnt || tr || est)
      RVK_CUDA(cudaMemcpyAsync(hout, dout, s.L.o_mask, cudaMemcpyDeviceToHost, sc));
    s.packed = packed;
    if (mask && packed) {
      uint8_t* dbits = reinterpret_cast<uint8_t*>(dout + s.L.o_bits);
      launch_pack_mask(o.mask, P, dbits, sc);
      check_launch();
      RVK_CUDA(cudaMemcpyAsync(s.pin_mask ? static_cast<void*>(mask) : hout + s.L.o_bits,
                               dbits, packed_bytes(P), cudaMemcpyDeviceToHost, sc));
    } else if (mask) {
      RVK_CUDA(cudaMemcpyAsync(s.pin_mask ? static_cast<void*>(mask) : hout + s.L.o_mask,
                               o.mask, P, cudaMemcpyDeviceToHost, sc));
    }
    RVK_CUDA(cudaEventRecord(s.done, sc));
    s.ticket = k;
    s.C = n_clusters;
    s.P = P;
    s.cnt = cnt;
    s.tr = tr;
    s.mask = mask;
    s.est = est;
    return RVK_OK;
  }

  int wait(int64_t ticket) {
    if (ticket < 0 || ticket >= next) return fail(RVK_EINVAL, "rvk_stream_wait: unknown ticket");
    DeviceGuard guard(device);
    StreamSlot& s = slots[ticket % depth];
    if (s.ticket == ticket) complete(s);
    return RVK_OK;  // older tickets were completed when their slot was reused
  }
};

}  // namespace

void count_launch() { ++g_launches; }

}  // namespace rvk_gpu

using namespace rvk_gpu;

struct rvk_frame_stream {
  FrameStream impl;
};

extern "C" {

int32_t rvk_abi_version(void) { return RVK_GPU_ABI_VERSION; }
const char* rvk_last_error(void) { return g_error.c_str(); }
int32_t rvk_last_error_cluster(void) { return g_error_cluster; }
int64_t rvk_kernel_launches(void) { return g_launches; }
void rvk_reset_kernel_launches(void) { g_launches = 0; }

int rvk_run_ransac(int32_t n_clusters, const int64_t* offsets, const double* azimuth,
                   const double* doppler, const rvk_ransac_params* params,
                   const int32_t* rng_cluster_index, int32_t /*workers*/, int32_t* inlier_count,
                   int32_t* winning_trial, uint8_t* mask) {
  return guarded([&]() -> int {
    return ransac_estimate_host(0, n_clusters, offsets, azimuth, doppler, nullptr, params,
                                rng_cluster_index, inlier_count, winning_trial, mask, nullptr,
                                false);
  });
}

int rvk_ransac_estimate(int64_t frame_id, int32_t n_clusters, const int64_t* offsets,
                        const double* azimuth, const double* doppler, const int32_t* cluster_ids,
                        const rvk_ransac_params* params, const int32_t* rng_cluster_index,
                        int32_t* inlier_count, int32_t* winning_trial, uint8_t* mask,
                        rvk_estimate* out) {
  return guarded([&]() -> int {
    return ransac_estimate_host(frame_id, n_clusters, offsets, azimuth, doppler, cluster_ids,
                                params, rng_cluster_index, inlier_count, winning_trial, mask, out,
                                true);
  });
}

int rvk_ransac_estimate_packed(int64_t frame_id, int32_t n_clusters, const int64_t* offsets,
                               const double* azimuth, const double* doppler,
                               const int32_t* cluster_ids, const rvk_ransac_params* params,
                               const int32_t* rng_cluster_index, int32_t* inlier_count,
                               int32_t* winning_trial, uint8_t* mask_bits, rvk_estimate* out) {
  return guarded([&]() -> int {
    return ransac_estimate_host(frame_id, n_clusters, offsets, azimuth, doppler, cluster_ids,
                                params, rng_cluster_index, inlier_count, winning_trial, mask_bits,
                                out, true, true);
  });
}

int rvk_ransac_estimate_multi(int32_t n_devices, const int32_t* devices, int64_t frame_id,
                              int32_t n_clusters, const int64_t* offsets, const double* azimuth,
                              const double* doppler, const int32_t* cluster_ids,
                              const rvk_ransac_params* params, const int32_t* rng_cluster_index,
                              int32_t* inlier_count, int32_t* winning_trial, uint8_t* mask,
                              rvk_estimate* out) {
  return guarded([&]() -> int {
    if (n_devices < 1 || devices == nullptr)
      return fail(RVK_EINVAL, "rvk_ransac_estimate_multi: need at least one device");
    // the reference's checks on the whole frame first, so messages and the
    // offending cluster index refer to the caller's frame
    int st = validate_params(params, "run_ransac");
    if (st != RVK_OK) return st;
    st = validate_offsets(n_clusters, offsets, kMinClusterSize, "run_ransac");
    if (st != RVK_OK) return st;
    if (n_clusters == 0) return RVK_OK;
    if ((azimuth == nullptr || doppler == nullptr) && offsets[n_clusters] > 0)
      return fail(RVK_EINVAL, "run_ransac: null point arrays");
    // contiguous cluster ranges of about equal points (the work is T x points)
    const int64_t P = offsets[n_clusters];
    std::vector<int32_t> cut(1, 0);
    for (int i = 1; i < n_devices; ++i) {
      int32_t c = cut.back();
      while (c < n_clusters && offsets[c] < P * i / n_devices) ++c;
      cut.push_back(c);
    }
    cut.push_back(n_clusters);
    struct Part {
      int status = RVK_OK;
      std::string error;
      int32_t error_cluster = -1;
    };
    std::vector<Part> part(n_devices);
    auto work = [&](int i) {
      const int32_t c0 = cut[i], nc = cut[i + 1] - cut[i];
      if (nc == 0) return;
      part[i].status = guarded([&]() -> int {
        RVK_CUDA(cudaSetDevice(devices[i]));
        std::vector<int64_t> off(static_cast<size_t>(nc) + 1);
        std::vector<int32_t> key(static_cast<size_t>(nc)), ids(static_cast<size_t>(nc));
        for (int32_t j = 0; j <= nc; ++j) off[j] = offsets[c0 + j] - offsets[c0];
        for (int32_t j = 0; j < nc; ++j) {  // RNG keys and ids stay frame-positional
          key[j] = rng_cluster_index ? rng_cluster_index[c0 + j] : c0 + j;
          ids[j] = cluster_ids ? cluster_ids[c0 + j] : c0 + j;
        }
        const int64_t p0 = offsets[c0];
        return ransac_estimate_host(frame_id, nc, off.data(), azimuth + p0, doppler + p0,
                                    ids.data(), params, key.data(),
                                    inlier_count ? inlier_count + c0 : nullptr,
                                    winning_trial ? winning_trial + c0 : nullptr,
                                    mask ? mask + p0 : nullptr, out ? out + c0 : nullptr, true);
      });
      part[i].error = g_error;
      part[i].error_cluster = g_error_cluster >= 0 ? g_error_cluster + c0 : -1;
    };
    int saved = 0;
    RVK_CUDA(cudaGetDevice(&saved));
    multi_pool().run(n_devices, work);
    cudaSetDevice(saved);
    for (const Part& q : part)
      if (q.status != RVK_OK) {
        g_error_cluster = q.error_cluster;
        return fail(q.status, "%s", q.error.c_str());
      }
    return RVK_OK;
  });
}

int rvk_estimate_all(int64_t frame_id, int32_t n_clusters, const int64_t* offsets,
                     const double* azimuth, const double* doppler, const int32_t* cluster_ids,
                     const uint8_t* mask, int32_t /*workers*/, rvk_estimate* out) {
  return guarded([&]() -> int {
    // estimate_all validates the mask count/size (src/velocity.cpp:95-106);
    // in the CSR form the mask is P bytes aligned with the points, so only
    // the structural checks remain.
    int st = validate_offsets(n_clusters, offsets, 0, "estimate_all");
    if (st != RVK_OK) return st;
    if (n_clusters == 0) return RVK_OK;
    if (mask == nullptr && offsets[n_clusters] > 0)
      return fail(RVK_EINVAL, "estimate_all: one mask per cluster required");
    Context& ctx = context();
    uint8_t* d_mask = nullptr;
    FrameDev f = stage_frame(ctx, frame_id, n_clusters, offsets, azimuth, doppler, cluster_ids,
                             nullptr, false, mask, &d_mask);
    rvk_estimate* d_est = ctx.out.get<rvk_estimate>(n_clusters);
    launch_refit(f, d_mask, d_est, ctx.stream);
    check_launch();
    void* h = ctx.stage_out.get(sizeof(rvk_estimate) * n_clusters);
    RVK_CUDA(cudaMemcpyAsync(h, d_est, sizeof(rvk_estimate) * n_clusters, cudaMemcpyDeviceToHost,
                             ctx.stream));
    RVK_CUDA(cudaStreamSynchronize(ctx.stream));
    std::memcpy(out, h, sizeof(rvk_estimate) * n_clusters);
    return RVK_OK;
  });
}

int rvk_ransac_estimate_device(int64_t frame_id, int32_t n_clusters, int64_t n_points,
                               const int64_t* d_offsets, const double* d_azimuth,
                               const double* d_doppler, const int32_t* d_cluster_ids,
                               const rvk_ransac_params* params, const int32_t* d_rng_cluster_index,
                               int32_t* d_inlier_count, int32_t* d_winning_trial, uint8_t* d_mask,
                               rvk_estimate* d_out, void* stream) {
  return guarded([&]() -> int {
    int st = validate_params(params, "run_ransac");
    if (st != RVK_OK) return st;
    if (n_clusters < 0 || n_points < 0) return fail(RVK_EINVAL, "run_ransac: negative sizes");
    if (n_clusters == 0) return RVK_OK;
    if (d_mask == nullptr) return fail(RVK_EINVAL, "run_ransac: device mask buffer required");
    Context& ctx = context();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    FrameDev f;
    f.n_clusters = n_clusters;
    f.n_points = n_points;
    f.offsets = d_offsets;
    f.azimuth = d_azimuth;
    f.doppler = d_doppler;
    f.cluster_ids = d_cluster_ids;
    f.keys = d_rng_cluster_index;
    f.order = nullptr;
    f.frame_id = frame_id;
    Scratch sc = scratch(ctx.workspace(s), n_clusters, n_points, params->max_trials);
    Outputs o;
    o.inlier_count = d_inlier_count;
    o.winning_trial = d_winning_trial;
    o.mask = d_mask;
    o.est = d_out;
    run_pipeline(f, *params, sc, o, s);
    return RVK_OK;
  });
}

int rvk_trial_counts(int32_t n_clusters, const int64_t* offsets, const double* azimuth,
                     const double* doppler, const rvk_ransac_params* params,
                     const int32_t* rng_cluster_index, int32_t* counts) {
  return guarded([&]() -> int {
    int st = validate_params(params, "run_ransac");
    if (st != RVK_OK) return st;
    st = validate_offsets(n_clusters, offsets, kMinClusterSize, "run_ransac");
    if (st != RVK_OK) return st;
    if (n_clusters == 0) return RVK_OK;
    Context& ctx = context();
    const int64_t P = offsets[n_clusters];
    FrameDev f = stage_frame(ctx, 0, n_clusters, offsets, azimuth, doppler, nullptr,
                             rng_cluster_index, false, nullptr, nullptr);
    Scratch s = scratch(ctx.workspace(ctx.stream), n_clusters, P, params->max_trials);
    const size_t nc = static_cast<size_t>(n_clusters) * params->max_trials;
    int32_t* d_counts = ctx.workspace(ctx.stream).aux.get<int32_t>(nc);
    launch_prep(f, params->threshold_scale, s, ctx.stream);
    launch_mad_exact(f, params->threshold_scale, s, ctx.stream);
    launch_exact_counts(f, *params, s, d_counts, ctx.stream);
    check_launch();
    void* h = ctx.stage_out.get(sizeof(int32_t) * nc);
    RVK_CUDA(cudaMemcpyAsync(h, d_counts, sizeof(int32_t) * nc, cudaMemcpyDeviceToHost,
                             ctx.stream));
    RVK_CUDA(cudaStreamSynchronize(ctx.stream));
    std::memcpy(counts, h, sizeof(int32_t) * nc);
    return RVK_OK;
  });
}

int rvk_seed_pairs(int32_t n_clusters, const int64_t* offsets, const rvk_ransac_params* params,
                   const int32_t* rng_cluster_index, int32_t* pairs) {
  return guarded([&]() -> int {
    int st = validate_params(params, "run_ransac");
    if (st != RVK_OK) return st;
    st = validate_offsets(n_clusters, offsets, 2, "draw_seed_pair");
    if (st != RVK_OK) {
      if (st == RVK_ECLUSTER_TOO_SMALL) return fail(RVK_EINVAL, "draw_seed_pair: need at least 2 points");
      return st;
    }
    if (n_clusters == 0) return RVK_OK;
    Context& ctx = context();
    const size_t nc = static_cast<size_t>(n_clusters) * params->max_trials;
    const size_t o_keys = align_up(sizeof(int64_t) * (n_clusters + 1));
    const size_t total = align_up(o_keys + sizeof(int32_t) * n_clusters);
    char* h = static_cast<char*>(ctx.stage_in.get(total));
    char* d = ctx.in.get<char>(total);
    std::memcpy(h, offsets, sizeof(int64_t) * (n_clusters + 1));
    if (rng_cluster_index) std::memcpy(h + o_keys, rng_cluster_index, sizeof(int32_t) * n_clusters);
    RVK_CUDA(cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, ctx.stream));
    FrameDev f;
    f.n_clusters = n_clusters;
    f.offsets = reinterpret_cast<const int64_t*>(d);
    f.keys = rng_cluster_index ? reinterpret_cast<const int32_t*>(d + o_keys) : nullptr;
    int32_t* d_pairs = ctx.workspace(ctx.stream).aux.get<int32_t>(2 * nc);
    launch_seed_pairs(f, *params, d_pairs, ctx.stream);
    check_launch();
    void* ho = ctx.stage_out.get(sizeof(int32_t) * 2 * nc);
    RVK_CUDA(cudaMemcpyAsync(ho, d_pairs, sizeof(int32_t) * 2 * nc, cudaMemcpyDeviceToHost,
                             ctx.stream));
    RVK_CUDA(cudaStreamSynchronize(ctx.stream));
    std::memcpy(pairs, ho, sizeof(int32_t) * 2 * nc);
    return RVK_OK;
  });
}

int rvk_cluster_thresholds(int32_t n_clusters, const int64_t* offsets, const double* azimuth,
                           const double* doppler, double threshold_scale, double* norm,
                           double* threshold) {
  return guarded([&]() -> int {
    int st = validate_offsets(n_clusters, offsets, 1, "normalize_cluster");
    if (st != RVK_OK) {
      if (st == RVK_ECLUSTER_TOO_SMALL) return fail(RVK_EINVAL, "normalize_cluster: empty cluster");
      return st;
    }
    if (n_clusters == 0) return RVK_OK;
    Context& ctx = context();
    const int64_t P = offsets[n_clusters];
    FrameDev f = stage_frame(ctx, 0, n_clusters, offsets, azimuth, doppler, nullptr, nullptr,
                             false, nullptr, nullptr);
    Scratch s = scratch(ctx.workspace(ctx.stream), n_clusters, P, 1);
    launch_prep(f, threshold_scale, s, ctx.stream);
    launch_mad_exact(f, threshold_scale, s, ctx.stream);
    check_launch();
    const size_t o_st = align_up(sizeof(double) * 4 * n_clusters);
    const size_t total = o_st + sizeof(double4) * n_clusters;
    char* h = static_cast<char*>(ctx.stage_out.get(total));
    RVK_CUDA(cudaMemcpyAsync(h, s.norm, sizeof(double) * 4 * n_clusters, cudaMemcpyDeviceToHost,
                             ctx.stream));
    RVK_CUDA(cudaMemcpyAsync(h + o_st, s.stat, sizeof(double4) * n_clusters,
                             cudaMemcpyDeviceToHost, ctx.stream));
    RVK_CUDA(cudaStreamSynchronize(ctx.stream));
    if (norm) std::memcpy(norm, h, sizeof(double) * 4 * n_clusters);
    const double4* stv = reinterpret_cast<const double4*>(h + o_st);
    if (threshold)
      for (int32_t c = 0; c < n_clusters; ++c) threshold[c] = stv[c].w;
    return RVK_OK;
  });
}

int rvk_stream_create(const rvk_ransac_params* params, int32_t depth, rvk_frame_stream** out) {
  return guarded([&]() -> int {
    if (out == nullptr) return fail(RVK_EINVAL, "rvk_stream_create: out is null");
    *out = nullptr;
    const int st = validate_params(params, "run_ransac");
    if (st != RVK_OK) return st;
    if (depth < 0 || depth > 8) return fail(RVK_EINVAL, "rvk_stream_create: depth must be in [0, 8]");
    auto* h = new rvk_frame_stream();
    FrameStream& fs = h->impl;
    fs.params = *params;
    fs.depth = depth ? depth : 3;
    try {
      RVK_CUDA(cudaGetDevice(&fs.device));
      RVK_CUDA(cudaStreamCreateWithFlags(&fs.copy, cudaStreamNonBlocking));
      for (auto& c : fs.compute) RVK_CUDA(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
      fs.slots.resize(fs.depth);
      for (auto& s : fs.slots) {
        RVK_CUDA(cudaEventCreateWithFlags(&s.landed, cudaEventDisableTiming));
        RVK_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
      }
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
    return RVK_OK;
  });
}

int rvk_stream_submit(rvk_frame_stream* s, int64_t frame_id, int32_t n_clusters,
                      const int64_t* offsets, const double* azimuth, const double* doppler,
                      const int32_t* cluster_ids, const int32_t* rng_cluster_index,
                      int32_t* inlier_count, int32_t* winning_trial, uint8_t* mask,
                      rvk_estimate* out, int64_t* ticket) {
  return guarded([&]() -> int {
    if (s == nullptr) return fail(RVK_EINVAL, "rvk_stream_submit: null stream");
    return s->impl.submit(frame_id, n_clusters, offsets, azimuth, doppler, cluster_ids,
                          rng_cluster_index, inlier_count, winning_trial, mask, out, ticket);
  });
}

int rvk_stream_submit_packed(rvk_frame_stream* s, int64_t frame_id, int32_t n_clusters,
                             const int64_t* offsets, const double* azimuth,
                             const double* doppler, const int32_t* cluster_ids,
                             const int32_t* rng_cluster_index, int32_t* inlier_count,
                             int32_t* winning_trial, uint8_t* mask_bits, rvk_estimate* out,
                             int64_t* ticket) {
  return guarded([&]() -> int {
    if (s == nullptr) return fail(RVK_EINVAL, "rvk_stream_submit: null stream");
    return s->impl.submit(frame_id, n_clusters, offsets, azimuth, doppler, cluster_ids,
                          rng_cluster_index, inlier_count, winning_trial, mask_bits, out, ticket,
                          true);
  });
}

int rvk_stream_wait(rvk_frame_stream* s, int64_t ticket) {
  return guarded([&]() -> int {
    if (s == nullptr) return fail(RVK_EINVAL, "rvk_stream_wait: null stream");
    return s->impl.wait(ticket);
  });
}

int rvk_stream_destroy(rvk_frame_stream* s) {
  return guarded([&]() -> int {
    if (s == nullptr) return RVK_OK;
    FrameStream& fs = s->impl;
    int rc = RVK_OK;
    DeviceGuard guard(fs.device);
    try {
      for (auto& sl : fs.slots) fs.complete(sl);
    } catch (const CudaError& e) {
      rc = fail(RVK_ECUDA, "CUDA error %s in %s", cudaGetErrorName(e.e), e.what);
    }
    for (auto& sl : fs.slots) {
      if (sl.landed) cudaEventDestroy(sl.landed);
      if (sl.done) cudaEventDestroy(sl.done);
      sl.ws.release();
      for (DevBuf* b : {&sl.in, &sl.out}) b->release();
      for (HostBuf* b : {&sl.small_in, &sl.big_in, &sl.stage_out}) b->release();
    }
    if (fs.copy) cudaStreamDestroy(fs.copy);
    for (auto& c : fs.compute)
      if (c) cudaStreamDestroy(c);
    delete s;
    return rc;
  });
}

int rvk_dbscan(int64_t n, const double* x, const double* y, const double* z,
               const rvk_clustering_params* params, int32_t* labels) {
  return guarded([&]() -> int {
    const int st = validate_clustering(params);
    if (st != RVK_OK) return st;
    if (n < 0) return fail(RVK_EINVAL, "dbscan: negative point count");
    if (n == 0) return RVK_OK;
    if (n >= (int64_t{1} << 31)) return fail(RVK_EINVAL, "dbscan: too many points");
    const bool xyz = params->features == RVK_FEATURES_XYZ;
    if (x == nullptr || y == nullptr || (xyz && z == nullptr) || labels == nullptr)
      return fail(RVK_EINVAL, "dbscan: null point arrays");
    Context& ctx = context();
    const FramePts f = upload_points(ctx, n, x, y, xyz ? z : nullptr, nullptr, nullptr);
    const DbscanLayout L = dbscan_layout(n, xyz);
    char* ws = ctx.db.get<char>(L.total);
    int32_t* d_labels = ctx.labels.get<int32_t>(static_cast<size_t>(n));
    launch_dbscan(n, f.x, f.y, f.z, params->eps, params->min_pts, L, ws, d_labels, ctx.stream);
    check_launch();
    int32_t* h = static_cast<int32_t*>(ctx.stage_out.get(sizeof(int32_t) * n));
    RVK_CUDA(cudaMemcpyAsync(h, d_labels, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx.stream));
    RVK_CUDA(cudaStreamSynchronize(ctx.stream));
    std::memcpy(labels, h, sizeof(int32_t) * n);
    return RVK_OK;
  });
}

int rvk_extract_clusters(int64_t n, int32_t* labels, int32_t min_cluster_size,
                         int32_t* n_clusters, int64_t* offsets, int32_t* point_indices) {
  return guarded([&]() -> int {
    if (min_cluster_size < 1)
      return fail(RVK_EINVAL, "extract_clusters: min_cluster_size must be at least 1");
    if (n < 0 || n >= (int64_t{1} << 31)) return fail(RVK_EINVAL, "extract_clusters: bad size");
    if (n_clusters) *n_clusters = 0;
    if (offsets) offsets[0] = 0;
    if (n == 0) return RVK_OK;
    if (labels == nullptr || n_clusters == nullptr || offsets == nullptr ||
        point_indices == nullptr)
      return fail(RVK_EINVAL, "extract_clusters: null arrays");
    int32_t max_label = -1;
    for (int64_t i = 0; i < n; ++i) max_label = std::max(max_label, labels[i]);
    if (max_label < 0) return RVK_OK;
    const int64_t k = static_cast<int64_t>(max_label) + 1;
    Context& ctx = context();
    const int64_t cap = std::max(n, k);
    const DbscanLayout L = dbscan_layout(cap, false);
    char* ws = ctx.db.get<char>(L.total);
    // device block: labels[n] | offsets[k+1] | point_indices[n] | count
    const size_t o_off = align_up(sizeof(int32_t) * n);
    const size_t o_pi = align_up(o_off + sizeof(int64_t) * (k + 1));
    const size_t o_m = align_up(o_pi + sizeof(int32_t) * n);
    const size_t total = o_m + 256;
    char* d = ctx.out.get<char>(total);
    char* h = static_cast<char*>(ctx.stage_out.get(total));
    std::memcpy(h, labels, sizeof(int32_t) * n);
    RVK_CUDA(cudaMemcpyAsync(d, h, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx.stream));
    launch_extract(n, reinterpret_cast<int32_t*>(d), static_cast<int32_t>(k), min_cluster_size, L,
                   ws, reinterpret_cast<int64_t*>(d + o_off), reinterpret_cast<int32_t*>(d + o_pi),
                   reinterpret_cast<int32_t*>(d + o_m), ctx.stream);
    check_launch();
    RVK_CUDA(cudaMemcpyAsync(h, d, total, cudaMemcpyDeviceToHost, ctx.stream));
    RVK_CUDA(cudaStreamSynchronize(ctx.stream));
    const int32_t m = *reinterpret_cast<int32_t*>(h + o_m);
    *n_clusters = m;
    std::memcpy(labels, h, sizeof(int32_t) * n);
    std::memcpy(offsets, h + o_off, sizeof(int64_t) * (m + 1));
    std::memcpy(point_indices, h + o_pi, sizeof(int32_t) * offsets[m]);
    return RVK_OK;
  });
}

int rvk_estimate_frame(int64_t frame_id, int64_t n, const double* x, const double* y,
                       const double* z, const double* doppler, const double* azimuth,
                       const rvk_clustering_params* cparams, int32_t min_cluster_size,
                       const rvk_ransac_params* rparams, int32_t* labels, int32_t* n_clusters,
                       int64_t* offsets, int32_t* point_indices, int32_t* inlier_count,
                       int32_t* winning_trial, uint8_t* mask, rvk_estimate* out) {
  return guarded([&]() -> int {
    int st = validate_clustering(cparams);
    if (st != RVK_OK) return st;
    if (min_cluster_size < 1)
      return fail(RVK_EINVAL, "extract_clusters: min_cluster_size must be at least 1");
    st = validate_params(rparams, "run_ransac");
    if (st != RVK_OK) return st;
    if (n < 0 || n >= (int64_t{1} << 31)) return fail(RVK_EINVAL, "dbscan: bad point count");
    if (n_clusters) *n_clusters = 0;
    if (offsets) offsets[0] = 0;
    if (n == 0) return RVK_OK;
    const bool xyz = cparams->features == RVK_FEATURES_XYZ;
    if (x == nullptr || y == nullptr || (xyz && z == nullptr) || doppler == nullptr ||
        azimuth == nullptr || labels == nullptr || n_clusters == nullptr || offsets == nullptr ||
        point_indices == nullptr)
      return fail(RVK_EINVAL, "estimate_frame: null arrays");
    Context& ctx = context();
    const FramePts f = upload_points(ctx, n, x, y, xyz ? z : nullptr, doppler, azimuth);
    const DbscanLayout L = dbscan_layout(n, xyz);
    char* ws = ctx.db.get<char>(L.total);
    // device: labels[n] | offsets[n+1] | point_indices[n] | m | gaz[n] | gdop[n]
    const size_t o_off = align_up(sizeof(int32_t) * n);
    const size_t o_pi = align_up(o_off + sizeof(int64_t) * (n + 1));
    const size_t o_m = align_up(o_pi + sizeof(int32_t) * n);
    const size_t o_gaz = align_up(o_m + 256);
    const size_t o_gdop = align_up(o_gaz + sizeof(double) * n);
    const size_t total = align_up(o_gdop + sizeof(double) * n);
    char* d = ctx.labels.get<char>(total);
    int32_t* d_labels = reinterpret_cast<int32_t*>(d);
    int64_t* d_off = reinterpret_cast<int64_t*>(d + o_off);
    int32_t* d_pi = reinterpret_cast<int32_t*>(d + o_pi);
    launch_dbscan(n, f.x, f.y, f.z, cparams->eps, cparams->min_pts, L, ws, d_labels, ctx.stream);
    launch_extract(n, d_labels, static_cast<int32_t>(n), min_cluster_size, L, ws, d_off, d_pi,
                   reinterpret_cast<int32_t*>(d + o_m), ctx.stream);
    check_launch();
    // the cluster count and offsets decide the launch shapes: one sync
    char* h = static_cast<char*>(ctx.stage_out.get(o_m + 256));
    RVK_CUDA(cudaMemcpyAsync(h, d, o_m + 256, cudaMemcpyDeviceToHost, ctx.stream));
    RVK_CUDA(cudaStreamSynchronize(ctx.stream));
    const int32_t m = *reinterpret_cast<int32_t*>(h + o_m);
    *n_clusters = m;
    std::memcpy(labels, h, sizeof(int32_t) * n);
    std::memcpy(offsets, h + o_off, sizeof(int64_t) * (m + 1));
    const int64_t P = offsets[m];
    std::memcpy(point_indices, h + o_pi, sizeof(int32_t) * P);
    if (m == 0) return RVK_OK;
    st = validate_offsets(m, offsets, kMinClusterSize, "run_ransac");  // ransac.cpp:147-156
    if (st != RVK_OK) return st;
    double* gaz = reinterpret_cast<double*>(d + o_gaz);
    double* gdop = reinterpret_cast<double*>(d + o_gdop);
    launch_gather(P, d_pi, f.az, f.dop, gaz, gdop, ctx.stream);
    FrameDev fd;
    fd.n_clusters = m;
    fd.n_points = P;
    fd.offsets = d_off;
    fd.azimuth = gaz;
    fd.doppler = gdop;
    fd.frame_id = frame_id;  // keys / cluster ids: positional = the compact ids
    Scratch scr = scratch(ctx.workspace(ctx.stream), m, P, rparams->max_trials);
    const OutLayout OL(m, P);
    char* dout = ctx.out.get<char>(OL.total);
    Outputs o;
    o.inlier_count = reinterpret_cast<int32_t*>(dout + OL.o_cnt);
    o.winning_trial = reinterpret_cast<int32_t*>(dout + OL.o_tr);
    o.est = reinterpret_cast<rvk_estimate*>(dout + OL.o_est);
    o.mask = reinterpret_cast<uint8_t*>(dout + OL.o_mask);
    run_pipeline(fd, *rparams, scr, o, ctx.stream);
    char* hout = static_cast<char*>(ctx.stage_out.get(OL.total));
    RVK_CUDA(cudaMemcpyAsync(hout, dout, OL.total, cudaMemcpyDeviceToHost, ctx.stream));
    RVK_CUDA(cudaStreamSynchronize(ctx.stream));
    if (inlier_count) std::memcpy(inlier_count, hout + OL.o_cnt, sizeof(int32_t) * m);
    if (winning_trial) std::memcpy(winning_trial, hout + OL.o_tr, sizeof(int32_t) * m);
    if (out) std::memcpy(out, hout + OL.o_est, sizeof(rvk_estimate) * m);
    if (mask) std::memcpy(mask, hout + OL.o_mask, P);
    return RVK_OK;
  });
}

int rvk_combine_masks(int64_t n, const int32_t* labels, int32_t n_masks, const int32_t* mask_ids,
                      const int64_t* mask_offsets, const uint8_t* masks, uint8_t* result) {
  return guarded([&]() -> int {
    if (n < 0 || n >= (int64_t{1} << 31) || n_masks < 0)
      return fail(RVK_EINVAL, "combine_masks: bad sizes");
    if (n == 0) return RVK_OK;
    if (result == nullptr) return fail(RVK_EINVAL, "combine_masks: null result");
    if (n_masks == 0 || labels == nullptr) {  // src/ransac.cpp:220-222
      std::memset(result, 0, static_cast<size_t>(n));
      return RVK_OK;
    }
    if (mask_ids == nullptr || mask_offsets == nullptr)
      return fail(RVK_EINVAL, "combine_masks: null mask arrays");
    const int64_t P = mask_offsets[n_masks];
    // ids sorted ascending, the lowest mask index first among equal ids
    std::vector<int32_t> order(static_cast<size_t>(n_masks));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return mask_ids[a] < mask_ids[b]; });
    Context& ctx = context();
    const size_t o_ids = align_up(sizeof(int32_t) * n);
    const size_t o_of = align_up(o_ids + sizeof(int32_t) * n_masks);
    const size_t o_off = align_up(o_of + sizeof(int32_t) * n_masks);
    const size_t o_m = align_up(o_off + sizeof(int64_t) * (n_masks + 1));
    const size_t o_res = align_up(o_m + static_cast<size_t>(P));
    const size_t total = align_up(o_res + static_cast<size_t>(n));
    char* h = static_cast<char*>(ctx.stage_in.get(total));
    char* d = ctx.in.get<char>(total);
    std::memcpy(h, labels, sizeof(int32_t) * n);
    int32_t* hid = reinterpret_cast<int32_t*>(h + o_ids);
    int32_t* hof = reinterpret_cast<int32_t*>(h + o_of);
    for (int32_t k = 0; k < n_masks; ++k) {
      hid[k] = mask_ids[order[static_cast<size_t>(k)]];
      hof[k] = order[static_cast<size_t>(k)];
    }
    std::memcpy(h + o_off, mask_offsets, sizeof(int64_t) * (n_masks + 1));
    if (P > 0) std::memcpy(h + o_m, masks, static_cast<size_t>(P));
    RVK_CUDA(cudaMemcpyAsync(d, h, o_res, cudaMemcpyHostToDevice, ctx.stream));
    const DbscanLayout L = dbscan_layout(n, false);
    char* ws = ctx.db.get<char>(L.total);
    launch_combine_masks(n, reinterpret_cast<int32_t*>(d), n_masks,
                         reinterpret_cast<int32_t*>(d + o_ids), reinterpret_cast<int32_t*>(d + o_of),
                         reinterpret_cast<int64_t*>(d + o_off),
                         reinterpret_cast<uint8_t*>(d + o_m), L, ws,
                         reinterpret_cast<uint8_t*>(d + o_res), ctx.stream);
    check_launch();
    RVK_CUDA(cudaMemcpyAsync(h + o_res, d + o_res, static_cast<size_t>(n), cudaMemcpyDeviceToHost,
                             ctx.stream));
    RVK_CUDA(cudaStreamSynchronize(ctx.stream));
    std::memcpy(result, h + o_res, static_cast<size_t>(n));
    return RVK_OK;
  });
}

void rvk_profile_enable(int32_t on) { g_prof.on = on != 0; }

int rvk_profile_read(double* ms, int64_t* launches, int32_t n_stages) {
  return guarded([&]() -> int {
    for (int i = 0; i < n_stages; ++i) {
      if (ms) ms[i] = 0.0;
      if (launches) launches[i] = 0;
    }
    for (const StageRec& r : g_prof.recs) {
      RVK_CUDA(cudaEventSynchronize(r.b));
      float t = 0.f;
      RVK_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
      if (r.stage < n_stages) {
        if (ms) ms[r.stage] += t;
        if (launches) launches[r.stage] += 1;
      }
      g_prof.pool.push_back(r.a);
      g_prof.pool.push_back(r.b);
    }
    g_prof.recs.clear();
    return RVK_OK;
  });
}

}  // extern "C"
