// sm_100a DBSCAN + extract_clusters: the clustering stage upstream of the
// velocity-profile path, bit-exact with
//
//   rvk::dbscan            src/clustering.cpp:24-114
//   rvk::extract_clusters  src/clustering.cpp:116-155
//
// The reference builds O(N^2) neighbour lists; here points are hashed into a
// uniform grid of cell size eps * (1 + 2^-20) (every eps-neighbour lies in
// one of the 3^d adjacent cells: the margin covers the FP64 rounding of the
// distance test and of the cell coordinates), sorted by cell with a radix
// sort, and every query scans the adjacent cells with the reference's exact
// FP64 test  dx*dx + dy*dy (+ dz*dz) <= eps*eps  (squared_distance,
// clustering.cpp:11-20, no FMA contraction). Then
//   core      |N_eps(p)| >= min_pts, N_eps including p itself (:56-60);
//   clusters  connected components of the core-core eps-graph by lock-free
//             union-find linking larger roots under smaller ones, so every
//             root is its component's smallest core index; ids are the
//             ranks of those roots, i.e. the order in which the reference's
//             ascending BFS loop meets the components (:62-89);
//   border    a non-core point with core neighbours joins the cluster of the
//             nearest one, ties to the lowest index (:91-113);
//   extract   clusters below min_cluster_size become noise, surviving ids are
//             compacted in order, members listed in ascending point order
//             (a stable radix sort by label) (:116-155).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>

#include "rvk_kernels.cuh"

namespace rvk_gpu {
namespace {

constexpr int kDbThreads = 256;
constexpr double kCellMargin = 1.0 + 0x1p-20;

struct Pts {
  const double* x;
  const double* y;
  const double* z;  // sorted copies (cell order)
  bool xyz;
};

// squared_distance (src/clustering.cpp:11-20), FP64 round-to-nearest in the
// reference's operation order. (a - b)^2 == (b - a)^2 exactly, so the
// argument order does not matter.
__device__ __forceinline__ double sq_dist(const Pts& p, int64_t i, int64_t j) {
  const double dx = __dsub_rn(p.x[i], p.x[j]);
  const double dy = __dsub_rn(p.y[i], p.y[j]);
  double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  if (p.xyz) {
    const double dz = __dsub_rn(p.z[i], p.z[j]);
    d2 = __dadd_rn(d2, __dmul_rn(dz, dz));
  }
  return d2;
}

__device__ __forceinline__ uint32_t cell_hash(long long cx, long long cy, long long cz,
                                              uint32_t mask) {
  uint64_t h = static_cast<uint64_t>(cx) * 0x9E3779B97F4A7C15ull;
  h ^= static_cast<uint64_t>(cy) * 0xC2B2AE3D27D4EB4Full;
  h ^= static_cast<uint64_t>(cz) * 0x165667B19E3779F9ull;
  h ^= h >> 29;
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= h >> 32;
  return static_cast<uint32_t>(h) & mask;
}

__device__ __forceinline__ void cell_of(double x, double y, double z, double inv_cs,
                                        long long& cx, long long& cy, long long& cz) {
  cx = static_cast<long long>(floor(x * inv_cs));
  cy = static_cast<long long>(floor(y * inv_cs));
  cz = static_cast<long long>(floor(z * inv_cs));
}

__global__ void db_keys(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                        const double* __restrict__ z, double inv_cs, uint32_t mask,
                        uint32_t* __restrict__ keys, int32_t* __restrict__ idx) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long cx, cy, cz;
  cell_of(x[i], y[i], z ? z[i] : 0.0, inv_cs, cx, cy, cz);
  keys[i] = cell_hash(cx, cy, cz, mask);
  idx[i] = static_cast<int32_t>(i);
}

// Cell ranges of the sorted keys and the coordinates in cell order.
__global__ void db_cells(int64_t n, const uint32_t* __restrict__ skeys,
                         const int32_t* __restrict__ sidx, const double* __restrict__ x,
                         const double* __restrict__ y, const double* __restrict__ z,
                         int32_t* __restrict__ cstart, int32_t* __restrict__ cend,
                         double* __restrict__ sx, double* __restrict__ sy, double* __restrict__ sz) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const uint32_t k = skeys[s];
  if (s == 0 || skeys[s - 1] != k) cstart[k] = static_cast<int32_t>(s);
  if (s == n - 1 || skeys[s + 1] != k) cend[k] = static_cast<int32_t>(s + 1);
  const int32_t i = sidx[s];
  sx[s] = x[i];
  sy[s] = y[i];
  if (z) sz[s] = z[i];
}

// The distinct buckets of the 3^d cells around sorted point s.
struct Nbr {
  uint32_t key[27];
  int cnt;
};
__device__ __forceinline__ void neighbour_buckets(const Pts& p, int64_t s, double inv_cs,
                                                  uint32_t mask, Nbr& nb) {
  long long cx, cy, cz;
  cell_of(p.x[s], p.y[s], p.xyz ? p.z[s] : 0.0, inv_cs, cx, cy, cz);
  nb.cnt = 0;
  const int dzr = p.xyz ? 1 : 0;
  for (int dz = -dzr; dz <= dzr; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const uint32_t k = cell_hash(cx + dx, cy + dy, cz + dz, mask);
        bool seen = false;
        for (int q = 0; q < nb.cnt; ++q) seen |= nb.key[q] == k;
        if (!seen) nb.key[nb.cnt++] = k;
      }
}

// core[s] = |N_eps| >= min_pts (the point itself included: d2 = 0).
__global__ void db_core(int64_t n, Pts p, double inv_cs, uint32_t mask, double eps2, int min_pts,
                        const int32_t* __restrict__ cstart, const int32_t* __restrict__ cend,
                        uint8_t* __restrict__ core) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  Nbr nb;
  neighbour_buckets(p, s, inv_cs, mask, nb);
  int count = 0;
  for (int q = 0; q < nb.cnt && count < min_pts; ++q) {
    const int32_t e = cend[nb.key[q]];
    for (int32_t t = cstart[nb.key[q]]; t < e && count < min_pts; ++t)
      count += sq_dist(p, s, t) <= eps2;
  }
  core[s] = count >= min_pts;
}

// Root of a (path halving). Parents only ever move to smaller indices
// (roots are linked under smaller roots, halving jumps to an ancestor), so
// the walk terminates under concurrent updates.
__device__ __forceinline__ int32_t uf_find(int32_t* parent_, int32_t a) {
  volatile int32_t* parent = parent_;
  int32_t cur = parent[a];
  while (cur != a) {
    const int32_t next = parent[cur];
    if (next != cur) atomicCAS(parent_ + a, cur, next);
    a = cur;
    cur = next;
  }
  return a;
}

// Links a and b; the smaller root survives, so a component's root is its
// smallest member (in ORIGINAL point indices, which `parent` is keyed by).
__device__ __forceinline__ void uf_union(int32_t* parent, int32_t a, int32_t b) {
  for (;;) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    if (a > b) {
      const int32_t t = a;
      a = b;
      b = t;
    }
    if (atomicCAS(&parent[b], b, a) == b) return;
  }
}

__global__ void db_parent_init(int64_t n, const int32_t* __restrict__ sidx,
                               const uint8_t* __restrict__ core, int32_t* __restrict__ parent) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int32_t i = sidx[s];
  parent[i] = core[s] ? i : -1;
}

// Hooking: every core point points at its smallest core eps-neighbour (or
// itself). Every pointer is a core-core edge and points to a smaller index,
// so this is already a union-find forest of the graph; the union pass then
// only has to merge the local trees.
__global__ void db_hook(int64_t n, Pts p, double inv_cs, uint32_t mask, double eps2,
                        const int32_t* __restrict__ cstart, const int32_t* __restrict__ cend,
                        const int32_t* __restrict__ sidx, const uint8_t* __restrict__ core,
                        int32_t* __restrict__ parent) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n || !core[s]) return;
  const int32_t i = sidx[s];
  int32_t m = i;
  Nbr nb;
  neighbour_buckets(p, s, inv_cs, mask, nb);
  for (int q = 0; q < nb.cnt; ++q) {
    const int32_t e = cend[nb.key[q]];
    for (int32_t t = cstart[nb.key[q]]; t < e; ++t) {
      if (!core[t]) continue;
      const int32_t j = sidx[t];
      if (j < m && sq_dist(p, s, t) <= eps2) m = j;
    }
  }
  parent[i] = m;
}

// Pointer jumping after hooking: every core point hangs directly under its
// tree's root, so the union pass recognises same-tree edges with one load.
__global__ void db_compress(int64_t n, int32_t* parent) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || parent[i] < 0) return;
  parent[i] = uf_find(parent, static_cast<int32_t>(i));
}

// Core-core eps edges: each edge once (from the endpoint with the larger
// sorted position). An edge whose far end already hangs directly under this
// point's current root is skipped with one load; otherwise both roots are
// found and linked.
__global__ void db_union(int64_t n, Pts p, double inv_cs, uint32_t mask, double eps2,
                         const int32_t* __restrict__ cstart, const int32_t* __restrict__ cend,
                         const int32_t* __restrict__ sidx, const uint8_t* __restrict__ core,
                         int32_t* parent) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n || !core[s]) return;
  const int32_t i = sidx[s];
  int32_t r = uf_find(parent, i);
  Nbr nb;
  neighbour_buckets(p, s, inv_cs, mask, nb);
  for (int q = 0; q < nb.cnt; ++q) {
    const int32_t b = cstart[nb.key[q]];
    const int32_t e = min(cend[nb.key[q]], static_cast<int32_t>(s));  // edges to t < s
    for (int32_t t = b; t < e; ++t) {
      if (!core[t]) continue;
      const int32_t j = sidx[t];
      // a possibly stale (L1) read is enough to prove j is in i's tree:
      // parents only ever move within a component
      const int32_t pj = __ldca(parent + j);
      if (pj == r || j == r) continue;
      if (sq_dist(p, s, t) > eps2) continue;
      const int32_t rj = uf_find(parent, j);
      if (rj == r) continue;
      uf_union(parent, r, rj);
      r = uf_find(parent, i);
    }
  }
}

// Roots of the core points; rep flag = "is the smallest core of its component".
__global__ void db_roots(int64_t n, int32_t* parent, int32_t* __restrict__ rep) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (parent[i] < 0) {
    rep[i] = 0;
    return;
  }
  const int32_t r = uf_find(parent, static_cast<int32_t>(i));
  rep[i] = r == i;
}

__global__ void db_flatten(int64_t n, const int32_t* __restrict__ parent_in,
                           int32_t* __restrict__ root) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t r = parent_in[i];
  if (r >= 0)
    while (parent_in[r] != r) r = parent_in[r];
  root[i] = r;
}

// Cluster id of core points: rank of their component's root among roots
// (exclusive scan of the rep flags); others -1 for now.
__global__ void db_label_core(int64_t n, const int32_t* __restrict__ root,
                              const int32_t* __restrict__ rep_rank, int32_t* __restrict__ labels) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t r = root[i];
  labels[i] = r >= 0 ? rep_rank[r] : -1;
}

// Border points: nearest core neighbour (lowest index on ties) -- compared in
// ORIGINAL indices, as the reference's neighbour scan.
__global__ void db_border(int64_t n, Pts p, double inv_cs, uint32_t mask, double eps2,
                          const int32_t* __restrict__ cstart, const int32_t* __restrict__ cend,
                          const int32_t* __restrict__ sidx, const uint8_t* __restrict__ core,
                          int32_t* __restrict__ labels) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n || core[s]) return;
  Nbr nb;
  neighbour_buckets(p, s, inv_cs, mask, nb);
  int32_t best = -1;
  double best_d2 = 0.0;
  for (int q = 0; q < nb.cnt; ++q) {
    const int32_t e = cend[nb.key[q]];
    for (int32_t t = cstart[nb.key[q]]; t < e; ++t) {
      if (!core[t]) continue;
      const double d2 = sq_dist(p, s, t);
      if (d2 > eps2) continue;
      const int32_t j = sidx[t];
      if (best == -1 || d2 < best_d2 || (d2 == best_d2 && j < best)) {
        best = j;
        best_d2 = d2;
      }
    }
  }
  if (best != -1) labels[sidx[s]] = labels[best];
}

// ---- extract_clusters
__global__ void ex_count(int64_t n, const int32_t* __restrict__ labels, int32_t* __restrict__ count) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t l = labels[i];
  if (l >= 0) atomicAdd(&count[l], 1);
}
__global__ void ex_keep(int64_t k, const int32_t* __restrict__ count, int32_t min_size,
                        int32_t* __restrict__ keep, int32_t* __restrict__ kept_count) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= k) return;
  const bool kp = count[l] >= min_size;
  keep[l] = kp;
  kept_count[l] = kp ? count[l] : 0;
}
// labels -> compact ids (or noise); sort keys: kept label, else UINT_MAX
__global__ void ex_remap(int64_t n, int32_t* __restrict__ labels, const int32_t* __restrict__ keep,
                         const int32_t* __restrict__ new_id, uint32_t* __restrict__ key,
                         int32_t* __restrict__ idx) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t l = labels[i];
  if (l >= 0) l = keep[l] ? new_id[l] : -1;
  labels[i] = l;
  key[i] = l >= 0 ? static_cast<uint32_t>(l) : 0xFFFFFFFFu;
  idx[i] = static_cast<int32_t>(i);
}
// offsets[c] for the compact ids: scatter the scanned kept counts
__global__ void ex_offsets(int64_t k, const int32_t* __restrict__ keep,
                           const int32_t* __restrict__ new_id, const int64_t* __restrict__ start,
                           const int32_t* __restrict__ count, int64_t* __restrict__ offsets,
                           const int32_t* __restrict__ n_kept) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l < k && keep[l]) offsets[new_id[l]] = start[l];
  if (l == k - 1) {
    const int32_t m = *n_kept;
    offsets[m] = start[l] + (keep[l] ? count[l] : 0);
  }
}
__global__ void ex_nkept(int64_t k, const int32_t* __restrict__ keep,
                         const int32_t* __restrict__ new_id, int32_t* __restrict__ n_kept) {
  *n_kept = k > 0 ? new_id[k - 1] + keep[k - 1] : 0;
}
__global__ void ex_count_reps(int64_t n, const int32_t* __restrict__ rep,
                              const int32_t* __restrict__ rank, int32_t* __restrict__ k) {
  *k = n > 0 ? rank[n - 1] + rep[n - 1] : 0;
}

__global__ void gather_kernel(int64_t p, const int32_t* __restrict__ pi,
                              const double* __restrict__ az, const double* __restrict__ dop,
                              double* __restrict__ gaz, double* __restrict__ gdop) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= p) return;
  const int32_t i = pi[k];
  gaz[k] = az[i];
  gdop[k] = dop[i];
}

// ---- combine_masks (src/ransac.cpp:217-242)
__global__ void cm_keys(int64_t n, const int32_t* __restrict__ labels, uint32_t* __restrict__ key,
                        int32_t* __restrict__ idx) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t l = labels[i];
  key[i] = l >= 0 ? static_cast<uint32_t>(l) : 0xFFFFFFFFu;
  idx[i] = static_cast<int32_t>(i);
}
// run starts of the sorted labels: s where the label changes, else 0 (max-scanned)
__global__ void cm_bounds(int64_t n, const uint32_t* __restrict__ skey, int32_t* __restrict__ b) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  b[s] = (s == 0 || skey[s - 1] != skey[s]) ? static_cast<int32_t>(s) : 0;
}
// Point sidx[s]: position within its label = s - run start; its mask = the
// first mask whose cluster_id equals the label (ids sorted on the host with
// the lowest mask index first, as unordered_map::emplace keeps the first).
__global__ void cm_apply(int64_t n, const uint32_t* __restrict__ skey,
                         const int32_t* __restrict__ sidx, const int32_t* __restrict__ run,
                         int32_t n_masks, const int32_t* __restrict__ ids_sorted,
                         const int32_t* __restrict__ mask_of, const int64_t* __restrict__ moff,
                         const uint8_t* __restrict__ masks, uint8_t* __restrict__ result) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const uint32_t k = skey[s];
  uint8_t v = 0;
  if (k != 0xFFFFFFFFu) {
    const int32_t label = static_cast<int32_t>(k);
    int lo = 0, hi = n_masks;  // first id >= label
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (ids_sorted[mid] < label) lo = mid + 1;
      else hi = mid;
    }
    if (lo < n_masks && ids_sorted[lo] == label) {
      const int32_t m = mask_of[lo];
      const int64_t pos = s - run[s];
      if (pos < moff[m + 1] - moff[m]) v = masks[moff[m] + pos];
    }
  }
  result[sidx[s]] = v;
}

unsigned blocks(int64_t n) { return static_cast<unsigned>((n + kDbThreads - 1) / kDbThreads); }

}  // namespace

void launch_combine_masks(int64_t n, const int32_t* labels, int32_t n_masks,
                          const int32_t* ids_sorted, const int32_t* mask_of,
                          const int64_t* moff, const uint8_t* masks, const DbscanLayout& L,
                          char* ws, uint8_t* result, cudaStream_t st) {
  if (n <= 0) return;
  auto P = [&](size_t o) { return ws + o; };
  uint32_t* key = reinterpret_cast<uint32_t*>(P(L.o_keys));
  int32_t* idx = reinterpret_cast<int32_t*>(P(L.o_idx));
  uint32_t* skey = reinterpret_cast<uint32_t*>(P(L.o_skeys));
  int32_t* sidx = reinterpret_cast<int32_t*>(P(L.o_sidx));
  int32_t* bnd = reinterpret_cast<int32_t*>(P(L.o_rep));
  int32_t* run = reinterpret_cast<int32_t*>(P(L.o_rank));
  void* cub_tmp = P(L.o_cub);
  cm_keys<<<blocks(n), kDbThreads, 0, st>>>(n, labels, key, idx);
  count_launch();
  size_t cb = L.cub_bytes;
  cub::DeviceRadixSort::SortPairs(cub_tmp, cb, key, skey, idx, sidx, static_cast<int>(n), 0, 32,
                                  st);
  cm_bounds<<<blocks(n), kDbThreads, 0, st>>>(n, skey, bnd);
  count_launch();
  cb = L.cub_bytes;
  cub::DeviceScan::InclusiveScan(cub_tmp, cb, bnd, run, cub::Max(), static_cast<int>(n), st);
  cm_apply<<<blocks(n), kDbThreads, 0, st>>>(n, skey, sidx, run, n_masks, ids_sorted, mask_of,
                                             moff, masks, result);
  count_launch();
}

void launch_gather(int64_t p, const int32_t* point_indices, const double* az, const double* dop,
                   double* gaz, double* gdop, cudaStream_t st) {
  if (p <= 0) return;
  gather_kernel<<<blocks(p), kDbThreads, 0, st>>>(p, point_indices, az, dop, gaz, gdop);
  count_launch();
}

// Scratch layout of one dbscan/extract call (carved from one allocation).
DbscanLayout dbscan_layout(int64_t n, bool xyz) {
  DbscanLayout L;
  int bits = 4;
  while ((int64_t{1} << bits) < 2 * n && bits < 30) ++bits;
  L.table_bits = bits;
  const size_t T = size_t{1} << bits;
  size_t cub_bytes = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr),
                                  static_cast<const int32_t*>(nullptr),
                                  static_cast<int32_t*>(nullptr), static_cast<int>(n));
  cub_bytes = b > cub_bytes ? b : cub_bytes;
  b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<const int32_t*>(nullptr),
                                static_cast<int32_t*>(nullptr), static_cast<int>(n));
  cub_bytes = b > cub_bytes ? b : cub_bytes;
  b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<const int32_t*>(nullptr),
                                static_cast<int64_t*>(nullptr), static_cast<int>(n));
  cub_bytes = b > cub_bytes ? b : cub_bytes;
  b = 0;
  cub::DeviceScan::InclusiveScan(nullptr, b, static_cast<const int32_t*>(nullptr),
                                 static_cast<int32_t*>(nullptr), cub::Max(), static_cast<int>(n));
  cub_bytes = b > cub_bytes ? b : cub_bytes;
  auto take = [&](size_t bytes) {
    const size_t o = L.total;
    L.total += (bytes + 255) / 256 * 256;
    return o;
  };
  const size_t N = static_cast<size_t>(n > 0 ? n : 1);
  L.o_keys = take(4 * N);
  L.o_idx = take(4 * N);
  L.o_skeys = take(4 * N);
  L.o_sidx = take(4 * N);
  L.o_sx = take(8 * N);
  L.o_sy = take(8 * N);
  L.o_sz = take(xyz ? 8 * N : 8);
  L.o_cstart = take(4 * T);
  L.o_cend = take(4 * T);
  L.o_core = take(N);
  L.o_parent = take(4 * N);
  L.o_root = take(4 * N);
  L.o_rep = take(4 * N);
  L.o_rank = take(4 * N);
  L.o_count = take(4 * N);
  L.o_keep = take(4 * N);
  L.o_kept = take(4 * N);
  L.o_start = take(8 * N);
  L.o_small = take(64);
  L.o_cub = take(cub_bytes);
  L.cub_bytes = cub_bytes;
  return L;
}

void launch_dbscan(int64_t n, const double* x, const double* y, const double* z, double eps,
                   int min_pts, const DbscanLayout& L, char* ws, int32_t* labels,
                   cudaStream_t st) {
  if (n <= 0) return;
  const bool xyz = z != nullptr;
  const uint32_t mask = (1u << L.table_bits) - 1u;
  const double cs = eps * kCellMargin;
  const double inv_cs = 1.0 / cs;
  const double eps2 = eps * eps;  // clustering.cpp:37
  auto P = [&](size_t o) { return ws + o; };
  uint32_t* keys = reinterpret_cast<uint32_t*>(P(L.o_keys));
  int32_t* idx = reinterpret_cast<int32_t*>(P(L.o_idx));
  uint32_t* skeys = reinterpret_cast<uint32_t*>(P(L.o_skeys));
  int32_t* sidx = reinterpret_cast<int32_t*>(P(L.o_sidx));
  double* sx = reinterpret_cast<double*>(P(L.o_sx));
  double* sy = reinterpret_cast<double*>(P(L.o_sy));
  double* sz = xyz ? reinterpret_cast<double*>(P(L.o_sz)) : nullptr;
  int32_t* cstart = reinterpret_cast<int32_t*>(P(L.o_cstart));
  int32_t* cend = reinterpret_cast<int32_t*>(P(L.o_cend));
  uint8_t* core = reinterpret_cast<uint8_t*>(P(L.o_core));
  int32_t* parent = reinterpret_cast<int32_t*>(P(L.o_parent));
  int32_t* root = reinterpret_cast<int32_t*>(P(L.o_root));
  int32_t* rep = reinterpret_cast<int32_t*>(P(L.o_rep));
  int32_t* rank = reinterpret_cast<int32_t*>(P(L.o_rank));
  void* cub_tmp = P(L.o_cub);
  const size_t T = size_t{1} << L.table_bits;

  db_keys<<<blocks(n), kDbThreads, 0, st>>>(n, x, y, z, inv_cs, mask, keys, idx);
  count_launch();
  size_t cb = L.cub_bytes;
  cub::DeviceRadixSort::SortPairs(cub_tmp, cb, keys, skeys, idx, sidx, static_cast<int>(n), 0,
                                  L.table_bits, st);
  cudaMemsetAsync(cstart, 0, 4 * T, st);
  cudaMemsetAsync(cend, 0, 4 * T, st);
  db_cells<<<blocks(n), kDbThreads, 0, st>>>(n, skeys, sidx, x, y, z, cstart, cend, sx, sy, sz);
  count_launch();
  const Pts p{sx, sy, sz, xyz};
  db_core<<<blocks(n), kDbThreads, 0, st>>>(n, p, inv_cs, mask, eps2, min_pts, cstart, cend, core);
  count_launch();
  db_parent_init<<<blocks(n), kDbThreads, 0, st>>>(n, sidx, core, parent);
  count_launch();
  db_hook<<<blocks(n), kDbThreads, 0, st>>>(n, p, inv_cs, mask, eps2, cstart, cend, sidx, core,
                                            parent);
  count_launch();
  db_compress<<<blocks(n), kDbThreads, 0, st>>>(n, parent);
  count_launch();
  db_union<<<blocks(n), kDbThreads, 0, st>>>(n, p, inv_cs, mask, eps2, cstart, cend, sidx, core,
                                             parent);
  count_launch();
  db_roots<<<blocks(n), kDbThreads, 0, st>>>(n, parent, rep);
  count_launch();
  db_flatten<<<blocks(n), kDbThreads, 0, st>>>(n, parent, root);
  count_launch();
  cb = L.cub_bytes;
  cub::DeviceScan::ExclusiveSum(cub_tmp, cb, rep, rank, static_cast<int>(n), st);
  db_label_core<<<blocks(n), kDbThreads, 0, st>>>(n, root, rank, labels);
  count_launch();
  db_border<<<blocks(n), kDbThreads, 0, st>>>(n, p, inv_cs, mask, eps2, cstart, cend, sidx, core,
                                              labels);
  count_launch();
  // number of clusters (max label + 1) for extract_clusters
  int32_t* small = reinterpret_cast<int32_t*>(P(L.o_small));
  ex_count_reps<<<1, 1, 0, st>>>(n, rep, rank, small);
  count_launch();
}

void launch_extract(int64_t n, int32_t* labels, int32_t n_labels_max, int min_size,
                    const DbscanLayout& L, char* ws, int64_t* offsets, int32_t* point_indices,
                    int32_t* d_n_clusters, cudaStream_t st) {
  auto P = [&](size_t o) { return ws + o; };
  int32_t* count = reinterpret_cast<int32_t*>(P(L.o_count));
  int32_t* keep = reinterpret_cast<int32_t*>(P(L.o_keep));
  int32_t* kept = reinterpret_cast<int32_t*>(P(L.o_kept));
  int32_t* new_id = reinterpret_cast<int32_t*>(P(L.o_rank));
  int64_t* start = reinterpret_cast<int64_t*>(P(L.o_start));
  uint32_t* key = reinterpret_cast<uint32_t*>(P(L.o_keys));
  int32_t* idx = reinterpret_cast<int32_t*>(P(L.o_idx));
  uint32_t* skey = reinterpret_cast<uint32_t*>(P(L.o_skeys));
  void* cub_tmp = P(L.o_cub);
  const int64_t k = n_labels_max;  // labels are < k
  if (n <= 0 || k <= 0) {
    cudaMemsetAsync(d_n_clusters, 0, 4, st);
    cudaMemsetAsync(offsets, 0, 8, st);
    return;
  }
  cudaMemsetAsync(count, 0, 4 * static_cast<size_t>(k), st);
  ex_count<<<blocks(n), kDbThreads, 0, st>>>(n, labels, count);
  count_launch();
  ex_keep<<<blocks(k), kDbThreads, 0, st>>>(k, count, min_size, keep, kept);
  count_launch();
  size_t cb = L.cub_bytes;
  cub::DeviceScan::ExclusiveSum(cub_tmp, cb, keep, new_id, static_cast<int>(k), st);
  cb = L.cub_bytes;
  cub::DeviceScan::ExclusiveSum(cub_tmp, cb, kept, start, static_cast<int>(k), st);
  ex_nkept<<<1, 1, 0, st>>>(k, keep, new_id, d_n_clusters);
  count_launch();
  ex_offsets<<<blocks(k), kDbThreads, 0, st>>>(k, keep, new_id, start, count, offsets,
                                               d_n_clusters);
  count_launch();
  ex_remap<<<blocks(n), kDbThreads, 0, st>>>(n, labels, keep, new_id, key, idx);
  count_launch();
  cb = L.cub_bytes;
  // stable: members stay in ascending point order within each cluster
  cub::DeviceRadixSort::SortPairs(cub_tmp, cb, key, skey, idx, point_indices, static_cast<int>(n),
                                  0, 32, st);
}

}  // namespace rvk_gpu
