// tcgen05 kind::tf32 probe (development tool, not shipped): one M=128 x N=256
// x K=8 MMA per CTA with the split-operand layout the scoring kernel uses,
//   hyp row  h: [A1, A1, A2, B1, B1, B2, C1, C2]
//   point    p: [x1, x2, x1, y1, y2, y1, 1, 1]
// so D[h][p] = A x + B y + C to ~2^-22 relative. Checks the smem descriptor
// layout (K-major, no swizzle: 8x16 B core matrices, LBO = K-chunk stride,
// SBO = 8-row-group stride) against an FP64 host reference and reports the
// largest |D - exact| / S (S = |A| + |B| + |C|) over many random tiles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_probe tools/tc_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

constexpr int M = 128, N = 256, K = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// core-matrix offset (bytes) of element (row, k) in a K-major no-swizzle tile
__host__ __device__ inline int kmaj_off(int row, int k) {
  return (row >> 3) * 256 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(128 >> 4) << 16;  // LBO: next 16 B K-chunk
  d |= static_cast<uint64_t>(256 >> 4) << 32;  // SBO: next 8-row group
  d |= static_cast<uint64_t>(1) << 46;         // version (sm100)
  return d;                                    // base offset 0, SWIZZLE_NONE
}

__global__ void __launch_bounds__(128) tc_kernel(const float* __restrict__ A_g,
                                                 const float* __restrict__ B_g,
                                                 float* __restrict__ D_g, int n_cols) {
  __shared__ __align__(1024) float sA[M * K];
  __shared__ __align__(1024) float sB[N * K];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const float* Ab = A_g + static_cast<size_t>(blockIdx.x) * M * K;
  const float* Bb = B_g + static_cast<size_t>(blockIdx.x) * N * K;
  // global arrays are already in the core-matrix byte layout
  for (int i = tid; i < M * K; i += blockDim.x) sA[i] = Ab[i];
  for (int i = tid; i < N * K; i += blockDim.x) sB[i] = Bb[i];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint64_t da = desc_kmajor(smem_u32(sA));
    const uint64_t db = desc_kmajor(smem_u32(sB));
    // kind::tf32: D f32 (bit 4), A tf32 (2 << 7), B tf32 (2 << 10), K-major
    // both, N >> 3 at bit 17, M >> 4 at bit 24
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                           (static_cast<uint32_t>(n_cols >> 3) << 17) | ((M >> 4) << 24);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  // wait for the MMA
  asm volatile(
      "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
          smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < n_cols; c0 += 8) {
    uint32_t r[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "r"(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j)
      D_g[(static_cast<size_t>(blockIdx.x) * M + row) * N + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// round-to-nearest (ties away) to tf32, the value keeps 10 explicit mantissa bits
static float tf32_rna(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}
static void split(double v, float& hi, float& lo) {
  hi = tf32_rna(static_cast<float>(v));
  lo = tf32_rna(static_cast<float>(v - static_cast<double>(hi)));
}

int main(int argc, char** argv) {
  const int tiles = argc > 1 ? atoi(argv[1]) : 512;
  std::mt19937_64 rng(12345);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<float> A(static_cast<size_t>(tiles) * M * K), B(static_cast<size_t>(tiles) * N * K);
  std::vector<double> hA(static_cast<size_t>(tiles) * M * 3), hP(static_cast<size_t>(tiles) * N * 2);
  for (int t = 0; t < tiles; ++t) {
    for (int h = 0; h < M; ++h) {
      // a line through two random points of the unit square, normalized
      const double xa = U(rng), ya = U(rng), xb = U(rng), yb = U(rng);
      const double dx = (xb - xa) == 0 ? 1e-3 : xb - xa;
      const double m = (yb - ya) / dx * (h % 7 == 0 ? 100.0 : 1.0), c = ya - m * xa;
      const double den = std::sqrt(m * m + 1);
      const double a = -m / den, b = 1 / den, cc = -c / den;
      double* H = &hA[(static_cast<size_t>(t) * M + h) * 3];
      H[0] = a, H[1] = b, H[2] = cc;
      float a1, a2, b1, b2, c1, c2;
      split(a, a1, a2), split(b, b1, b2), split(cc, c1, c2);
      const float row[8] = {a1, a1, a2, b1, b1, b2, c1, c2};
      float* At = &A[static_cast<size_t>(t) * M * K];
      for (int k = 0; k < 8; ++k) At[kmaj_off(h, k) / 4] = row[k];
    }
    for (int p = 0; p < N; ++p) {
      const double x = U(rng), y = U(rng);
      double* Pp = &hP[(static_cast<size_t>(t) * N + p) * 2];
      Pp[0] = x, Pp[1] = y;
      float x1, x2, y1, y2;
      split(x, x1, x2), split(y, y1, y2);
      const float row[8] = {x1, x2, x1, y1, y2, y1, 1.f, 1.f};
      float* Bt = &B[static_cast<size_t>(t) * N * K];
      for (int k = 0; k < 8; ++k) Bt[kmaj_off(p, k) / 4] = row[k];
    }
  }
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dD, static_cast<size_t>(tiles) * M * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  tc_kernel<<<tiles, 128>>>(dA, dB, dD, N);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> D(static_cast<size_t>(tiles) * M * N);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  double worst = 0, worst_abs = 0;
  long bad = 0;
  for (int t = 0; t < tiles; ++t)
    for (int h = 0; h < M; ++h) {
      const double* H = &hA[(static_cast<size_t>(t) * M + h) * 3];
      const double S = std::fabs(H[0]) + std::fabs(H[1]) + std::fabs(H[2]);
      for (int p = 0; p < N; ++p) {
        const double* Pp = &hP[(static_cast<size_t>(t) * N + p) * 2];
        const double ex = H[0] * Pp[0] + H[1] * Pp[1] + H[2];
        const double got = D[(static_cast<size_t>(t) * M + h) * N + p];
        const double err = std::fabs(got - ex);
        worst_abs = std::max(worst_abs, err);
        worst = std::max(worst, err / S);
        if (err > 1e-3 * S) ++bad;
      }
    }
  printf("tiles=%d evals=%ld max|D-exact|/S = %.3e (= 2^%.2f), max abs %.3e, gross errors %ld\n",
         tiles, static_cast<long>(tiles) * M * N, worst, std::log2(worst), worst_abs, bad);
  // print one sample for layout debugging
  {
    const double* H = &hA[0];
    const double* Pp = &hP[0];
    printf("sample D[0][0]=%.9g exact=%.9g  D[1][0]=%.9g  D[0][1]=%.9g\n", D[0],
           H[0] * Pp[0] + H[1] * Pp[1] + H[2], D[N], D[1]);
  }
  return bad ? 2 : 0;
}
