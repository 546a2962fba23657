// Dev check: the beta = 1 latency AQIF (csrc/aqif1.cuh) against the general
// warp engine (aqif_factor_group + zsolve_group with BETA = 1): bit-identical
// solutions / breakdown flags in EXACT mode, plus cycle counts.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        tools/aqif1_check.cu -o /tmp/aqif1_check && /tmp/aqif1_check 512 64
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>
#include "../paper_2008_03276_b200/csrc/aqif_warp.cuh"
#include "../paper_2008_03276_b200/csrc/zsolve.cuh"
#include "../paper_2008_03276_b200/csrc/aqif1.cuh"

using namespace paqif;
constexpr int kB = 1;

struct Pol1 {
  static constexpr bool kFuseW = true;
  static constexpr bool kResidual = false;
  static constexpr bool kFastDiv = false;
  static constexpr bool kLazyBreakdown = false;
  static constexpr bool kRecordW = false;
  using PL = PivotLayout<kB>;
  const double* band;
  const double* rhs;
  double* zs;
  int n;
  __device__ __forceinline__ const double* raw_ptr(int i, int d) const {
    return band + (size_t)(d + kB) * n + i;
  }
  __device__ __forceinline__ double raw(int i, int d) const { return *raw_ptr(i, d); }
  __device__ __forceinline__ const uint32_t* pin_ptr(int) const { return nullptr; }
  __device__ __forceinline__ bool pinned(int) const { return false; }
  __device__ __forceinline__ const double* frhs_ptr(int i) const { return rhs + i; }
  __device__ __forceinline__ double frhs(int i) const { return rhs[i]; }
  __device__ __forceinline__ void on_level(int k, const double* pb, int gl, int G) {
    for (int idx = gl; idx < PL::kSize; idx += G) zs[(size_t)k * PL::kSize + idx] = pb[idx];
  }
  __device__ __forceinline__ void on_w(int, int, double, double) {}
  __device__ __forceinline__ void on_resid(int, int, double) {}
};

__host__ __device__ inline size_t scr_doubles(int n) {
  return 3 * (size_t)n + 2 * (size_t)n + (size_t)(n / 2 + 1) * PivotLayout<kB>::kSize + 32;
}

template <bool EXACT>
__global__ void engine_kernel(const double* bands, const double* rhss, int n, double* scratch_all,
                              double* x_out, int* st_out, long long* cyc) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  double* band = scratch_all + (size_t)b * scr_doubles(n);
  double* rhs = band + 3 * (size_t)n;
  double* x = rhs + n;
  double* zs = x + n;
  for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) band[i] = bands[(size_t)b * 3 * n + i];
  for (int i = threadIdx.x; i < n; i += blockDim.x) rhs[i] = rhss[(size_t)b * n + i];
  __syncthreads();
  EngineSmem<kB>& eng = *reinterpret_cast<EngineSmem<kB>*>(sm);
  double* ring = sm + sizeof(EngineSmem<kB>) / 8;
  __shared__ int flag;
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    constexpr int G = Group<kB>::G;
    const int lane = threadIdx.x;
    const bool alive = lane < G;
    Pol1 pol{band, rhs, zs, n};
    int fst = aqif_factor_group<kB, EXACT>(pol, n, 1e-14, eng, lane % G, alive);
    fst = __shfl_sync(0xffffffffu, fst, 0);
    int zst = 0;
    if (fst == 0) {
      zst = zsolve_group<kB, EXACT, true>(zs, n, x, ring, lane % G, alive);
      zst = __shfl_sync(0xffffffffu, zst, 0);
    }
    if (lane == 0) flag = (fst || zst) ? 1 : 0;
  }
  __syncthreads();
  long long t1 = clock64();
  for (int i = threadIdx.x; i < n; i += blockDim.x) x_out[(size_t)b * n + i] = x[i];
  if (threadIdx.x == 0) { st_out[b] = flag; cyc[b] = t1 - t0; }
}

template <bool EXACT>
__global__ void aqif1_kernel(const double* bands, const double* rhss, int n, double* x_out,
                             int* st_out, long long* cyc) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  double* band = sm;
  double* rhs = band + aqif1_band_doubles(n);
  double* rec = rhs + aqif1_rhs_doubles(n);
  __shared__ int flag;
  aqif1_zero_pads(band, rhs, n);
  for (int i = threadIdx.x; i < 3 * n; i += blockDim.x)
    band1_ref(band, n, i % n, i / n - 1) = bands[(size_t)b * 3 * n + i];
  for (int i = threadIdx.x; i < n; i += blockDim.x) rhs[kBandPad + i] = rhss[(size_t)b * n + i];
  __syncthreads();
  long long t0 = clock64();
  const int st = aqif1_solve<EXACT>(band, rhs, n, rec, band, &flag);
  long long t1 = clock64();
  for (int i = threadIdx.x; i < n; i += blockDim.x) x_out[(size_t)b * n + i] = band[i];
  if (threadIdx.x == 0) { st_out[b] = st & 1; cyc[b] = t1 - t0; }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 512;
  const int B = argc > 2 ? atoi(argv[2]) : 64;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-1, 1), U2(0.05, 1);
  std::vector<double> bands((size_t)B * 3 * n, 0.0), rhs((size_t)B * n);
  for (int b = 0; b < B; ++b) {
    double* bd = &bands[(size_t)b * 3 * n];
    const int kind = b % 4;  // 0 dominant, 1 weakly dominant, 2 wild, 3 near-singular
    for (int i = 0; i < n; ++i) {
      double sum = 0;
      for (int d = -1; d <= 1; d += 2) {
        const int j = i + d;
        if (j < 0 || j >= n) continue;
        const double v = U(rng) * (kind == 2 ? 10.0 : 1.0);
        bd[(d + 1) * n + i] = v;
        sum += fabs(v);
      }
      double diag = kind == 0 ? sum + U2(rng) : kind == 1 ? 0.5 * sum + U2(rng) : U(rng);
      if (kind == 3 && i == n / 2 + 7) diag = 0.0;
      bd[n + i] = diag;
      rhs[(size_t)b * n + i] = U(rng);
    }
    if (b % 8 == 5)  // tiny entries: checked redo
      for (int i = 0; i < 3 * n; ++i) bd[i] = ldexp(bd[i], -600);
    if (b % 8 == 6)  // decaying fill through the subnormal range
      for (int i = 0; i < n; ++i) { bd[i] *= 1e-3; bd[2 * n + i] *= 1e-3; }
    if (kind == 3) {
      const int h = n / 2;
      if ((b / 4) % 3 == 0) {  // singular middle block
        bd[n + h - 1] = 1.0; bd[2 * n + h - 1] = 2.0; bd[h] = 2.0; bd[n + h] = 4.0;
      } else if ((b / 4) % 3 == 1) {  // last row zero
        for (int d = -1; d <= 1; ++d) bd[(d + 1) * n + n - 1] = 0.0;
      } else {
        const int r = h - 4;
        for (int d = -1; d <= 1; ++d) bd[(d + 1) * n + r] = 0.0;
      }
    }
  }
  double *db, *dr, *dx1, *dx2, *scr; int *s1, *s2; long long *c1, *c2;
  cudaMalloc(&db, bands.size() * 8); cudaMalloc(&dr, rhs.size() * 8);
  cudaMalloc(&dx1, rhs.size() * 8); cudaMalloc(&dx2, rhs.size() * 8);
  cudaMalloc(&scr, (size_t)B * scr_doubles(n) * 8);
  cudaMalloc(&s1, B * 4); cudaMalloc(&s2, B * 4); cudaMalloc(&c1, B * 8); cudaMalloc(&c2, B * 8);
  cudaMemcpy(db, bands.data(), bands.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, rhs.data(), rhs.size() * 8, cudaMemcpyHostToDevice);
  const size_t sm1 = sizeof(EngineSmem<kB>) + ZChunk<kB>::kRing * 8 + 64;
  const size_t sm2 = (aqif1_band_doubles(n) + aqif1_rhs_doubles(n) + aqif1_rec_doubles(n)) * 8;
  cudaFuncSetAttribute(aqif1_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  cudaFuncSetAttribute(aqif1_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  int total_bad = 0;
  for (int exact = 1; exact >= 0; --exact) {
    for (int rep = 0; rep < 2; ++rep) {
      if (exact) {
        engine_kernel<true><<<B, 256, sm1>>>(db, dr, n, scr, dx1, s1, c1);
        aqif1_kernel<true><<<B, 256, sm2>>>(db, dr, n, dx2, s2, c2);
      } else {
        engine_kernel<false><<<B, 256, sm1>>>(db, dr, n, scr, dx1, s1, c1);
        aqif1_kernel<false><<<B, 256, sm2>>>(db, dr, n, dx2, s2, c2);
      }
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<double> x1(rhs.size()), x2(rhs.size());
    std::vector<int> t1(B), t2(B); std::vector<long long> k1(B), k2(B);
    cudaMemcpy(x1.data(), dx1, x1.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(x2.data(), dx2, x2.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(t1.data(), s1, B * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(t2.data(), s2, B * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(k1.data(), c1, B * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(k2.data(), c2, B * 8, cudaMemcpyDeviceToHost);
    int mism = 0, stm = 0, fails = 0; double maxrel = 0;
    for (int b = 0; b < B; ++b) {
      if ((t1[b] != 0) != (t2[b] != 0)) ++stm;
      if (t1[b]) { ++fails; continue; }
      for (int i = 0; i < n; ++i) {
        const double a = x1[(size_t)b * n + i], c = x2[(size_t)b * n + i];
        if (memcmp(&a, &c, 8) != 0 && !(a == 0.0 && c == 0.0)) {
          ++mism;
          maxrel = fmax(maxrel, fabs(a - c) / fmax(1e-300, fabs(a)));
        }
      }
    }
    double ce = 0, ca = 0;
    for (int b = 0; b < B; ++b) { ce += k1[b]; ca += k2[b]; }
    printf("n=%d exact=%d: status mismatches %d (engine breakdowns %d), x mismatches %d (max rel %.3g)"
           " | cycles/solve engine %.0f aqif1 %.0f\n", n, exact, stm, fails, mism, maxrel, ce / B, ca / B);
    if (exact) total_bad += stm + mism;
  }
  return total_bad ? 2 : 0;
}
