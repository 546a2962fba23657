// Dev check: the two-lane beta=2 AQIF (csrc/aqif2.cuh) against the general
// warp engine (aqif_factor_group + zsolve_group via solve_line_system):
// bit-identical solutions / breakdown levels in EXACT mode, and per-solve
// cycle counts of both.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//        tools/aqif2_check.cu -o /tmp/aqif2_check
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>
#include "../paper_2008_03276_b200/csrc/ehl_solve.cuh"
#include "../paper_2008_03276_b200/csrc/aqif2.cuh"

using namespace paqif;

template <bool EXACT>
__global__ void engine_kernel(const double* bands, const double* rhss, int n, double* scratch_all,
                              double* x_out, int* st_out, long long* cyc) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  double* scratch = scratch_all + (size_t)b * line_scratch_doubles(n);
  for (int i = threadIdx.x; i < 5 * n; i += blockDim.x) scratch[i] = bands[(size_t)b * 5 * n + i];
  for (int i = threadIdx.x; i < n; i += blockDim.x) scratch[5 * n + i] = rhss[(size_t)b * n + i];
  __syncthreads();
  EngineSmem<2>& eng = *reinterpret_cast<EngineSmem<2>*>(sm);
  double* ring = sm + sizeof(EngineSmem<2>) / 8;
  int* flag = reinterpret_cast<int*>(ring + ZChunk<2>::kRing);
  long long t0 = clock64();
  int st = solve_line_system<EXACT>(scratch, n, eng, ring, flag);
  long long t1 = clock64();
  const double* x = line_solution(scratch, n);
  for (int i = threadIdx.x; i < n; i += blockDim.x) x_out[(size_t)b * n + i] = x[i];
  if (threadIdx.x == 0) { st_out[b] = st; cyc[b] = t1 - t0; }
}

template <bool EXACT>
__global__ void aqif2_kernel(const double* bands, const double* rhss, int n, double* x_out,
                             int* st_out, long long* cyc) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  double* band = sm;
  double* rhs = band + aqif2_band_doubles(n);
  double* x = rhs + aqif2_rhs_doubles(n);
  double* rec = x + n;
  __shared__ int flag;
  aqif2_zero_pads(band, rhs, n);
  for (int i = threadIdx.x; i < 5 * n; i += blockDim.x)
    band2_ref(band, n, i % n, i / n - 2) = bands[(size_t)b * 5 * n + i];
  for (int i = threadIdx.x; i < n; i += blockDim.x) rhs[kBandPad + i] = rhss[(size_t)b * n + i];
  __syncthreads();
  long long t0 = clock64(), t1 = 0, t2 = 0;
  if (threadIdx.x < 32) {
    bool ok = aqif2_factor<EXACT, false>(band, rhs, n, rec, threadIdx.x);
    __syncwarp();
    t1 = clock64();
    bool bad = aqif2_breakdown(rec, n, 1e-14, threadIdx.x);
    ok = aqif2_zsolve<EXACT, false>(rec, n, threadIdx.x) && ok;
    if (!ok) {
      aqif2_factor<EXACT, true>(band, rhs, n, rec, threadIdx.x);
      __syncwarp();
      bad = aqif2_breakdown(rec, n, 1e-14, threadIdx.x);
      aqif2_zsolve<EXACT, true>(rec, n, threadIdx.x);
    }
    __syncwarp();
    aqif2_gather(rec, n, band, threadIdx.x);  // x over the band, as the EHL kernels do
    __syncwarp();
    for (int i = threadIdx.x; i < n; i += 32) x[i] = band[i];
    if (threadIdx.x == 0) flag = bad ? 1 : 0;
    t2 = clock64();
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) x_out[(size_t)b * n + i] = x[i];
  if (threadIdx.x == 0) { st_out[b] = flag; cyc[2 * b] = t1 - t0; cyc[2 * b + 1] = t2 - t1; }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 512;
  const int B = argc > 2 ? atoi(argv[2]) : 64;
  std::mt19937_64 rng(11);
  std::uniform_real_distribution<double> U(-1, 1), U2(0.05, 1);
  std::vector<double> bands((size_t)B * 5 * n, 0.0), rhs((size_t)B * n);
  for (int b = 0; b < B; ++b) {
    double* bd = &bands[(size_t)b * 5 * n];
    const int kind = b % 4;  // 0 dominant, 1 weakly dominant, 2 nonsymmetric wild, 3 near-singular
    for (int i = 0; i < n; ++i) {
      double sum = 0;
      for (int d = -2; d <= 2; ++d) {
        if (d == 0) continue;
        const int j = i + d;
        if (j < 0 || j >= n) continue;
        double v = U(rng) * (kind == 2 ? 10.0 : 1.0);
        bd[(d + 2) * n + i] = v;
        sum += fabs(v);
      }
      double diag = kind == 0 ? sum + U2(rng) : kind == 1 ? 0.5 * sum + U2(rng) : U(rng);
      if (kind == 3 && i == n / 2 + 7) diag = 0.0;
      bd[2 * n + i] = diag;
      rhs[(size_t)b * n + i] = U(rng);
    }
    if (b % 8 == 5) {  // tiny entries: divisions leave the Markstein range (checked redo)
      for (int i = 0; i < 5 * n; ++i) bd[i] = ldexp(bd[i], -600);
    }
    if (kind == 3) {
      const int h = n / 2;
      if ((b / 4) % 3 == 0) {  // singular middle 2x2 block: breakdown at level 1
        bd[2 * n + h - 1] = 1.0; bd[3 * n + h - 1] = 2.0; bd[1 * n + h] = 2.0; bd[2 * n + h] = 4.0;
      } else if ((b / 4) % 3 == 1) {  // last row zero: only the Z solve's level s breaks
        for (int d = -2; d <= 2; ++d) bd[(d + 2) * n + n - 1] = 0.0;
      } else {  // exact cancellation a few levels out
        const int r = h - 4;
        for (int d = -2; d <= 2; ++d) bd[(d + 2) * n + r] = 0.0;
      }
    }
  }
  double *db, *dr, *dx1, *dx2, *scr; int *s1, *s2; long long *c1, *c2;
  cudaMalloc(&db, bands.size() * 8); cudaMalloc(&dr, rhs.size() * 8);
  cudaMalloc(&dx1, rhs.size() * 8); cudaMalloc(&dx2, rhs.size() * 8);
  cudaMalloc(&scr, (size_t)B * line_scratch_doubles(n) * 8);
  cudaMalloc(&s1, B * 4); cudaMalloc(&s2, B * 4); cudaMalloc(&c1, B * 8); cudaMalloc(&c2, 2 * B * 8);
  cudaMemcpy(db, bands.data(), bands.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, rhs.data(), rhs.size() * 8, cudaMemcpyHostToDevice);
  size_t sm1 = sizeof(EngineSmem<2>) + ZChunk<2>::kRing * 8 + 64;
  size_t sm2 = (aqif2_band_doubles(n) + aqif2_rhs_doubles(n) + n + (size_t)(n / 2 + 1) * kRec2) * 8;
  cudaFuncSetAttribute(aqif2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  cudaFuncSetAttribute(aqif2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  for (int exact = 1; exact >= 0; --exact) {
    for (int rep = 0; rep < 2; ++rep) {
      if (exact) {
        engine_kernel<true><<<B, 256, sm1>>>(db, dr, n, scr, dx1, s1, c1);
        aqif2_kernel<true><<<B, 256, sm2>>>(db, dr, n, dx2, s2, c2);
      } else {
        engine_kernel<false><<<B, 256, sm1>>>(db, dr, n, scr, dx1, s1, c1);
        aqif2_kernel<false><<<B, 256, sm2>>>(db, dr, n, dx2, s2, c2);
      }
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<double> x1(rhs.size()), x2(rhs.size());
    std::vector<int> t1(B), t2(B); std::vector<long long> k1(B), k2(2 * B);
    cudaMemcpy(x1.data(), dx1, x1.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(x2.data(), dx2, x2.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(t1.data(), s1, B * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(t2.data(), s2, B * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(k1.data(), c1, B * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(k2.data(), c2, 2 * B * 8, cudaMemcpyDeviceToHost);
    int mism = 0, stm = 0, fails = 0; double maxrel = 0;
    for (int b = 0; b < B; ++b) {
      if ((t1[b] != 0) != (t2[b] != 0)) ++stm;
      if (t1[b]) { ++fails; continue; }
      for (int i = 0; i < n - 1; ++i) {
        const double a = x1[(size_t)b * n + i], c = x2[(size_t)b * n + i];
        if (memcmp(&a, &c, 8) != 0) {
          ++mism;
          maxrel = fmax(maxrel, fabs(a - c) / fmax(1e-300, fabs(a)));
        }
      }
    }
    double ce = 0, cf = 0, cz = 0;
    for (int b = 0; b < B; ++b) { ce += k1[b]; cf += k2[2 * b]; cz += k2[2 * b + 1]; }
    printf("n=%d exact=%d: status mismatches %d (engine breakdowns %d), x mismatches %d (max rel %.3g)\n",
           n, exact, stm, fails, mism, maxrel);
    printf("  cycles/solve: engine %.0f | aqif2 factor %.0f + z %.0f = %.0f\n", ce / B, cf / B,
           cz / B, (cf + cz) / B);
  }
  return 0;
}
