// Dev tool: cycles per level of aqif2_zsolve / aqif2_factor on one lane.
#include <cstdio>
#include "../paper_2008_03276_b200/csrc/aqif2.cuh"
using namespace paqif;
template <bool EXACT>
__global__ void kz(const double* recg, int n, double* xout, long long* cyc) {
  extern __shared__ double sm[];
  double* rec = sm;
  double* x = rec + (n / 2 + 1) * kRec2;
  for (int i = threadIdx.x; i < (n / 2 + 1) * kRec2; i += blockDim.x) rec[i] = recg[i];
  __syncthreads();
  if (threadIdx.x < 32) {
    long long t0 = clock64();
    aqif2_zsolve<EXACT, false>(rec, n, threadIdx.x);
    int st = 0;
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      cyc[0] = (t1 - t0) / (n / 2);
      cyc[1] = st;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) xout[i] = x[i];
}
int main() {
  const int n = 512, s = n / 2;
  double* h = new double[(s + 1) * kRec2];
  for (int k = 0; k <= s; ++k) {
    double* r = h + k * kRec2;
    for (int j = 0; j < 12; ++j) r[j] = 0.01 * ((k * 7 + j * 3) % 11 - 5);
    r[0] = 4.0; r[9] = 4.0; r[3] = 0.1; r[6] = 0.2;
    r[12] = 1.0; r[13] = -1.0;
    r[14] = r[0] * r[9] - r[6] * r[3];
    r[15] = 1.0 / r[14];
  }
  double *d, *x; long long* c;
  cudaMalloc(&d, (s + 1) * kRec2 * 8); cudaMalloc(&x, n * 8); cudaMalloc(&c, 16);
  cudaMemcpy(d, h, (s + 1) * kRec2 * 8, cudaMemcpyHostToDevice);
  size_t sm = ((s + 1) * kRec2 + n) * 8;
  for (int rep = 0; rep < 2; ++rep) {
    kz<true><<<1, 256, sm>>>(d, n, x, c);
    long long r[2]; cudaMemcpy(r, c, 16, cudaMemcpyDeviceToHost);
    printf("exact z: %lld cycles/level (st %lld)\n", r[0], r[1]);
    kz<false><<<1, 256, sm>>>(d, n, x, c);
    cudaMemcpy(r, c, 16, cudaMemcpyDeviceToHost);
    printf("fast  z: %lld cycles/level (st %lld)\n", r[0], r[1]);
  }
}
