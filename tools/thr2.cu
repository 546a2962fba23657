// Dev tool: single-warp issue/latency costs relevant to the line solver.
#include <cstdio>
__device__ __noinline__ double slow(double a) { return a * 1.0001 + sqrt(a); }
__global__ void k(double* out, long long* cyc, double a, double b, int iters) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  __shared__ double sh[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) sh[i] = i * 1e-3;
  __syncwarp();
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
    x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, a); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, a);
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 100 / (8ll * iters);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x0 = __dadd_rn(x0, a); x0 = __dmul_rn(x0, b); x0 = __dadd_rn(x0, a); x0 = __dmul_rn(x0, b);
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) * 100 / (4ll * iters);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x1 = fma(x1, a, b);
    if (__double2hiint(x1) == 0x12345678) x1 = slow(x1);  // never taken
    x1 = fma(x1, a, b);
    if (__double2hiint(x1) == 0x12345679) x1 = slow(x1);
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) * 100 / (2ll * iters);
  t0 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    x2 = x2 + sh[(idx + i) & 1023] + sh[(idx + i + 7) & 1023] + sh[(idx + i + 13) & 1023] +
         sh[(idx + i + 29) & 1023];
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) * 100 / (1ll * iters);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x3 = __dmul_rn(x3, b); x4 = __dmul_rn(x4, b); x5 = __dmul_rn(x5, b); x6 = __dmul_rn(x6, b);
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) * 100 / (4ll * iters);
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8192); cudaMalloc(&c, 128);
  k<<<1, 32>>>(o, c, 0.999, 1.0001, 100);
  k<<<1, 32>>>(o, c, 0.999, 1.0001, 4000);
  long long h[5]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("dadd issue %.2f | dadd/dmul dep latency %.2f | fma+never-taken-branch %.2f per step | 4 lds + 4 dadd chain %.2f per iter | dmul issue %.2f\n",
         h[0] / 100.0, h[1] / 100.0, h[2] / 100.0, h[3] / 100.0, h[4] / 100.0);
}
