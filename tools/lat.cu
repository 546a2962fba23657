// Dev tool: dependent-chain latencies of the fp64 / warp ops the engine uses.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int iters) {
  double x = threadIdx.x * 1e-3 + 1.0;
  __shared__ double sh[64];
  sh[threadIdx.x] = x;
  __syncwarp();
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) / (4ll * iters);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __dadd_rn(x, a); x = __dadd_rn(x, b); x = __dadd_rn(x, a); x = __dadd_rn(x, b); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) / (4ll * iters);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __dmul_rn(x, a); x = __dmul_rn(x, b); x = __dmul_rn(x, a); x = __dmul_rn(x, b); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) / (4ll * iters);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __drcp_rn(x) + 1.0; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) / (iters);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __ddiv_rn(a, x) + 1.0; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) / (iters);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __shfl_sync(0xffffffff, x, (threadIdx.x + 1) & 31) + 1.0; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) / (iters);
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = sh[idx] + x; idx = (int)x & 31; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) / (iters);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { __syncwarp(); x += 1.0; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0) / (iters);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x += __any_sync(0xffffffff, x > 1e300) ? 1.0 : 0.5; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[8] = (t1 - t0) / (iters);
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMalloc(&c, 128);
  k<<<1, 32>>>(o, c, 0.999, 1e-3, 1000);
  k<<<1, 32>>>(o, c, 0.999, 1e-3, 10000);
  long long h[9]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("latency cycles: dfma %lld dadd %lld dmul %lld drcp+add %lld ddiv+add %lld shfl+dadd %lld lds+dadd+cvt %lld syncwarp+dadd %lld vote+dadd %lld\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8]);
}
