// Dev tool: issue cost (cycles per warp instruction) of fp64 ops with 8
// independent chains, for 1, 2 and 32 active lanes of a single warp.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int iters, int lanes) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  if ((int)threadIdx.x < lanes) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 100 / (8ll * iters);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      x0 = __shfl_xor_sync(0xffffffffu >> (32 - lanes), x0, 1) + x1;
      x2 = __shfl_xor_sync(0xffffffffu >> (32 - lanes), x2, 1) + x3;
      x4 = __shfl_xor_sync(0xffffffffu >> (32 - lanes), x4, 1) + x5;
      x6 = __shfl_xor_sync(0xffffffffu >> (32 - lanes), x6, 1) + x7;
    }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = (t1 - t0) * 100 / (4ll * iters);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      x0 = __drcp_rn(x0); x1 = __drcp_rn(x1); x2 = __drcp_rn(x2); x3 = __drcp_rn(x3);
    }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = (t1 - t0) * 100 / (4ll * iters);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x0 = __drcp_rn(x0); }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[3] = (t1 - t0) * 100 / (1ll * iters);
  }
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8192); cudaMalloc(&c, 128);
  for (int lanes : {1, 2, 32}) {
    k<<<1, 32>>>(o, c, 0.999, 1e-3, 100, lanes);
    k<<<1, 32>>>(o, c, 0.999, 1e-3, 2000, lanes);
    long long h[4]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%2d lanes: dfma/instr %.2f  shfl+dadd pair %.2f  drcp x4 ILP %.2f  drcp latency %.2f cycles\n",
           lanes, h[0] / 100.0, h[1] / 100.0, h[2] / 100.0, h[3] / 100.0);
  }
}
