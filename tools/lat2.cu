// Dev tool: fp64 dependent-chain latency as seen by ONE active lane (the
// line-solve situation) vs a full warp, and an smem-load + DFMA chain.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int iters, int mode) {
  __shared__ double sh[256];
  sh[threadIdx.x] = threadIdx.x * 1e-3;
  __syncthreads();
  double x = threadIdx.x * 1e-3 + 1.0;
  const bool act = mode == 0 ? threadIdx.x == 0 : threadIdx.x < 32;
  if (act) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / (4ll * iters);
    t0 = clock64();
    int idx = 0;
    for (int i = 0; i < iters; ++i) { x = fma(sh[idx], a, x); idx = ((int)x) & 127; }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = (t1 - t0) / iters;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = x * a; x = x + b; }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = (t1 - t0) / (2ll * iters);
    float f = (float)x;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { f = fmaf(f, (float)a, (float)b); f = fmaf(f, (float)a, (float)b); }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[3] = (t1 - t0) / (2ll * iters);
    x += f;
  }
  __syncthreads();
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8192); cudaMalloc(&c, 128);
  for (int mode = 0; mode < 2; ++mode) {
    for (int threads : {32, 256}) {
      k<<<1, threads>>>(o, c, 0.999, 1e-3, 1000, mode);
      k<<<1, threads>>>(o, c, 0.999, 1e-3, 20000, mode);
      long long h[4]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
      printf("%s, %d threads: dfma %lld  lds->dfma %lld  dmul/dadd %lld  ffma %lld cycles\n",
             mode == 0 ? "one lane" : "full warp", threads, h[0], h[1], h[2], h[3]);
    }
  }
}
