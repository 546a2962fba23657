// Dev tool: Z-solve level cost on one warp for division variants
// (0 full mdiv, 1 mdiv without the midpoint fix, 2 plain Markstein, 3 a*y).
#include <cstdio>
#include "../paper_2008_03276_b200/csrc/aqif2.cuh"
using namespace paqif;
template <int V>
__device__ __forceinline__ double vdiv(double a, double b, double y, bool& safe) {
  if (V == 0) return mdiv(a, b, y, safe);
  if (V == 1) {
    const unsigned ea = ((unsigned)__double2hiint(a) >> 20) & 0x7ffu;
    const bool tiny = ea < 524u;
    const double up = tiny ? 0x1p600 : 1.0, dn = tiny ? 0x1p-600 : 1.0;
    const double as = a * up;
    const double q = __dmul_rn(as, y);
    const double r0 = fma(-q, b, as);
    const double qs = fma(r0, y, q);
    safe = safe && (exp_safe(as) || is_zero(a));
    return qs * dn;
  }
  if (V == 2) return mdiv_lite(a, b, y, safe);
  return a * y;
}
template <int V>
__global__ void kz(const double* recg, int n, long long* cyc, double* out) {
  extern __shared__ double sm[];
  double* rec = sm;
  for (int i = threadIdx.x; i < (n / 2 + 1) * kRec2; i += blockDim.x) rec[i] = recg[i];
  __syncthreads();
  if (threadIdx.x < 32) {
    using A = Arith<true>;
    int z0; asm volatile("mov.u32 %0, 0;" : "=r"(z0));
    const double* c0 = rec + z0;
    const int s = n / 2;
    double xl0 = 0, xl1 = 0, xr0 = 0, xr1 = 0, acc = 0;
    bool safe = true;
    long long t0 = clock64();
    for (int p = 2; p < s; ++p) {
      const double* c = c0 + (size_t)(s - p) * kRec2;
      double at = c[12], ab = c[13];
      at = A::axpy_neg(at, c[2], xl0); ab = A::axpy_neg(ab, c[8], xl0);
      at = A::axpy_neg(at, c[4], xr0); ab = A::axpy_neg(ab, c[10], xr0);
      at = A::axpy_neg(at, c[1], xl1); ab = A::axpy_neg(ab, c[7], xl1);
      at = A::axpy_neg(at, c[5], xr1); ab = A::axpy_neg(ab, c[11], xr1);
      const double det = c[14], y = c[15];
      const double xp = vdiv<V>(A::det2(c[9], at, c[3], ab), det, y, safe);
      const double xq = vdiv<V>(A::det2(c[0], ab, c[6], at), det, y, safe);
      acc += xp;
      xl0 = xl1; xl1 = xp; xr1 = xr0; xr0 = xq;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[V] = (t1 - t0) / (s - 2); out[V] = acc + safe; }
  }
}
int main() {
  const int n = 512, s = n / 2;
  double* h = new double[(s + 1) * kRec2];
  for (int k = 0; k <= s; ++k) {
    double* r = h + k * kRec2;
    for (int j = 0; j < 12; ++j) r[j] = 0.01 * ((k * 7 + j * 3) % 11 - 5);
    r[0] = 4.0; r[9] = 4.0; r[3] = 0.1; r[6] = 0.2; r[12] = 1.0; r[13] = -1.0;
    r[14] = r[0] * r[9] - r[6] * r[3]; r[15] = 1.0 / r[14];
  }
  double *d, *o; long long* c;
  cudaMalloc(&d, (s + 1) * kRec2 * 8); cudaMalloc(&c, 64); cudaMalloc(&o, 64);
  cudaMemcpy(d, h, (s + 1) * kRec2 * 8, cudaMemcpyHostToDevice);
  size_t sm = (s + 1) * kRec2 * 8;
  for (int rep = 0; rep < 2; ++rep) {
    kz<0><<<1, 256, sm>>>(d, n, c, o); kz<1><<<1, 256, sm>>>(d, n, c, o);
    kz<2><<<1, 256, sm>>>(d, n, c, o); kz<3><<<1, 256, sm>>>(d, n, c, o);
  }
  long long r[4]; cudaMemcpy(r, c, 32, cudaMemcpyDeviceToHost);
  printf("z cycles/level: full mdiv %lld | no midpoint fix %lld | plain Markstein %lld | a*y %lld\n", r[0], r[1], r[2], r[3]);
}
