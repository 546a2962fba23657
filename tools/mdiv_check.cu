// Dev check: aqif2's branch-free quotient (mdiv: scaled Markstein with the
// subnormal midpoint correction) against __ddiv_rn, bit for bit, on random
// operands and on operands built so that a/b lands next to a midpoint of
// the subnormal grid.
#include <cstdio>
#include <cstdint>
#include "../paper_2008_03276_b200/csrc/aqif2.cuh"
using namespace paqif;
__device__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}
__global__ void k(unsigned long long* bad, unsigned long long* unsafe_cnt, int mode, int iters,
                  unsigned long long* bad_fix) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    uint64_t h = mix(tid * 1000003ull + it * 7919ull + mode * 0x9e3779b97f4a7c15ull);
    double b = 1.0 + (double)(h >> 12) * 0x1p-52;           // [1, 2)
    b = ldexp(b, (int)((h >> 4) & 63) - 32);                  // 2^-32 .. 2^31
    if (h & 1) b = -b;
    double a;
    uint64_t g = mix(h);
    if (mode == 0) {  // random a over a wide exponent range incl. subnormal quotients
      a = (1.0 + (double)(g >> 12) * 0x1p-52) * ldexp(1.0, (int)(g % 1100) - 1074);
    } else {          // a/b next to a subnormal midpoint (2j+1) 2^-1075
      b = fabs(b) < 1.0 ? b * 0x1p40 : b;              // keep a = m b above the subnormal range
      const double ms = (double)(2 * (g % 4096) + 1) * 0x1p-475;  // midpoint, scaled by 2^600
      a = __dmul_rn(ms, b) * 0x1p-600;                 // a/b within ~1 ulp(a) of the midpoint
    }
    if (g & 8) a = -a;
    const double y = __drcp_rn(b);
    bool safe = true;
    const double q1 = mdiv(a, b, y, safe);
    const double q2 = __ddiv_rn(a, b);
    bool safe_fix = true;
    const double q3 = mdiv_fix(a, b, y, safe_fix);
    if (safe_fix && __double_as_longlong(q3) != __double_as_longlong(q2)) {
      const unsigned long long c = atomicAdd(bad_fix, 1ull);
      if (c < 6) printf("a=%a b=%a mdiv_fix=%a ieee=%a\n", a, b, q3, q2);
    }
    if (!safe) {
      const unsigned long long c = atomicAdd(unsafe_cnt, 1ull);
      if (c < 3) printf("unsafe: a=%a b=%a\n", a, b);
    }
    else if (__double_as_longlong(q1) != __double_as_longlong(q2)) {
      const unsigned long long c = atomicAdd(bad, 1ull);
      if (c < 6) printf("a=%a b=%a mdiv=%a ieee=%a\n", a, b, q1, q2);
    }
  }
}
int main() {
  unsigned long long *d, h[3];
  cudaMalloc(&d, 24);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(d, 0, 24);
    k<<<1184, 256>>>(d, d + 1, mode, 64, d + 2);
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("mode %d: %d samples, mdiv mismatches %llu, flagged unsafe %llu; mdiv_fix mismatches %llu\n",
           mode, 1184 * 256 * 64, h[0], h[1], h[2]);
  }
}
