// 2-D elastic deformation of the point contact by fp64 FFT convolution
// (replaces scipy.fft.rfftn/irfftn in FilmModel.deformation_full,
// paqif/ehl/film.py:43-56, 72-76).
//
//   D[j][i] = sum_{j',i'} t[|j-j'|][|i-i'|] u[j'][i']
//
// is the central (n+1)^2 window of the linear convolution of u with the
// mirrored (2n+1)^2 kernel K[r][c] = t[|r-n|][|c-n|].  In a circular
// convolution of period P the window needs K at offsets in [0, 2n] only; for
// P >= 2n those never wrap except 2n -> 0, where K[2n] = K[0] (= t[n] taps).
// So P = 2n is exact on the window; the driver uses the next power of two
// >= 2n.
//
// One cooperative kernel, three phases separated by grid barriers; no
// transposes and no P x P complex buffers:
//   R  rows r < N: real row of length P packed as H = P/2 complex points
//      (even + i odd), DIF FFT of length H in shared memory, split into the
//      H+1 non-redundant bins of the real row's spectrum  -> W[r][0..H]
//   C  columns k = 0..H: load W[.][k] (rows >= N are zero), DIF FFT of
//      length P (bit-reversed result), multiply by the kernel spectrum
//      (stored in the same bit-reversed order), inverse DIT FFT (natural
//      order), keep the N output rows n..2n (wrapped)   -> W[m][k]
//   I  output rows m < N: merge bins k and H-k back into H complex points,
//      inverse DIT FFT of length H, unpack even/odd, scale 1/(P H) -> D[m]
// The kernel spectrum is made once by phases R and C of the same kernel
// (plan mode).  Butterflies are radix-2^2 (two radix-2 stages per barrier,
// 4 points per thread), twiddles staged in shared memory.
// Every launch takes a device `gate`: with *gate == 0 it returns at once, so
// the sweep drivers can enqueue a fold after every line and let the device
// decide (film.py:83-91 fold rule).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

namespace paqif {

struct FftPlan {
  int n;        // intervals; grid N = n+1
  int P;        // power of two >= 2n
  int logP;
  double2* W;   // P rows x (P/2 + 1) bins: half spectra / column results
  double2* KT;  // (P/2 + 1) columns x P: kernel spectrum, bit-reversed rows
  double2* tw;  // P/2 twiddles exp(-2 pi i t / P)
};

// Complex arithmetic with the rounding spelled out (explicit FMA / RN
// intrinsics): the compiler's contraction choices would otherwise differ
// between the kernels that inline the same row / column functions (the
// one-kernel fold and the sharded phases), and bit-identical results across
// them are part of the contract (fft_shard.cuh).
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)),
                      __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double half_(double v) { return __dmul_rn(0.5, v); }
__device__ __forceinline__ int bitrev(int k, int bits) { return (int)(__brev(k) >> (32 - bits)); }

// Shared-memory position of element i of a transform buffer: the low three
// index bits (the 16-byte slot within a 128-byte bank row) XOR-folded with
// every higher 3-bit group.  Bijective; 32 consecutive elements still fill 8
// distinct slots four times, and so do the strided and bit-reversed access
// patterns of the short-span stages and of the half-spectrum split (which
// would otherwise hit one slot: up to 32-way bank conflicts,
// profiles/fold_ncu_r02.txt).
__device__ __forceinline__ int sw(int i) {
  int f = i >> 3;
  f ^= f >> 3;
  f ^= f >> 6;
  f ^= f >> 12;
  return i ^ (f & 7);
}

// Twiddles by level: stage tables W_{2^L}^t (t < 2^(L-1)) stored one after
// the other in shared memory, level L at offset 2^(L-1), for L < logP; the
// top level (W_P^t) is read from the global table (consecutive t: coalesced,
// L1-resident).  A butterfly stage reads consecutive t of ONE level, so the
// shared reads are conflict-free -- the strided reads of a single W_P table
// (every 2^s-th entry) were 59 % of the fold's excess shared wavefronts
// (profiles/fold_ncu_r02.txt).  Same values, so the output is unchanged.
struct Twiddles {
  const double2* lv;  // shared: levels 1 .. logP-1
  const double2* top; // global: W_P^t, t < P/2
  int logP;
  __device__ __forceinline__ double2 at(int L, int t, int inverse) const {
    const double2 w = L == logP ? top[t] : lv[(1 << (L - 1)) + t];
    return inverse ? make_double2(w.x, -w.y) : w;
  }
};
// build the shared levels (P/2 entries, index 0 unused); all threads call
__device__ __forceinline__ void twiddle_levels(double2* lv, const double2* top, int logP) {
  const int half = 1 << (logP - 1);
  for (int idx = 1 + threadIdx.x; idx < half; idx += blockDim.x) {
    const int L = 32 - __clz(idx);  // 2^(L-1) <= idx < 2^L
    const int t = idx - (1 << (L - 1));
    lv[idx] = top[t << (logP - L)];
  }
}

__global__ void fft_twiddles(double2* tw, int P) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < P / 2) {
    double s, c;
    sincospi(-2.0 * (double)t / (double)P, &s, &c);
    tw[t] = make_double2(c, s);
  }
}

// Decimation in frequency, natural order in -> bit-reversed order out, length
// L = 2^logL <= P (stage of span m uses the twiddles of levels log2 m and
// log2 m + 1).  Caller synchronises before; ends synchronised.
__device__ __forceinline__ void fft_dif_smem(double2* x, int L, int logL, const Twiddles& tw,
                                             int inverse) {
  int lm = logL - 1;  // m = 2^lm: current butterfly span
  for (; lm >= 1; lm -= 2) {
    const int m = 1 << lm, h = m >> 1;
    for (int j = threadIdx.x; j < L / 4; j += blockDim.x) {
      const int q = j & (h - 1);
      const int base = (j >> (lm - 1)) << (lm + 1);
      const double2 x0 = x[sw(base + q)], x1 = x[sw(base + q + h)];
      const double2 x2 = x[sw(base + q + m)], x3 = x[sw(base + q + m + h)];
      const double2 a0 = cadd(x0, x2), a1 = cadd(x1, x3);
      const double2 a2 = cmul(csub(x0, x2), tw.at(lm + 1, q, inverse));
      const double2 a3 = cmul(csub(x1, x3), tw.at(lm + 1, q + h, inverse));
      const double2 wb = tw.at(lm, q, inverse);
      x[sw(base + q)] = cadd(a0, a1);
      x[sw(base + q + h)] = cmul(csub(a0, a1), wb);
      x[sw(base + q + m)] = cadd(a2, a3);
      x[sw(base + q + m + h)] = cmul(csub(a2, a3), wb);
    }
    __syncthreads();
  }
  if (lm == 0) {  // odd log2 L: last span-1 stage, unit twiddles
    for (int j = threadIdx.x; j < L / 2; j += blockDim.x) {
      const double2 a = x[sw(2 * j)], b = x[sw(2 * j + 1)];
      x[sw(2 * j)] = cadd(a, b);
      x[sw(2 * j + 1)] = csub(a, b);
    }
    __syncthreads();
  }
}

// Decimation in time, bit-reversed order in -> natural order out.
__device__ __forceinline__ void fft_dit_smem(double2* x, int L, int logL, const Twiddles& tw,
                                             int inverse) {
  int s = 0;
  for (; s + 1 < logL; s += 2) {
    const int m = 1 << s;  // stage s pairs (q, q+m); stage s+1 pairs (q, q+2m)
    for (int j = threadIdx.x; j < L / 4; j += blockDim.x) {
      const int q = j & (m - 1);
      const int base = (j >> s) << (s + 2);
      const double2 w0 = tw.at(s + 1, q, inverse);
      const double2 x0 = x[sw(base + q)], x1 = x[sw(base + q + m)];
      const double2 x2 = x[sw(base + q + 2 * m)], x3 = x[sw(base + q + 3 * m)];
      const double2 t1 = cmul(x1, w0), t3 = cmul(x3, w0);
      const double2 a0 = cadd(x0, t1), a1 = csub(x0, t1);
      const double2 u2 = cmul(cadd(x2, t3), tw.at(s + 2, q, inverse));
      const double2 u3 = cmul(csub(x2, t3), tw.at(s + 2, q + m, inverse));
      x[sw(base + q)] = cadd(a0, u2);
      x[sw(base + q + 2 * m)] = csub(a0, u2);
      x[sw(base + q + m)] = cadd(a1, u3);
      x[sw(base + q + 3 * m)] = csub(a1, u3);
    }
    __syncthreads();
  }
  if (s < logL) {  // odd log2 L: last radix-2 stage
    const int m = 1 << s;
    for (int j = threadIdx.x; j < L / 2; j += blockDim.x) {
      const int k = j & (m - 1);
      const int base = (j >> s) << (s + 1);
      const double2 a = x[sw(base + k)];
      const double2 b = cmul(x[sw(base + k + m)], tw.at(s + 1, k, inverse));
      x[sw(base + k)] = cadd(a, b);
      x[sw(base + k + m)] = csub(a, b);
    }
    __syncthreads();
  }
}

// The three phases, per row / column, shared by the one-kernel fold and the
// sharded fold (fft_shard.cuh): the same arithmetic whichever block or GPU
// computes a row or column, so the results are bit-identical.
// Phase R, row r: half spectrum of the real row (plan_mode: of the mirrored
// table) -> out[0..H].  buf: P double2 of shared memory, tw: the twiddle levels.
__device__ __forceinline__ void fold_row_r(const FftPlan& p, const double* __restrict__ src, int r,
                                           int plan_mode, double2* buf, const Twiddles& tw,
                                           double2* out) {
  const int P = p.P, logP = p.logP, H = P >> 1, logH = logP - 1, n = p.n, N = n + 1;
  const int rows = plan_mode ? (2 * n + 1 < P ? 2 * n + 1 : P) : N;
  for (int c = threadIdx.x; c < H; c += blockDim.x) {
    const int c0 = 2 * c, c1 = 2 * c + 1;
    double v0 = 0.0, v1 = 0.0;
    if (!plan_mode) {
      const double* row = src + (size_t)r * N;
      if (c0 < N) v0 = row[c0];
      if (c1 < N) v1 = row[c1];
    } else {
      const double* row = src + (size_t)abs(r - n) * N;
      if (c0 < rows) v0 = row[abs(c0 - n)];
      if (c1 < rows) v1 = row[abs(c1 - n)];
    }
    buf[sw(c)] = make_double2(v0, v1);
  }
  __syncthreads();
  fft_dif_smem(buf, H, logH, tw, 0);
  for (int k = threadIdx.x; k <= H; k += blockDim.x) {
    const double2 zk = buf[sw(bitrev(k & (H - 1), logH))];
    const double2 zm = buf[sw(bitrev((H - k) & (H - 1), logH))];
    const double2 e = make_double2(half_(__dadd_rn(zk.x, zm.x)), half_(__dsub_rn(zk.y, zm.y)));
    const double2 o = make_double2(half_(__dadd_rn(zk.y, zm.y)), -half_(__dsub_rn(zk.x, zm.x)));
    const double2 w = k < H ? tw.top[k] : make_double2(-1.0, 0.0);
    out[k] = cadd(e, cmul(w, o));
  }
  __syncthreads();
}

// Phase C, column k: load W[.][k] (rows >= `rows` zero), forward FFT; plan
// mode stores the spectrum in KT, else multiplies by it, inverse FFT and
// leaves the N output rows n..2n (wrapped) in buf[sw(wrap(m))] for the caller.
__device__ __forceinline__ void fold_col_c(const FftPlan& p, const double2* __restrict__ Wsrc,
                                           int k, int rows, int plan_mode, double2* buf,
                                           const Twiddles& tw) {
  const int P = p.P, logP = p.logP, ld = (P >> 1) + 1;
  for (int r = threadIdx.x; r < P; r += blockDim.x)
    buf[sw(r)] = r < rows ? Wsrc[(size_t)r * ld + k] : make_double2(0.0, 0.0);
  __syncthreads();
  fft_dif_smem(buf, P, logP, tw, 0);
  double2* kt = p.KT + (size_t)k * P;
  if (plan_mode) {
    for (int j = threadIdx.x; j < P; j += blockDim.x) kt[j] = buf[sw(j)];
    __syncthreads();
    return;
  }
  for (int j = threadIdx.x; j < P; j += blockDim.x) buf[sw(j)] = cmul(buf[sw(j)], kt[j]);
  __syncthreads();
  fft_dit_smem(buf, P, logP, tw, 1);
}
__device__ __forceinline__ int fold_wrap(int m, int n, int P) {
  return m + n < P ? m + n : m + n - P;  // row 2n wraps to 0 when P = 2n
}

// Phase I, output row m: merge the half spectrum in[0..H] and inverse FFT;
// the N outputs are ((c & 1) ? buf[c >> 1].y : .x) * scale, c = wrap(i).
__device__ __forceinline__ void fold_row_i(const FftPlan& p, const double2* __restrict__ in,
                                           double2* buf, const Twiddles& tw) {
  const int P = p.P, logP = p.logP, H = P >> 1, logH = logP - 1;
  for (int k = threadIdx.x; k < H; k += blockDim.x) {
    const double2 yk = in[k], ym = in[H - k];
    const double2 e = make_double2(half_(__dadd_rn(yk.x, ym.x)), half_(__dsub_rn(yk.y, ym.y)));
    const double2 o = cmul(make_double2(half_(__dsub_rn(yk.x, ym.x)), half_(__dadd_rn(yk.y, ym.y))),
                           tw.at(tw.logP, k, 1));
    buf[sw(bitrev(k, logH))] = make_double2(__dsub_rn(e.x, o.y), __dadd_rn(e.y, o.x));
  }
  __syncthreads();
  fft_dit_smem(buf, H, logH, tw, 1);
}
__device__ __forceinline__ double fold_out(const double2* buf, int i, int n, int P,
                                           double scale) {
  const int c = fold_wrap(i, n, P);
  const double2 v = buf[sw(c >> 1)];
  return __dmul_rn((c & 1) ? v.y : v.x, scale);
}

// plan_mode 0: D = deformation(src = u, N x N), gated; clears the gate and the
// pending count.  plan_mode 1: KT = spectrum of the mirrored table (src).
// Dynamic smem: P + P/2 double2.
__global__ void __launch_bounds__(256) fft_conv_kernel(FftPlan p, const double* __restrict__ src,
                                                       double* D, int* gate, int* pending_count,
                                                       int plan_mode) {
  if (gate && *gate == 0) return;  // every block reads the gate before anyone clears it
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double2 fsm[];
  const int P = p.P, H = P >> 1, n = p.n, N = n + 1;
  const int ld = H + 1;
  double2* buf = fsm;
  double2* twd = fsm + P;
  twiddle_levels(twd, p.tw, p.logP);
  const Twiddles tw{twd, p.tw, p.logP};
  const int rows = plan_mode ? (2 * n + 1 < P ? 2 * n + 1 : P) : N;

  // ---- R: half spectra of the real rows
  for (int r = blockIdx.x; r < rows; r += gridDim.x)
    fold_row_r(p, src, r, plan_mode, buf, tw, p.W + (size_t)r * ld);
  grid.sync();

  // ---- C: column transforms, kernel product, inverse, output rows
  for (int k = blockIdx.x; k <= H; k += gridDim.x) {
    fold_col_c(p, p.W, k, rows, plan_mode, buf, tw);
    if (plan_mode) continue;
    for (int m = threadIdx.x; m < N; m += blockDim.x)
      p.W[(size_t)m * ld + k] = buf[sw(fold_wrap(m, n, P))];
    __syncthreads();
  }
  if (plan_mode) return;
  grid.sync();

  // ---- I: real output rows from their half spectra
  const double scale = 1.0 / ((double)P * (double)H);
  for (int m = blockIdx.x; m < N; m += gridDim.x) {
    fold_row_i(p, p.W + (size_t)m * ld, buf, tw);
    double* out = D + (size_t)m * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) out[i] = fold_out(buf, i, n, P, scale);
    __syncthreads();
  }
  grid.sync();
  if (gate && blockIdx.x == 0 && threadIdx.x == 0) {
    *gate = 0;
    if (pending_count) *pending_count = 0;
  }
}

constexpr int kFftThreads = 256;
inline size_t fold_smem(int P) { return (size_t)(P + P / 2) * sizeof(double2); }

// cooperative grid of fft_conv_kernel (blocks resident at once), cached per P
inline unsigned fold_grid(int P) {
  static int cachedP = 0;
  static unsigned g = 0;
  if (cachedP != P) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = fold_smem(P);
    cudaFuncSetAttribute(fft_conv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fft_conv_kernel, kFftThreads, smem);
    g = (unsigned)(sms * (per > 0 ? per : 1));
    cachedP = P;
  }
  return g;
}

inline cudaError_t fft_conv_launch(const FftPlan& p, const double* src, double* D, int* gate,
                                   int* pending_count, int plan_mode, cudaStream_t st) {
  const size_t smem = fold_smem(p.P);
  FftPlan pp = p;
  const double* ss = src;
  double* dd = D;
  int* gg = gate;
  int* pc = pending_count;
  int pm = plan_mode;
  void* args[] = {&pp, &ss, &dd, &gg, &pc, &pm};
  return cudaLaunchCooperativeKernel((const void*)fft_conv_kernel, dim3(fold_grid(p.P)),
                                     dim3(kFftThreads), args, smem, st);
}

// D = deformation(u), gated; clears gate and pending count.
inline cudaError_t fft_fold(const FftPlan& p, const double* u, double* D, int* gate,
                            int* pending_count, cudaStream_t st) {
  return fft_conv_launch(p, u, D, gate, pending_count, 0, st);
}
inline cudaError_t fft_deformation(const FftPlan& p, const double* u, double* D, int* gate,
                                   int* pending_count, cudaStream_t st) {
  return fft_conv_launch(p, u, D, gate, pending_count, 0, st);
}

// Kernel spectrum KT for the table (N x N).
inline cudaError_t fft_plan_kernel(const FftPlan& p, const double* table, cudaStream_t st) {
  fft_twiddles<<<(p.P / 2 + 255) / 256, 256, 0, st>>>(p.tw, p.P);
  return fft_conv_launch(p, table, nullptr, nullptr, nullptr, 1, st);
}

inline size_t fft_w_elems(int P) { return (size_t)P * (P / 2 + 1); }
inline size_t fft_kt_elems(int P) { return (size_t)(P / 2 + 1) * P; }

}  // namespace paqif
