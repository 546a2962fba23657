// 2-D elastic deformation of the point contact by fp64 FFT convolution
// (replaces scipy.fft.rfftn/irfftn in FilmModel.deformation_full,
// paqif/ehl/film.py:43-56, 72-76).
//
//   D[j][i] = sum_{j',i'} t[|j-j'|][|i-i'|] u[j'][i']      (t symmetric)
//
// is the central (n+1)^2 window of the linear convolution of u with the
// mirrored (2n+1)^2 kernel; a circular convolution of period P >= 2n+1 is
// alias-free on that window, so P is the next power of two >= 2n+1.
// Pipeline (complex fp64, radix-2 in shared memory, one CTA per row):
//   pack u -> row FFT (rows < N) -> transpose -> row FFT (all P)
//   -> multiply by the transposed kernel spectrum -> inverse row FFT
//   -> transpose -> inverse row FFT (rows n..2n only) -> extract / P^2.
// Every kernel takes a device `gate`: with *gate == 0 it returns at once,
// so the sweep drivers can enqueue the fold pipeline after every line and
// let the device decide (film.py:83-91 fold rule).
#pragma once
#include <cuda_runtime.h>

namespace paqif {

struct FftPlan {
  int n;        // intervals; grid N = n+1
  int P;        // power of two >= 2n+1
  int logP;
  double2* W;   // P*P work
  double2* T;   // P*P work (transposed)
  double2* KT;  // P*P transposed kernel spectrum
  double2* tw;  // P/2 twiddles exp(-2 pi i t / P)
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__global__ void fft_twiddles(double2* tw, int P) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < P / 2) {
    double s, c;
    sincospi(-2.0 * (double)t / (double)P, &s, &c);
    tw[t] = make_double2(c, s);
  }
}

// In-place radix-2 FFT of `rows` rows of length P (row stride P), first row
// `row0`; inverse = conjugated twiddles, unnormalised.
__global__ void fft_rows_kernel(double2* data, int P, int logP, int row0, int rows,
                                const double2* __restrict__ tw, int inverse, const int* gate) {
  if (gate && *gate == 0) return;
  extern __shared__ double2 fsm[];
  const int r = row0 + blockIdx.x;
  if (blockIdx.x >= rows) return;
  double2* row = data + (size_t)r * P;
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    const int rev = __brev(k) >> (32 - logP);
    fsm[rev] = row[k];
  }
  __syncthreads();
  for (int s = 0; s < logP; ++s) {
    const int m = 1 << s;
    const int tstride = P >> (s + 1);
    for (int j = threadIdx.x; j < P / 2; j += blockDim.x) {
      const int k = j & (m - 1);
      const int base = (j >> s) << (s + 1);
      double2 w = tw[k * tstride];
      if (inverse) w.y = -w.y;
      const double2 a = fsm[base + k];
      const double2 b = cmul(fsm[base + k + m], w);
      fsm[base + k] = make_double2(a.x + b.x, a.y + b.y);
      fsm[base + k + m] = make_double2(a.x - b.x, a.y - b.y);
    }
    __syncthreads();
  }
  for (int k = threadIdx.x; k < P; k += blockDim.x) row[k] = fsm[k];
}

__global__ void transpose_kernel(const double2* __restrict__ in, double2* __restrict__ out, int P,
                                 const int* gate) {
  if (gate && *gate == 0) return;
  __shared__ double2 tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y)
    tile[y][threadIdx.x] = in[(size_t)(by + y) * P + bx + threadIdx.x];
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y)
    out[(size_t)(bx + y) * P + by + threadIdx.x] = tile[threadIdx.x][y];
}

// W[r][c] = u[r][c] (r, c < N), else 0; or, for the kernel, the mirrored table
__global__ void pack_kernel(double2* W, int P, int n, const double* __restrict__ src,
                            int mirrored_table, const int* gate) {
  if (gate && *gate == 0) return;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)P * P) return;
  const int r = (int)(idx / P), c = (int)(idx % P);
  const int N = n + 1;
  double v = 0.0;
  if (!mirrored_table) {
    if (r < N && c < N) v = src[(size_t)r * N + c];
  } else {
    if (r <= 2 * n && c <= 2 * n) v = src[(size_t)abs(r - n) * N + abs(c - n)];
  }
  W[idx] = make_double2(v, 0.0);
}

__global__ void cmul_kernel(double2* T, const double2* __restrict__ K, size_t count,
                            const int* gate) {
  if (gate && *gate == 0) return;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < count) T[idx] = cmul(T[idx], K[idx]);
}

// D[j][i] = Re W[j+n][i+n] / P^2; clears the gate (and the pending count)
__global__ void extract_kernel(const double2* __restrict__ W, int P, int n, double* D, int* gate,
                               int* pending_count) {
  if (gate && *gate == 0) return;
  const int N = n + 1;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double scale = 1.0 / ((double)P * (double)P);
  if (idx < (size_t)N * N) {
    const int j = (int)(idx / N), i = (int)(idx % N);
    D[idx] = W[(size_t)(j + n) * P + (i + n)].x * scale;
  }
}

__global__ void gate_clear_kernel(int* gate, int* pending_count) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && gate && *gate) {
    *gate = 0;
    if (pending_count) *pending_count = 0;
  }
}

inline int fft_threads(int P) { return P >= 1024 ? 512 : (P >= 256 ? 256 : 128); }

// Forward transform of the packed W: rows [0, nz_rows) nonzero; result in T
// (transposed spectrum).
inline void fft2_forward(const FftPlan& p, int nz_rows, const int* gate, cudaStream_t st) {
  const size_t smem = (size_t)p.P * sizeof(double2);
  fft_rows_kernel<<<nz_rows, fft_threads(p.P), smem, st>>>(p.W, p.P, p.logP, 0, nz_rows, p.tw, 0,
                                                          gate);
  dim3 tb(32, 8), tg(p.P / 32, p.P / 32);
  transpose_kernel<<<tg, tb, 0, st>>>(p.W, p.T, p.P, gate);
  fft_rows_kernel<<<p.P, fft_threads(p.P), smem, st>>>(p.T, p.P, p.logP, 0, p.P, p.tw, 0, gate);
}

// Sets cudaFuncAttributeMaxDynamicSharedMemorySize for the row kernel.
inline cudaError_t fft_prepare(int P) {
  return cudaFuncSetAttribute(fft_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(P * sizeof(double2)));
}

// Kernel spectrum KT for the table (N x N).
inline void fft_plan_kernel(const FftPlan& p, const double* table, cudaStream_t st) {
  const size_t PP = (size_t)p.P * p.P;
  fft_twiddles<<<(p.P / 2 + 255) / 256, 256, 0, st>>>(p.tw, p.P);
  pack_kernel<<<(unsigned)((PP + 255) / 256), 256, 0, st>>>(p.W, p.P, p.n, table, 1, nullptr);
  fft2_forward(p, 2 * p.n + 1, nullptr, st);
  cudaMemcpyAsync(p.KT, p.T, PP * sizeof(double2), cudaMemcpyDeviceToDevice, st);
}

// D = deformation(u), gated; clears gate and pending count at the end.
inline void fft_deformation(const FftPlan& p, const double* u, double* D, int* gate,
                            int* pending_count, cudaStream_t st) {
  const size_t PP = (size_t)p.P * p.P;
  const int N = p.n + 1;
  pack_kernel<<<(unsigned)((PP + 255) / 256), 256, 0, st>>>(p.W, p.P, p.n, u, 0, gate);
  fft2_forward(p, N, gate, st);
  cmul_kernel<<<(unsigned)((PP + 255) / 256), 256, 0, st>>>(p.T, p.KT, PP, gate);
  const size_t smem = (size_t)p.P * sizeof(double2);
  fft_rows_kernel<<<p.P, fft_threads(p.P), smem, st>>>(p.T, p.P, p.logP, 0, p.P, p.tw, 1, gate);
  dim3 tb(32, 8), tg(p.P / 32, p.P / 32);
  transpose_kernel<<<tg, tb, 0, st>>>(p.T, p.W, p.P, gate);
  fft_rows_kernel<<<N, fft_threads(p.P), smem, st>>>(p.W, p.P, p.logP, p.n, N, p.tw, 1, gate);
  extract_kernel<<<(unsigned)(((size_t)N * N + 255) / 256), 256, 0, st>>>(p.W, p.P, p.n, D, gate,
                                                                         pending_count);
  gate_clear_kernel<<<1, 32, 0, st>>>(gate, pending_count);
}

inline int fft_size_for(int n) {
  int P = 1;
  while (P < 2 * n + 1) P <<= 1;
  return P < 32 ? 32 : P;
}

}  // namespace paqif
