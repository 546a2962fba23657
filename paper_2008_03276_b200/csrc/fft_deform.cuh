// 2-D elastic deformation of the point contact by fp64 FFT convolution
// (replaces scipy.fft.rfftn/irfftn in FilmModel.deformation_full,
// paqif/ehl/film.py:43-56, 72-76).
//
//   D[j][i] = sum_{j',i'} t[|j-j'|][|i-i'|] u[j'][i']      (t symmetric)
//
// is the central (n+1)^2 window of the linear convolution of u with the
// mirrored (2n+1)^2 kernel K[c] = t[|c-n|], c = 0..2n.  In a circular
// convolution of period P the window needs K at offsets c = m - j in
// [0, 2n] only; for P >= 2n those never wrap except c = 2n -> 0, where
// K[2n] = K[0] = t[n].  So P = 2n is exact on the window; the driver uses the
// next power of two >= 2n.
// Pipeline (complex fp64, radix-2 in shared memory, one CTA per row):
//   pack u -> row FFT (rows < N) -> transpose -> row FFT (all P)
//   -> multiply by the transposed kernel spectrum -> inverse row FFT
//   -> transpose -> inverse row FFT (rows n..2n only) -> extract / P^2.
// Every kernel takes a device `gate`: with *gate == 0 it returns at once,
// so the sweep drivers can enqueue the fold pipeline after every line and
// let the device decide (film.py:83-91 fold rule).  Grids are capped
// (grid-stride loops), so a gated-off pipeline costs a few microseconds
// even at P = 4096 (an uncapped elementwise grid there is 65536 blocks).
#pragma once
#include <cooperative_groups.h>
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
  for (int rr = blockIdx.x; rr < rows; rr += gridDim.x) {
  const int r = row0 + rr;
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
  __syncthreads();
  }
}

__global__ void transpose_kernel(const double2* __restrict__ in, double2* __restrict__ out, int P,
                                 const int* gate) {
  if (gate && *gate == 0) return;
  __shared__ double2 tile[32][33];
  const int tiles_x = P / 32, tiles = tiles_x * tiles_x;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int bx = (t % tiles_x) * 32, by = (t / tiles_x) * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y)
      tile[y][threadIdx.x] = in[(size_t)(by + y) * P + bx + threadIdx.x];
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y)
      out[(size_t)(bx + y) * P + by + threadIdx.x] = tile[threadIdx.x][y];
    __syncthreads();
  }
}

// W[r][c] = u[r][c] (r, c < N), else 0; or, for the kernel, the mirrored table
__global__ void pack_kernel(double2* W, int P, int n, const double* __restrict__ src,
                            int mirrored_table, const int* gate) {
  if (gate && *gate == 0) return;
  const int N = n + 1;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (size_t)P * P;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / P), c = (int)(idx % P);
    double v = 0.0;
    if (!mirrored_table) {
      if (r < N && c < N) v = src[(size_t)r * N + c];
    } else {
      if (r <= 2 * n && c <= 2 * n) v = src[(size_t)abs(r - n) * N + abs(c - n)];
    }
    W[idx] = make_double2(v, 0.0);
  }
}

__global__ void cmul_kernel(double2* T, const double2* __restrict__ K, size_t count,
                            const int* gate) {
  if (gate && *gate == 0) return;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < count;
       idx += (size_t)gridDim.x * blockDim.x)
    T[idx] = cmul(T[idx], K[idx]);
}

// D[j][i] = Re W[j+n][i+n] / P^2; clears the gate (and the pending count)
__global__ void extract_kernel(const double2* __restrict__ W, int P, int n, double* D, int* gate,
                               int* pending_count) {
  if (gate && *gate == 0) return;
  const int N = n + 1;
  const double scale = 1.0 / ((double)P * (double)P);
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (size_t)N * N;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx / N), i = (int)(idx % N);
    const int rj = j + n < P ? j + n : j + n - P, ci = i + n < P ? i + n : i + n - P;
    D[idx] = W[(size_t)rj * P + ci].x * scale;
  }
}

__global__ void gate_clear_kernel(int* gate, int* pending_count) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && gate && *gate) {
    *gate = 0;
    if (pending_count) *pending_count = 0;
  }
}

// one radix-2 FFT of a row of P complex values through shared memory (fsm)
__device__ __forceinline__ void fft_row_smem(double2* row, int P, int logP,
                                             const double2* __restrict__ tw, int inverse,
                                             double2* fsm) {
  for (int k = threadIdx.x; k < P; k += blockDim.x) fsm[__brev(k) >> (32 - logP)] = row[k];
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
  __syncthreads();
}

// The whole gated fold as ONE cooperative kernel (grid-wide syncs between
// the phases): a fold that does not fire costs one launch, not ten.
// Phases as in fft_deformation below.  Dynamic smem: P double2.
__global__ void fft_fold_kernel(FftPlan p, const double* __restrict__ u, double* D, int* gate,
                                int* pending_count) {
  if (*gate == 0) return;  // every block reads the same gate before anyone clears it
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double2 fsm[];
  const int P = p.P, n = p.n, N = n + 1;
  const size_t PP = (size_t)P * P;
  const size_t gtid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t gthreads = (size_t)gridDim.x * blockDim.x;
  // pack u into W
  for (size_t idx = gtid; idx < PP; idx += gthreads) {
    const int r = (int)(idx / P), c = (int)(idx % P);
    p.W[idx] = make_double2((r < N && c < N) ? u[(size_t)r * N + c] : 0.0, 0.0);
  }
  grid.sync();
  for (int r = blockIdx.x; r < N; r += gridDim.x) fft_row_smem(p.W + (size_t)r * P, P, p.logP, p.tw, 0, fsm);
  grid.sync();
  auto transpose = [&](const double2* in, double2* out) {
    double2* tile = fsm;  // 32 x 33
    const int tiles_x = P / 32, tiles = tiles_x * tiles_x;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, ny = blockDim.x >> 5;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int bx = (t % tiles_x) * 32, by = (t / tiles_x) * 32;
      for (int y = ty; y < 32; y += ny) tile[y * 33 + tx] = in[(size_t)(by + y) * P + bx + tx];
      __syncthreads();
      for (int y = ty; y < 32; y += ny) out[(size_t)(bx + y) * P + by + tx] = tile[tx * 33 + y];
      __syncthreads();
    }
  };
  transpose(p.W, p.T);
  grid.sync();
  for (int r = blockIdx.x; r < P; r += gridDim.x) fft_row_smem(p.T + (size_t)r * P, P, p.logP, p.tw, 0, fsm);
  grid.sync();
  for (size_t idx = gtid; idx < PP; idx += gthreads) p.T[idx] = cmul(p.T[idx], p.KT[idx]);
  grid.sync();
  for (int r = blockIdx.x; r < P; r += gridDim.x) fft_row_smem(p.T + (size_t)r * P, P, p.logP, p.tw, 1, fsm);
  grid.sync();
  transpose(p.T, p.W);
  grid.sync();
  // output rows n..2n (row 2n wraps to row 0 when P = 2n)
  for (int rr = blockIdx.x; rr < N; rr += gridDim.x) {
    const int r = n + rr < P ? n + rr : n + rr - P;
    fft_row_smem(p.W + (size_t)r * P, P, p.logP, p.tw, 1, fsm);
  }
  grid.sync();
  const double scale = 1.0 / ((double)P * (double)P);
  for (size_t idx = gtid; idx < (size_t)N * N; idx += gthreads) {
    const int j = (int)(idx / N), i = (int)(idx % N);
    const int rj = j + n < P ? j + n : j + n - P, ci = i + n < P ? i + n : i + n - P;
    D[idx] = p.W[(size_t)rj * P + ci].x * scale;
  }
  grid.sync();
  if (gtid == 0) {
    *gate = 0;
    if (pending_count) *pending_count = 0;
  }
}

inline int fft_threads(int P) { return P >= 1024 ? 512 : (P >= 256 ? 256 : 128); }

// cooperative grid of fft_fold_kernel (blocks resident at once), cached per P
inline unsigned fold_grid(int P) {
  static int cachedP = 0;
  static unsigned g = 0;
  if (cachedP != P) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = (size_t)P * sizeof(double2) > 33 * 32 * sizeof(double2)
                            ? (size_t)P * sizeof(double2) : 33 * 32 * sizeof(double2);
    cudaFuncSetAttribute(fft_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fft_fold_kernel, fft_threads(P), smem);
    g = (unsigned)(sms * (per > 0 ? per : 1));
    cachedP = P;
  }
  return g;
}

inline cudaError_t fft_fold(const FftPlan& p, const double* u, double* D, int* gate,
                            int* pending_count, cudaStream_t st) {
  const size_t smem = (size_t)p.P * sizeof(double2) > 33 * 32 * sizeof(double2)
                          ? (size_t)p.P * sizeof(double2) : 33 * 32 * sizeof(double2);
  FftPlan pp = p;
  const double* uu = u;
  double* dd = D;
  int* gg = gate;
  int* pc = pending_count;
  void* args[] = {&pp, &uu, &dd, &gg, &pc};
  return cudaLaunchCooperativeKernel((const void*)fft_fold_kernel, dim3(fold_grid(p.P)),
                                     dim3(fft_threads(p.P)), args, smem, st);
}
// capped grids: elementwise / transpose tiles / FFT rows
constexpr unsigned kFftEwBlocks = 148 * 8;
inline unsigned ew_grid(size_t count) {
  const size_t b = (count + 255) / 256;
  return (unsigned)(b < kFftEwBlocks ? (b ? b : 1) : kFftEwBlocks);
}
inline unsigned row_grid(int rows, int P) {
  const int cap = P >= 4096 ? 148 * 3 : 148 * 6;
  return (unsigned)(rows < cap ? rows : cap);
}
inline unsigned tile_grid(int P) {
  const int tiles = (P / 32) * (P / 32);
  return (unsigned)(tiles < 148 * 8 ? tiles : 148 * 8);
}

// Forward transform of the packed W: rows [0, nz_rows) nonzero; result in T
// (transposed spectrum).
inline void fft2_forward(const FftPlan& p, int nz_rows, const int* gate, cudaStream_t st) {
  const size_t smem = (size_t)p.P * sizeof(double2);
  fft_rows_kernel<<<row_grid(nz_rows, p.P), fft_threads(p.P), smem, st>>>(p.W, p.P, p.logP, 0,
                                                                          nz_rows, p.tw, 0, gate);
  dim3 tb(32, 8);
  transpose_kernel<<<tile_grid(p.P), tb, 0, st>>>(p.W, p.T, p.P, gate);
  fft_rows_kernel<<<row_grid(p.P, p.P), fft_threads(p.P), smem, st>>>(p.T, p.P, p.logP, 0, p.P,
                                                                      p.tw, 0, gate);
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
  pack_kernel<<<ew_grid(PP), 256, 0, st>>>(p.W, p.P, p.n, table, 1, nullptr);
  // the mirrored table has 2n+1 rows; with P = 2n the row 2n wraps onto row 0,
  // which holds the same tap t[n] (so P = 2n is exact for the central window)
  fft2_forward(p, 2 * p.n + 1 < p.P ? 2 * p.n + 1 : p.P, nullptr, st);
  cudaMemcpyAsync(p.KT, p.T, PP * sizeof(double2), cudaMemcpyDeviceToDevice, st);
}

// D = deformation(u), gated; clears gate and pending count at the end.
inline void fft_deformation(const FftPlan& p, const double* u, double* D, int* gate,
                            int* pending_count, cudaStream_t st) {
  const size_t PP = (size_t)p.P * p.P;
  const int N = p.n + 1;
  pack_kernel<<<ew_grid(PP), 256, 0, st>>>(p.W, p.P, p.n, u, 0, gate);
  fft2_forward(p, N, gate, st);
  cmul_kernel<<<ew_grid(PP), 256, 0, st>>>(p.T, p.KT, PP, gate);
  const size_t smem = (size_t)p.P * sizeof(double2);
  fft_rows_kernel<<<row_grid(p.P, p.P), fft_threads(p.P), smem, st>>>(p.T, p.P, p.logP, 0, p.P,
                                                                      p.tw, 1, gate);
  dim3 tb(32, 8);
  transpose_kernel<<<tile_grid(p.P), tb, 0, st>>>(p.T, p.W, p.P, gate);
  // output rows n..2n; with P = 2n the last one wraps to row 0
  const int r1 = p.n + N <= p.P ? N : p.P - p.n;
  fft_rows_kernel<<<row_grid(r1, p.P), fft_threads(p.P), smem, st>>>(p.W, p.P, p.logP, p.n, r1,
                                                                     p.tw, 1, gate);
  if (r1 < N)
    fft_rows_kernel<<<row_grid(N - r1, p.P), fft_threads(p.P), smem, st>>>(p.W, p.P, p.logP, 0,
                                                                           N - r1, p.tw, 1, gate);
  extract_kernel<<<ew_grid((size_t)N * N), 256, 0, st>>>(p.W, p.P, p.n, D, gate, pending_count);
  gate_clear_kernel<<<1, 32, 0, st>>>(gate, pending_count);
}


}  // namespace paqif
