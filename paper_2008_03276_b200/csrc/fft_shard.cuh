// Sharded point-contact deformation fold across the GPUs of one node
// (config 5): the x/y line chains stay in the reference's
// Gauss-Seidel order, replicated on every rank (deterministic kernels, so
// every rank holds the same pressure and takes the same fold decisions);
// each full deformation is split over the ranks instead of computed by all:
//
//   R  rank r: half spectra of its slab of the N input rows, written into
//      EVERY rank's half-spectrum buffer W (peer stores over NVLink)
//   |  barrier (system-scope counters in every rank's memory)
//   C  rank r: its slab of the H+1 columns (forward FFT, kernel product,
//      inverse), the N output rows of each column written into every W
//   |  barrier
//   I  rank r: its slab of the N output rows (merge + inverse row FFT),
//      written into every rank's deformation base D
//   |  barrier, then the gate / pending count are cleared
//
// The pressure exchange the survey plans as an allgather before each fold
// is unnecessary here (replicated pressures); the transposes of the FFT are
// the exchange, done as stores straight into the peers' buffers by the
// kernels that produce the data.  Every row and column runs the same device
// function as the one-kernel fold (fft_deform.cuh), so the result is
// bit-identical to the single-GPU fold for any number of ranks
// (tests/test_ehl_point_shard_gpu.py checks it with emulated ranks).
// Peer pointers come from CUDA IPC handles exchanged by the host
// (paqif_ehl_point_ipc_handles / paqif_ehl_point_attach_peers).
#pragma once
#include "fft_deform.cuh"

namespace paqif {

constexpr int kFoldMaxRanks = 8;

struct FoldPeers {
  int rank, world;
  double2* W[kFoldMaxRanks];    // every rank's half-spectrum buffer (own included)
  double* D[kFoldMaxRanks];     // every rank's deformation base
  unsigned* bar[kFoldMaxRanks]; // every rank's barrier words: [0] arrivals, [1] expected
};

__host__ __device__ inline int fold_slab_lo(int count, int rank, int world) {
  return (int)(((long long)count * rank) / world);
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// R: rows [lo, hi) of the N input rows
__global__ void __launch_bounds__(256) fold_shard_r_kernel(FftPlan p, const double* __restrict__ u,
                                                           FoldPeers q, int vrank,
                                                           const int* gate) {
  if (*gate == 0) return;
  extern __shared__ double2 fsm[];
  const int P = p.P, H = P >> 1, N = p.n + 1, ld = H + 1;
  double2* buf = fsm;
  double2* twd = fsm + P;
  twiddle_levels(twd, p.tw, p.logP);
  const Twiddles tw{twd, p.tw, p.logP};
  __syncthreads();
  const int lo = fold_slab_lo(N, vrank, q.world), hi = fold_slab_lo(N, vrank + 1, q.world);
  double2* own = q.W[q.rank];
  for (int r = lo + blockIdx.x; r < hi; r += gridDim.x) {
    fold_row_r(p, u, r, 0, buf, tw, own + (size_t)r * ld);
    for (int pr = 0; pr < q.world; ++pr) {
      if (q.W[pr] == own) continue;
      double2* dst = q.W[pr] + (size_t)r * ld;
      for (int k = threadIdx.x; k <= H; k += blockDim.x) dst[k] = own[(size_t)r * ld + k];
    }
  }
  __threadfence_system();
}

// C: columns [lo, hi) of the H+1 kept columns
__global__ void __launch_bounds__(256) fold_shard_c_kernel(FftPlan p, FoldPeers q, int vrank,
                                                           const int* gate) {
  if (*gate == 0) return;
  extern __shared__ double2 fsm[];
  const int P = p.P, H = P >> 1, n = p.n, N = n + 1, ld = H + 1;
  double2* buf = fsm;
  double2* twd = fsm + P;
  twiddle_levels(twd, p.tw, p.logP);
  const Twiddles tw{twd, p.tw, p.logP};
  __syncthreads();
  const int lo = fold_slab_lo(H + 1, vrank, q.world), hi = fold_slab_lo(H + 1, vrank + 1, q.world);
  for (int k = lo + blockIdx.x; k < hi; k += gridDim.x) {
    fold_col_c(p, q.W[q.rank], k, N, 0, buf, tw);
    for (int pr = 0; pr < q.world; ++pr)
      for (int m = threadIdx.x; m < N; m += blockDim.x)
        q.W[pr][(size_t)m * ld + k] = buf[sw(fold_wrap(m, n, P))];
    __syncthreads();
  }
  __threadfence_system();
}

// I: output rows [lo, hi)
__global__ void __launch_bounds__(256) fold_shard_i_kernel(FftPlan p, FoldPeers q, int vrank,
                                                           const int* gate) {
  if (*gate == 0) return;
  extern __shared__ double2 fsm[];
  const int P = p.P, H = P >> 1, n = p.n, N = n + 1, ld = H + 1;
  double2* buf = fsm;
  double2* twd = fsm + P;
  twiddle_levels(twd, p.tw, p.logP);
  const Twiddles tw{twd, p.tw, p.logP};
  __syncthreads();
  const double scale = 1.0 / ((double)P * (double)H);
  const int lo = fold_slab_lo(N, vrank, q.world), hi = fold_slab_lo(N, vrank + 1, q.world);
  for (int m = lo + blockIdx.x; m < hi; m += gridDim.x) {
    fold_row_i(p, q.W[q.rank] + (size_t)m * ld, buf, tw);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const double v = fold_out(buf, i, n, P, scale);
      for (int pr = 0; pr < q.world; ++pr) q.D[pr][(size_t)m * N + i] = v;
    }
    __syncthreads();
  }
  __threadfence_system();
}

// Cross-rank barrier: one arrival on every rank's counter, then wait for
// all of this barrier's arrivals on our own.  The expected count advances
// only when the barrier runs (gated like the fold), so ranks that skip a
// fold together stay in step.  A peer that never arrives (a rank died)
// ends the wait after ~seconds with err bit 64 instead of hanging the GPU.
__global__ void fold_xbar_kernel(FoldPeers q, const int* gate, int* err) {
  if (*gate == 0 || threadIdx.x != 0 || blockIdx.x != 0) return;
  __threadfence_system();
  unsigned* mine = q.bar[q.rank];
  const unsigned e = mine[1] + (unsigned)q.world;
  mine[1] = e;
  for (int pr = 0; pr < q.world; ++pr) atomicAdd_system(q.bar[pr], 1u);
  long long spins = 0;
  while ((int)(ld_acquire_sys(mine) - e) < 0) {
    __nanosleep(200);
    if (++spins > (1ll << 25)) {
      atomicOr(err, 64);
      break;
    }
  }
  __threadfence_system();
}

__global__ void fold_clear_kernel(int* gate, int* pending_count) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && *gate) {
    *gate = 0;
    if (pending_count) *pending_count = 0;
  }
}

inline unsigned fold_shard_grid(int P) { return fold_grid(P); }  // blocks resident at once

// One sharded fold of u into every rank's D (enqueued on st, gated).
inline void fold_sharded(const FftPlan& p, const double* u, const FoldPeers& q, int* gate,
                         int* pending_count, int* err, cudaStream_t st) {
  const size_t smem = fold_smem(p.P);
  const unsigned g = fold_shard_grid(p.P);
  static bool attrs = false;
  if (!attrs) {
    const int sm = (int)fold_smem(8192);
    cudaFuncSetAttribute(fold_shard_r_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(fold_shard_c_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(fold_shard_i_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    attrs = true;
  }
  fold_shard_r_kernel<<<g, kFftThreads, smem, st>>>(p, u, q, q.rank, gate);
  fold_xbar_kernel<<<1, 32, 0, st>>>(q, gate, err);
  fold_shard_c_kernel<<<g, kFftThreads, smem, st>>>(p, q, q.rank, gate);
  fold_xbar_kernel<<<1, 32, 0, st>>>(q, gate, err);
  fold_shard_i_kernel<<<g, kFftThreads, smem, st>>>(p, q, q.rank, gate);
  fold_xbar_kernel<<<1, 32, 0, st>>>(q, gate, err);
  fold_clear_kernel<<<1, 32, 0, st>>>(gate, pending_count);
}

// The same decomposition with `world` ranks emulated one after another on
// this GPU (every "peer" buffer is the local one, no barriers: the phases
// run in order) -- checks the slab arithmetic on one GPU.
inline void fold_sharded_emulated(const FftPlan& p, const double* u, double* D, int world,
                                  int* gate, int* pending_count, cudaStream_t st) {
  FoldPeers q{};
  q.rank = 0;
  q.world = world;
  for (int r = 0; r < world; ++r) {
    q.W[r] = p.W;
    q.D[r] = D;
    q.bar[r] = nullptr;
  }
  const size_t smem = fold_smem(p.P);
  const unsigned g = fold_shard_grid(p.P);
  const int sm = (int)fold_smem(8192);
  cudaFuncSetAttribute(fold_shard_r_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(fold_shard_c_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(fold_shard_i_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  for (int r = 0; r < world; ++r) fold_shard_r_kernel<<<g, kFftThreads, smem, st>>>(p, u, q, r, gate);
  for (int r = 0; r < world; ++r) fold_shard_c_kernel<<<g, kFftThreads, smem, st>>>(p, q, r, gate);
  for (int r = 0; r < world; ++r) fold_shard_i_kernel<<<g, kFftThreads, smem, st>>>(p, q, r, gate);
  fold_clear_kernel<<<1, 32, 0, st>>>(gate, pending_count);
}

}  // namespace paqif
