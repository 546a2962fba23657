// Microbenchmarks for the roofline denominators MEASURED_PEAKS.json lacks:
// fp64 DFMA throughput and L2-resident read bandwidth (plus an HBM copy
// cross-check).  nvcc -O3 -gencode arch=compute_100a,code=sm_100a peaks.cu -o peaks
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 1.2345) out[threadIdx.x] = s;
}

__global__ void read_kernel(const double2* __restrict__ p, size_t n, int reps, double* out) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(p + i);
      acc += v.x + v.y;
    }
  if (acc == 1.2345) out[0] = acc;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // DFMA
  const int iters = 4096, threads = 256, blocks = sms * 8;
  dfma_kernel<<<blocks, threads>>>(out, 16, 0.999, 1e-3);
  cudaEventRecord(e0);
  dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 64 * (double)iters * threads * blocks;
  printf("{\"dfma_tflops\": %.3f, ", flops / (ms * 1e-3) / 1e12);
  // L2-resident read: 48 MB buffer, many repetitions
  size_t nl2 = (48ull << 20) / 16;
  double2* buf;
  cudaMalloc(&buf, 2ull << 30);
  cudaMemset(buf, 0, 2ull << 30);
  read_kernel<<<sms * 8, 512>>>(buf, nl2, 2, out);
  cudaEventRecord(e0);
  read_kernel<<<sms * 8, 512>>>(buf, nl2, 20, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("\"l2_read_gbs\": %.1f, ", 20.0 * nl2 * 16 / (ms * 1e-3) / 1e9);
  // HBM read of 1 GB
  size_t nh = (1ull << 30) / 16;
  cudaEventRecord(e0);
  read_kernel<<<sms * 8, 512>>>(buf, nh, 1, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("\"hbm_read_gbs\": %.1f, ", nh * 16 / (ms * 1e-3) / 1e9);
  // HBM copy 1 GB -> 1 GB (read + write bytes)
  copy_kernel<<<sms * 8, 512>>>(buf, buf + nh, nh);
  cudaEventRecord(e0);
  copy_kernel<<<sms * 8, 512>>>(buf, buf + nh, nh);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("\"hbm_copy_gbs\": %.1f, \"sms\": %d}\n", 2.0 * nh * 16 / (ms * 1e-3) / 1e9, sms);
  return 0;
}
