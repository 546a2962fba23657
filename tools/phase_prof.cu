// Dev tool: per-phase cycle split of the fused LCP kernel (factor / corner
// normal equations / Z solve / complementarity check) on config-2-shaped
// random systems.  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//   -DPAQIF_PROFILE_PHASES tools/phase_prof.cu -o phase_prof
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include "../paper_2008_03276_b200/csrc/lcp.cu"

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 4096;
  const int exact = argc > 2 ? atoi(argv[2]) : 1;
  const int n = 1026, beta = 8, nd = 2 * beta + 1;
  std::vector<double> bands((size_t)B * nd * n, 0.0), f((size_t)B * n, 0.0);
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-1, 1), U2(0.1, 1);
  std::normal_distribution<double> N(0, 1);
  for (int b = 0; b < B; ++b) {
    double* bd = &bands[(size_t)b * nd * n];
    for (int i = 0; i < n - 1; ++i) {
      double sum = 0;
      for (int d = -beta; d <= beta; ++d) {
        if (d == 0) continue;
        int j = i + d;
        if (j < 0 || j >= n - 1) continue;
        double v = U(rng);
        bd[(size_t)(d + beta) * n + i] = v;
        sum += fabs(v);
      }
      bd[(size_t)beta * n + i] = sum + U2(rng);
      f[(size_t)b * n + i] = N(rng);
    }
    bd[(size_t)beta * n + n - 1] = 1.0;
  }
  double *db, *df, *du, *dr; uint8_t* da; int64_t *dp, *ds; char* ws;
  size_t wsb = paqif_lcp_workspace_bytes(B, n, beta);
  cudaMalloc(&db, bands.size() * 8); cudaMalloc(&df, f.size() * 8);
  cudaMalloc(&du, f.size() * 8); cudaMalloc(&da, f.size()); cudaMalloc(&dp, B * 8);
  cudaMalloc(&dr, B * 8); cudaMalloc(&ds, B * 8); cudaMalloc(&ws, wsb);
  cudaMemcpy(db, bands.data(), bands.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(df, f.data(), f.size() * 8, cudaMemcpyHostToDevice);
  unsigned flags = exact ? PAQIF_FLAG_EXACT : 0;
  paqif_lcp_batch(B, n, beta, db, df, 1e-10, 100, flags, du, da, dp, dr, ds, ws, wsb, 0);
  cudaDeviceSynchronize();
  unsigned long long zero[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbol(g_phase_cycles, zero, sizeof(zero));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  paqif_lcp_batch(B, n, beta, db, df, 1e-10, 100, flags, du, da, dp, dr, ds, ws, wsb, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc[4];
  cudaMemcpyFromSymbol(cyc, g_phase_cycles, sizeof(cyc));
  std::vector<int64_t> passes(B);
  cudaMemcpy(passes.data(), dp, B * 8, cudaMemcpyDeviceToHost);
  double mp = 0; for (auto p : passes) mp += p; mp /= B;
  double tot = cyc[0] + cyc[1] + cyc[2] + cyc[3];
  printf("B=%d exact=%d ms=%.3f passes=%.3f | per system-pass kcycles: factor %.1f corner %.1f zsolve %.1f check %.1f | shares %.2f %.2f %.2f %.2f (%s)\n",
         B, exact, ms, mp, cyc[0] / (B * mp) / 1e3, cyc[1] / (B * mp) / 1e3, cyc[2] / (B * mp) / 1e3,
         cyc[3] / (B * mp) / 1e3, cyc[0] / tot, cyc[1] / tot, cyc[2] / tot, cyc[3] / tot,
         cudaGetErrorString(cudaGetLastError()));
#ifdef PAQIF_ENGINE_PROF
  unsigned long long sg[9];
  cudaMemcpyFromSymbol(sg, g_engine_seg, sizeof(sg));
  const double L = sg[5] ? (double)sg[5] : 1.0;
  printf("  engine cycles/level (pipe: chain, bulk, rec+hooks, hookwait, hookread, handoff, sync; row engine: head, div, update, hookwait, shift, -, handoff, syncwarp): %.0f %.0f %.0f %.0f %.0f %.0f %.0f (levels %llu)\n",
         sg[0] / L, sg[1] / L, sg[2] / L, sg[3] / L, sg[4] / L, sg[6] / L, sg[7] / L, sg[5]);
#endif
  return 0;
}
