// Software-pipelined AQIF level loop, FMA arithmetic: the latency form of
// aqif_warp.cuh's engine for the LCP batch (same lane map: one wing row per
// lane, 2*BETA lanes per system; same per-entry arithmetic, so the factors
// are bit-identical to aqif_factor_group<BETA, false>).
//
// Restates paqif/_kernels.py:62-149 (factor_batch) with the W solve of
// :152-172 fused.  What changes is the order of work inside a level.  The
// recurrence's critical chain is
//
//     pivot 2x2 of level k -> det -> reciprocal -> multipliers of the rows
//     that become level k+1's pivots -> their distance-1 entries -> pivot
//     2x2 of level k+1
//
// and everything else (the other distance columns of every wing row, the
// hand-off of the full pivot rows, the record, the hooks) only has to be
// done before the NEXT level's rank-2 update.  So each level first updates
// the distance-1 column of every row, passes the four entries that form the
// next pivot 2x2 from the two hand-off lanes by warp shuffles, and issues
// the next determinant and reciprocal; the bulk of the update, the hand-off
// through shared memory and the hooks are issued under that latency.  A
// level then costs about its instruction issue instead of the sum of its
// dependent latencies.
//
// Breakdown: not tested here (the LCP defers the level test to the Z solve
// and the corner system, which read every record: kDeferBreakdown).
#pragma once
#include "aqif_warp.cuh"

namespace paqif {

template <int BETA, class Pol>
__device__ void aqif_factor_pipe(Pol& pol, const int n, EngineSmem<BETA>& sm, const int gl,
                                 const bool alive)
{
  static_assert(Pol::kFuseW && !Pol::kResidual && !Pol::kRecordW && DeferBrkOf<Pol>::value,
                "pipelined engine: LCP policy (fused W, deferred breakdown test)");
  using A = Arith<false>;
  using PL = PivotLayout<BETA>;
  using HL = HookLayout<BETA>;
  constexpr int BP1 = BETA + 1;
  constexpr int G = Group<BETA>::G;
  constexpr unsigned FULL = 0xffffffffu;
  const int s = n / 2;
  const bool on = gl < 2 * BETA;
  const int side = on ? gl / BETA : 0;
  const int r = gl % BETA;
  const int step = side == 0 ? -BETA : BETA;
  const int own_off = side * 2 * BP1;  // zi(own_win, e, 0) = own_off + 2e
  const int crs_off = (1 - side) * 2 * BP1;
  const int gbase = (threadIdx.x & 31) & ~(G - 1);  // lane 0 of the group in the warp
  double* pbuf = sm.pbuf;

  double wo[BP1], wc[BP1];
  double rhs = 0.0;
  bool cur_pin = false;
  int row;

  HookPlan<BETA, G> hp;
  hp.init(pol, n, gl, alive);

  // ---------------------------------------------------------------- setup
  {
    const int rt = s - 1, rb = s;
    const int prow = side == 0 ? rt : rb;
    if (alive && on && imod(prow, BETA) == r) {
      double* pb = pbuf + 1 * PL::kSize;
#pragma unroll
      for (int e = 0; e < BP1; ++e) {
        pb[PL::zi(0, e, side)] = full_entry<BETA>(pol, n, prow, rt - e);
        pb[PL::zi(1, e, side)] = full_entry<BETA>(pol, n, prow, rb + e);
      }
      pb[side == 0 ? PL::kYT : PL::kYB] = !pol.pinned(prow) ? pol.frhs(prow) : 0.0;
    }
    row = side == 0 ? (rt - BETA) + imod(r - (rt - BETA), BETA)
                    : (rb + 1) + imod(r - (rb + 1), BETA);
    const bool ld = alive && on;
#pragma unroll
    for (int e = 0; e < BP1; ++e) {
      const double vl = ld ? full_entry<BETA>(pol, n, row, rt - e) : 0.0;
      const double vr = ld ? full_entry<BETA>(pol, n, row, rb + e) : 0.0;
      wo[e] = side == 0 ? vl : vr;
      wc[e] = side == 0 ? vr : vl;
    }
    const bool ok = ld && row >= 0 && row < n;
    cur_pin = ok && pol.pinned(row);
    rhs = (ok && !cur_pin) ? pol.frhs(row) : 0.0;
    for (int kk = 1; kk <= HOOK_AHEAD; ++kk) {
      hp.issue(sm, kk);
      cp_async_commit();
    }
  }
  __syncwarp();

  // level 1's pivot 2x2 and reciprocal
  double a11, a12, a21, a22, y;
  {
    const double2* pb2 = reinterpret_cast<const double2*>(pbuf + PL::kSize);
    const double2 c0 = pb2[PL::zi(0, 0, 0) / 2], c1 = pb2[PL::zi(1, 0, 0) / 2];
    a11 = c0.x;
    a21 = c0.y;
    a12 = c1.x;
    a22 = c1.y;
    y = __drcp_rn(A::det2(a11, a22, a21, a12));
  }

#ifdef PAQIF_ENGINE_PROF
  unsigned long long seg[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif
  for (int k = 1; k <= s; ++k) {
    ENG_T(t0);
    const int rt = s - k, rb = s + k - 1;
    const double* pb = pbuf + (k & 1) * PL::kSize;
    double* pbn = pbuf + ((k + 1) & 1) * PL::kSize;
    const double2* po = reinterpret_cast<const double2*>(pb + own_off);
    const double2* pc = reinterpret_cast<const double2*>(pb + crs_off);
    // the record of level k: loaded now, stored after the update
    constexpr int NP = PL::kSize / 2;
    constexpr int NR = (NP + G - 1) / G;
    double2 recv[NR];
#pragma unroll
    for (int t = 0; t < NR; ++t) {
      const int idx = gl + t * G;
      recv[t] = reinterpret_cast<const double2*>(pb)[idx < NP ? idx : 0];
    }
    if (k == s) {  // no wings left (rt == 0, rb == n-1): the record only
      if (alive) {
        double2* dst = reinterpret_cast<double2*>(pol.record_out(k));
#pragma unroll
        for (int t = 0; t < NR; ++t)
          if (gl + t * G < NP) dst[gl + t * G] = recv[t];
      }
      break;
    }
    // ---- critical chain: multipliers, distance-1 column, next pivot 2x2
    const double2 po1 = po[1], pc1 = pc[1];
    const double b1 = side == 0 ? wo[0] : wc[0];
    const double b2 = side == 0 ? wc[0] : wo[0];
    const double w1 = fma_mult(a22, b1, a21, b2, y);
    const double w2 = fma_mult(a11, b2, a12, b1, y);
    wo[0] = A::rank2(wo[1], w1, po1.x, w2, po1.y);
    wc[0] = A::rank2(wc[1], w1, pc1.x, w2, pc1.y);
    // rows rt-1 (top lane imod(rt-1, BETA)) and rb+1 (bottom lane
    // BETA + imod(rb+1, BETA)) are level k+1's pivots; their distance-0
    // entries of level k+1 are the values just computed
    const int lt = gbase + imod(rt - 1, BETA), lb = gbase + BETA + imod(rb + 1, BETA);
    const double n11 = __shfl_sync(FULL, wo[0], lt);  // A(rt-1, rt-1)
    const double n12 = __shfl_sync(FULL, wc[0], lt);  // A(rt-1, rb+1)
    const double n22 = __shfl_sync(FULL, wo[0], lb);  // A(rb+1, rb+1)
    const double n21 = __shfl_sync(FULL, wc[0], lb);  // A(rb+1, rt-1)
    // branch-free reciprocal (volatile asm start: the compiler keeps it
    // here, ahead of the work it overlaps, instead of sinking it to its use
    // at the top of the next level; no slow-path branch that would end the
    // basic block and with it the scheduler's freedom to interleave)
    const double yn = rcp_nobranch(A::det2(n11, n22, n21, n12));
    ENG_T(t1);
    // ---- this level's hooks (copied HOOK_AHEAD levels ago; the groups of
    // the next HOOK_AHEAD-1 levels may still be in flight), read before the
    // bulk update so their latency hides under it
    cp_async_wait<HOOK_AHEAD - 1>();
    __syncwarp();
    const double* hk = sm.hooks[k & (HOOK_RING - 1)] + side * HL::kSide;
    int m = side == 0 ? row - (rt - BETA) : (rb + BETA) - row;
    m = m < 0 ? 0 : (m > BETA - 1 ? BETA - 1 : m);
    const double hcol = hk[HL::kCol + m];
    const bool npin = reinterpret_cast<const uint32_t*>(hk + HL::kPin)[0] != 0u;
    const double nf = hk[HL::kF];
    double nrw[BP1];
    {
      const double2* h2 = reinterpret_cast<const double2*>(hk + HL::kRow);
#pragma unroll
      for (int e = 0; e + 1 < BP1; e += 2) {
        const double2 v = h2[e / 2];
        nrw[e] = v.x;
        nrw[e + 1] = v.y;
      }
      if (BP1 & 1) nrw[BP1 - 1] = hk[HL::kRow + BP1 - 1];
    }
    hp.issue(sm, k + HOOK_AHEAD);
    cp_async_commit();
    ENG_T(t2);
    // ---- off the chain: the rest of the update, right side, record
#pragma unroll
    for (int e = 2; e < BP1; ++e) {
      const double2 vo = po[e], vc = pc[e];
      wo[e - 1] = A::rank2(wo[e], w1, vo.x, w2, vo.y);
      wc[e - 1] = A::rank2(wc[e], w1, vc.x, w2, vc.y);
    }
    const double2 yy = reinterpret_cast<const double2*>(pb)[PL::kYT / 2];  // (yt, yb)
    const bool row_ok = alive & on & (row >= 0) & (row < n);
    {
      const double nr = fma_wsub(rhs, yy.x, w1, yy.y, w2);
      rhs = row_ok ? nr : rhs;
    }
#ifndef PAQIF_DEV_NO_RECORD
    if (alive) {
      double2* dst = reinterpret_cast<double2*>(pol.record_out(k));
#pragma unroll
      for (int t = 0; t < NR; ++t)
        if (gl + t * G < NP) dst[gl + t * G] = recv[t];
    }
#endif
    ENG_T(t3);
    ENG_T(t4);
    // the column entering at distance BETA: band value in the own window,
    // anti-band fill (zero) in the cross one
    wo[BETA] = (row_ok & !cur_pin) ? hcol : 0.0;
    wc[BETA] = 0.0;
    // ---- hand-off: the next pivot rows into the other pivot buffer, the
    // entering row from the hook
    const int nrow = side == 0 ? rt - 1 : rb + 1;
    ENG_T(t5);
    if (alive & on & (row == nrow)) {
      double* pno = pbn + own_off + side;
      double* pnc = pbn + crs_off + side;
#pragma unroll
      for (int e = 0; e < BP1; ++e) {
        pno[2 * e] = wo[e];
        pnc[2 * e] = wc[e];
      }
      pbn[side == 0 ? PL::kYT : PL::kYB] = rhs;
      row += step;
      cur_pin = npin;
      rhs = npin ? 0.0 : nf;
#pragma unroll
      for (int e = 0; e < BP1; ++e) {
        wo[e] = npin ? pinned_entry(e == BETA ? 0 : 1, nrw[BETA]) : nrw[e];
        wc[e] = 0.0;
      }
    }
    a11 = n11;
    a12 = n12;
    a21 = n21;
    a22 = n22;
    y = yn;
    ENG_T(t6);
    __syncwarp();
#ifdef PAQIF_ENGINE_PROF
    ENG_T(t7);
    seg[0] += t1 - t0; seg[1] += t2 - t1; seg[2] += t3 - t2; seg[3] += t4 - t3;
    seg[4] += t5 - t4; seg[5] += 1; seg[6] += t6 - t5; seg[7] += t7 - t6;
#endif
  }
#ifdef PAQIF_ENGINE_PROF
  if (gl == 0 && alive)
    for (int q = 0; q < 9; ++q) atomicAdd(&g_engine_seg[q], seg[q]);
#endif
  cp_async_wait<0>();
  __syncwarp();
}

}  // namespace paqif
