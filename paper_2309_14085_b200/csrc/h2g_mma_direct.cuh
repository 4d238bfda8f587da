// h2g_mma_direct.cuh — batched-RHS engine, direct-load variant (sm_100a).
//
// Y (m x KB) = sum_terms A (m x ncols) X (ncols x KB) on the fp64 tensor pipe
// (mma.sync m8n8k4 f64), with the A fragments loaded straight from global
// memory: an operator entry is used by exactly one lane of one DMMA, so the
// pass through shared memory (TMA ring -> LDS) buys no reuse and, for
// m = 64, costs a 4-way bank conflict on every A fragment
// (profiles/ncu_r02_mma_summary.md).  Latency is hidden by a register queue
// of kDirectDepth k-steps per warp and 16 warps per SM (no shared memory).
//
// STATUS: experimental, off by default (H2G_MMA_DIRECT=1 selects it for the
// wide phases).  Parity-tested, but measured 1.65x SLOWER than the TMA-ring
// engine on cfg 2 with 16 RHS (2.84 vs 1.72 ms per pass; leaf phase 1.15 vs
// 0.63 ms): 16 warps x 2 k-steps of 8-byte loads keep ~12 KB per SM in
// flight where the HBM rate needs ~45 KB, and deeper queues (3, 4, 6
// k-steps) spill.  Kept as the measured baseline for that design.
//
// Work item = (task, up to 4 consecutive 8-row tiles); warps take items from
// a per-launch counter.  X fragments come from the batched arena through L1
// (the row groups of a task share them).  Deterministic: one warp computes a
// row group over the task's terms in order; no atomics on data.
#pragma once
#include <cstdint>

#include "h2g_kernels.cuh"

namespace h2g {

#ifndef H2G_DIRECT_DEPTH
#define H2G_DIRECT_DEPTH 2   // deeper queues spill at 4 CTAs per SM and lose (measured)
#endif
#ifndef H2G_MMA_DIRECT
#define H2G_MMA_DIRECT 0
#endif
constexpr bool kMmaDirectDefault = H2G_MMA_DIRECT != 0;  // env H2G_MMA_DIRECT overrides
constexpr int kDirectDepth = H2G_DIRECT_DEPTH;  // k-steps in flight per warp
constexpr int kDirectWarps = 4;                 // warps per CTA
#ifndef H2G_DIRECT_CTAS
#define H2G_DIRECT_CTAS 4
#endif
constexpr int kDirectCtasPerSm = H2G_DIRECT_CTAS;
constexpr int kDirectTiles = 4;                 // 8-row tiles per item (at most)

struct DItem {        // 8 bytes
  int32_t task;       // index into the batched schedule's tasks
  int16_t tile0;      // first 8-row tile
  int16_t ntile;      // tiles (1..kDirectTiles)
};

__device__ __forceinline__ void dmma_d(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int TPW, int NT>
__device__ __forceinline__ void direct_item(const Task& t, int tile0, const Term* __restrict__ terms,
                                            const double* __restrict__ blob,
                                            double* __restrict__ arena, int64_t ps, int lane) {
  constexpr int D = kDirectDepth;
  const int kq = lane & 3, rq = lane >> 2;
  const int m = t.m;
  bool rok[TPW];
#pragma unroll
  for (int i = 0; i < TPW; ++i) rok[i] = 8 * (tile0 + i) + rq < m;
  double c[TPW][NT][2];
#pragma unroll
  for (int i = 0; i < TPW; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) c[i][nt][0] = c[i][nt][1] = 0.0;

  // term headers as two 16-byte vectors (kept in registers), one term ahead
  longlong2 n_ax = make_longlong2(0, 0);  // a_off, x_off
  int4 n_i = make_int4(0, 0, 0, 0);       // lda, ncols, a_space, pad
  if (t.t_begin < t.t_end) {
    n_ax = __ldg(reinterpret_cast<const longlong2*>(terms + t.t_begin));
    n_i = __ldg(reinterpret_cast<const int4*>(terms + t.t_begin) + 1);
  }
  for (int k = t.t_begin; k < t.t_end; ++k) {
    const longlong2 ax = n_ax;
    const int4 ti = n_i;
    if (k + 1 < t.t_end) {
      n_ax = __ldg(reinterpret_cast<const longlong2*>(terms + k + 1));
      n_i = __ldg(reinterpret_cast<const int4*>(terms + k + 1) + 1);
    }
    const int ncols = ti.y;
    const int nks = (ncols + 3) >> 2;
    const int64_t lda = ti.x;
    const double* Ap = (ti.z ? arena : blob) + ax.x + kq * lda + 8 * tile0 + rq;
    const double* Xp = arena + (ax.y + kq) * 8 + rq;
    double a[D][TPW], b[D][NT];
    // load cursor: k-steps are loaded strictly in order, so the addresses
    // are two running pointers and a remaining-column count
    const double* Al = Ap;
    const double* Xl = Xp;
    const int64_t adv_a = 4 * lda;
    int left = ncols - kq;  // > 0: this lane's column of the next k-step exists
    auto load = [&](int slot) {
      const bool ok = left > 0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) b[slot][nt] = ok ? __ldg(Xl + nt * ps) : 0.0;
#pragma unroll
      for (int i = 0; i < TPW; ++i) a[slot][i] = (ok && rok[i]) ? ld_stream(Al + 8 * i) : 0.0;
      Al += adv_a;
      Xl += 32;
      left -= 4;
    };
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (d < nks) load(d);
    for (int j0 = 0; j0 < nks; j0 += D) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        if (j0 + d < nks) {
#pragma unroll
          for (int i = 0; i < TPW; ++i)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma_d(c[i][nt], a[d][i], b[d][nt]);
          if (j0 + d + D < nks) load(d);
        }
      }
    }
  }
  double* y = arena + t.y_off * 8;
#pragma unroll
  for (int i = 0; i < TPW; ++i) {
    const int row = 8 * (tile0 + i) + rq;
    if (row < m)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        *reinterpret_cast<double2*>(y + nt * ps + (int64_t)row * 8 + 2 * kq) =
            make_double2(c[i][nt][0], c[i][nt][1]);
  }
}

template <int KB>
__global__ void __launch_bounds__(32 * kDirectWarps, kDirectCtasPerSm)
direct_mma_kernel(const DItem* __restrict__ items, int n_items, const Task* __restrict__ tasks,
                  const Term* __restrict__ terms, const double* __restrict__ blob,
                  double* __restrict__ arena, int64_t ps, int* __restrict__ counter) {
  constexpr int NT = KB / 8;
  const int lane = threadIdx.x & 31;
  while (true) {
    int it = 0;
    if (lane == 0) it = atomicAdd(counter, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= n_items) break;
    const DItem di = items[it];
    const Task t = tasks[di.task];
    switch (di.ntile) {
      case 1: direct_item<1, NT>(t, di.tile0, terms, blob, arena, ps, lane); break;
      case 2: direct_item<2, NT>(t, di.tile0, terms, blob, arena, ps, lane); break;
      case 3: direct_item<3, NT>(t, di.tile0, terms, blob, arena, ps, lane); break;
      default: direct_item<4, NT>(t, di.tile0, terms, blob, arena, ps, lane); break;
    }
  }
}

}  // namespace h2g
