// h2g_p2p.cuh — kernel-evaluation ("recompute", P2P-style) engine (sm_100a).
//
// In the NCA construction the M2L coupling blocks are raw kernel blocks,
// m2l[(X, Y)] = K[t_i(X), s_o(Y)] (reference engine.py:176-179), and the
// near blocks are K[t^X, t^Y] (engine.py:309-318; the reference itself can
// evaluate them lazily, store_near=False).  Streaming them costs 8 bytes of
// HBM per entry; evaluating them costs ~12 fp64 instructions per entry,
// which on B200 (64 DFMA/clk/SM, measured tools/ubench_fp64.cu) is ~1.45x
// faster than the 6.55 TB/s copy roofline for 1/r, and needs no storage
// (the only way to hold BASELINE config 5, whose stored M2L+near exceed HBM).
//
// The plan builds, from its regular Task/Term schedule, a P2P task per
// output slice: rows = a run of point RECORDS (double4 x, y, z, -), stored
// GEMV terms (L2L, L2P, BLR U, ...) and a list of evaluated CHUNKS, each
// <= 32 columns of one kernel-evaluated block: records [rec, rec + n) times
// x = arena[x_off ...], flagged "self" when row and column runs may share
// points (near diagonal blocks).  Entry rule = Kernel.block
// (kernels.py:36-57): i == j -> (diag if set else zero_value) + shift;
// r == 0, i != j -> zero_value; else f(r).
//
// Mapping: one CTA (kP2PWarps warps) per task, fetched dynamically from a
// per-launch counter; chunk k of a task belongs to warp k % kP2PWarps.
// Inside a warp, lanes form G = 32 / L groups of L; lane (g, l) owns rows
// l + L j (j < J) and the chunk's columns g, g + G, ...  Groups are combined
// by a fixed xor-shuffle tree, warps in warp order through smem: the
// summation order is fixed (deterministic, no atomics on data).  Column
// records + x values are staged through a per-warp smem double buffer (the
// warp's next chunk in flight while the current one is evaluated).
#pragma once
#include <cstdint>

#include "h2g_eval.cuh"
#include "h2g_kernels.cuh"

namespace h2g {

#ifndef H2G_P2P_WARPS
#define H2G_P2P_WARPS 4
#endif
#ifndef H2G_P2P_CTAS
#define H2G_P2P_CTAS 4
#endif
constexpr int kP2PWarps = H2G_P2P_WARPS;  // warps per CTA (one task per CTA)
constexpr int kP2PCtasPerSm = H2G_P2P_CTAS;
#ifndef H2G_P2P_HYBRID_CTAS
#define H2G_P2P_HYBRID_CTAS 2
#endif
// P2P CTAs per SM beside one streaming-engine CTA (hybrid phases): 2 x 128
// threads x 128 registers + 160 x 168 fit the 64K-register file
constexpr int kP2PHybridCtas = H2G_P2P_HYBRID_CTAS;
constexpr int kP2PThreads = 32 * kP2PWarps;
constexpr int kP2PChunk = 32;
constexpr int kRecompute = 2;  // Term.a_space of a kernel-evaluated block (host schedule)
constexpr int kSelfBit = 1 << 16;

// Host-built work lists of the P2P engine (from the Task/Term schedule):
struct P2PTask {       // 32 bytes
  int64_t y_off;       // arena slot of y[0]
  int32_t m;           // rows (<= kMaxRows)
  int32_t row_rec;     // record of row 0
  int32_t t_begin;     // stored GEMV terms [t_begin, t_end) of the Term table
  int32_t t_end;
  int32_t k_begin;     // evaluated chunks [k_begin, k_end) of the chunk table
  int32_t k_end;
};

struct P2PChunk {      // 16 bytes: <= 32 columns of one evaluated block
  int64_t x_off;       // arena slot of x for column 0
  int32_t rec;         // record of column 0
  int32_t n_self;      // columns | kSelfBit (row and column runs share points)
};

template <int KT, int DIM, int L, int J>
__device__ __forceinline__ void p2p_task(const P2PTask& tk, const Term* __restrict__ terms,
                                         const P2PChunk* __restrict__ chunks,
                                         const double4* __restrict__ recs,
                                         const double* __restrict__ blob, double* arena,
                                         const P2PKernel& kp, double4 (*srec)[kP2PChunk],
                                         double (*sx)[kP2PChunk], double* red, int lane,
                                         int warp) {
  constexpr int G = 32 / L;
  const int g = lane / L, rl = lane % L;
  const int m = tk.m;
  const int64_t row0 = tk.row_rec;
  double px[J], py[J], pz[J], acc[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int r = min(rl + L * j, m - 1);
    const double4 p = recs[row0 + r];
    px[j] = p.x;
    py[j] = p.y;
    pz[j] = p.z;
    acc[j] = 0.0;
  }
  // stored terms are read after the evaluation: start pulling them into L2 now
  if (warp == 0)
    for (int t = tk.t_begin + lane; t < tk.t_end; t += 32) {
      const Term tm = terms[t];
      if (tm.ncols > 0)
        prefetch_l2((tm.a_space ? arena : blob) + tm.a_off,
                    8ull * ((uint64_t)(tm.ncols - 1) * tm.lda + m));
    }
  // ---- evaluated chunks k = k_begin + warp, + kP2PWarps, ...: the next
  // chunk's records / x are loaded (registers) while the current one is
  // evaluated from the warp's smem buffer
  int k = tk.k_begin + warp;
  P2PChunk cd{};
  double4 nrec = make_double4(0, 0, 0, 0);
  double nx = 0.0;
  if (k < tk.k_end) {
    cd = chunks[k];
    if (lane < (cd.n_self & 0xffff)) {
      nrec = recs[cd.rec + lane];
      nx = arena[cd.x_off + lane];
    }
  }
  int buf = 0;
  while (k < tk.k_end) {
    const int n = cd.n_self & 0xffff;
    const bool self = (cd.n_self & kSelfBit) != 0;
    const int64_t col0 = cd.rec;  // record index of column 0 (self test)
    srec[buf][lane] = nrec;
    sx[buf][lane] = nx;
    __syncwarp();
    k += kP2PWarps;
    if (k < tk.k_end) {  // next chunk's loads in flight during the evaluation
      cd = chunks[k];
      if (lane < (cd.n_self & 0xffff)) {
        nrec = recs[cd.rec + lane];
        nx = arena[cd.x_off + lane];
      }
    }
    if (self) {
      for (int c = g; c < n; c += G) {
        const double4 s = srec[buf][c];
        const double xv = sx[buf][c];
        const int64_t ci = col0 + c;
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const double r2 = dist2<DIM>(px[j], py[j], pz[j], s);
          double kv = kfun<KT>(r2, kp);
          kv = r2 == 0.0 ? kp.zero_value : kv;
          kv = (row0 + rl + L * j == ci) ? kp.self_value : kv;
          acc[j] = fma(kv, xv, acc[j]);
        }
      }
    } else if (kp.check) {
#pragma unroll 2
      for (int c = g; c < n; c += G) {
        const double4 s = srec[buf][c];
        const double xv = sx[buf][c];
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const double r2 = dist2<DIM>(px[j], py[j], pz[j], s);
          double kv = kfun<KT>(r2, kp);
          kv = r2 == 0.0 ? kp.zero_value : kv;
          acc[j] = fma(kv, xv, acc[j]);
        }
      }
    } else {
#pragma unroll 2
      for (int c = g; c < n; c += G) {
        const double4 s = srec[buf][c];
        const double xv = sx[buf][c];
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const double r2 = dist2<DIM>(px[j], py[j], pz[j], s);
          acc[j] = fma(kfun<KT>(r2, kp), xv, acc[j]);
        }
      }
    }
    buf ^= 1;
  }
  // ---- stored terms (L2L, L2P, BLR U, stored blocks): columns dealt over
  // (warp, lane group) pairs, direct coalesced loads down each column
  for (int t = tk.t_begin; t < tk.t_end; ++t) {
    const Term tm = terms[t];
    const double* A = (tm.a_space ? arena : blob) + tm.a_off;
    const double* x = arena + tm.x_off;
#pragma unroll 2
    for (int c = warp * G + g; c < tm.ncols; c += kP2PWarps * G) {
      const double xv = x[c];
      const double* col = A + (int64_t)c * tm.lda;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int r = rl + L * j;
        if (r < m) acc[j] = fma(ld_stream(col + r), xv, acc[j]);
      }
    }
  }
  // ---- combine: lane groups by a fixed xor tree, then the warps in warp
  // order through smem; one store per row
#pragma unroll
  for (int j = 0; j < J; ++j)
#pragma unroll
    for (int off = L; off < 32; off <<= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
  if (g == 0) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int r = rl + L * j;
      if (r < m) red[warp * kMaxRows + r] = acc[j];
    }
  }
  __syncthreads();
  double* y = arena + tk.y_off;
  for (int r = threadIdx.x; r < m; r += kP2PThreads) {
    double sum = red[r];
#pragma unroll
    for (int w = 1; w < kP2PWarps; ++w) sum += red[w * kMaxRows + r];
    y[r] = sum;
  }
}

// rows-per-lane layout for m rows: J ~ kP2PRowsPerLane independent row
// chains per lane, L = clamp(pow2ceil(ceil(m / JT)), 4, 32) lanes per column
// group, J = ceil(m / L) (<= 8 since m <= kMaxRows = 256)
#ifndef H2G_P2P_JT
#define H2G_P2P_JT 8
#endif
constexpr int kP2PRowsPerLane = H2G_P2P_JT;

template <int KT, int DIM>
__device__ __forceinline__ void p2p_dispatch(const P2PTask& tk, const Term* __restrict__ terms,
                                             const P2PChunk* __restrict__ chunks,
                                             const double4* __restrict__ recs,
                                             const double* __restrict__ blob, double* arena,
                                             const P2PKernel& kp, double4 (*srec)[kP2PChunk],
                                             double (*sx)[kP2PChunk], double* red, int lane,
                                             int warp) {
  const int m = tk.m;
  constexpr int JT = kP2PRowsPerLane;
  int L = 4;
  while (L < 32 && L * JT < m) L <<= 1;
  const int J = (m + L - 1) / L;
#define H2G_P2P(Lv, Jv)                                                                     \
  p2p_task<KT, DIM, Lv, Jv>(tk, terms, chunks, recs, blob, arena, kp, srec, sx, red, lane, \
                            warp)
#define H2G_P2P_J(Lv)                                                  \
  switch (J) {                                                         \
    case 1: if constexpr (Lv == 4) { H2G_P2P(Lv, 1); } else { __trap(); } break;          \
    case 2: if constexpr (Lv == 4) { H2G_P2P(Lv, 2); } else { __trap(); } break;          \
    case 3: if constexpr (Lv == 4 || JT <= 4) { H2G_P2P(Lv, 3); } else { __trap(); } break; \
    case 4: H2G_P2P(Lv, 4); break;                                     \
    case 5: if constexpr (JT > 4 || Lv == 32) { H2G_P2P(Lv, 5); } else { __trap(); } break; \
    case 6: if constexpr (JT > 4 || Lv == 32) { H2G_P2P(Lv, 6); } else { __trap(); } break; \
    case 7: if constexpr (JT > 4 || Lv == 32) { H2G_P2P(Lv, 7); } else { __trap(); } break; \
    default: if constexpr (JT > 4 || Lv == 32) { H2G_P2P(Lv, 8); } else { __trap(); } break; \
  }
  if (L == 4) {
    H2G_P2P_J(4)
  } else if (L == 8) {
    H2G_P2P_J(8)
  } else if (L == 16) {
    H2G_P2P_J(16)
  } else {
    H2G_P2P_J(32)
  }
#undef H2G_P2P_J
#undef H2G_P2P
}

// One CTA per task, fetched dynamically from ctr[0] (largest tasks first, the
// host sorts them); the last CTA to leave resets the counters for the next
// launch (graph replays reuse them).  Counters schedule work only: every
// output is written once, in a fixed summation order.
template <int KT, int DIM>
__global__ void __launch_bounds__(kP2PThreads, kP2PCtasPerSm)
p2p_tasks_kernel(const P2PTask* __restrict__ tasks, int n_tasks, const Term* __restrict__ terms,
                 const P2PChunk* __restrict__ chunks, const double4* __restrict__ recs,
                 const double* __restrict__ blob, double* arena, P2PKernel kp, int* ctr) {
  __shared__ double4 srec[kP2PWarps][2][kP2PChunk];
  __shared__ double sx[kP2PWarps][2][kP2PChunk];
  __shared__ double red[kP2PWarps * kMaxRows];
  __shared__ int s_task;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  griddep_launch_dependents();
  griddep_wait();  // x (and the counters' reset) come from earlier phases
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(ctr, 1);
    __syncthreads();
    const int t = s_task;
    if (t >= n_tasks) break;
    const P2PTask tk = tasks[t];
    p2p_dispatch<KT, DIM>(tk, terms, chunks, recs, blob, arena, kp, srec[warp], sx[warp], red,
                          lane, warp);
    __syncthreads();  // red / s_task reuse
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      __threadfence();
    }
  }
}

}  // namespace h2g
