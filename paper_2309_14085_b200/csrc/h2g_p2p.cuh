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
#include "h2g_stream.cuh"

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
#ifndef H2G_P2P_STAGE_BYTES
#define H2G_P2P_STAGE_BYTES 4096
#endif
constexpr int kP2PStageBytes = H2G_P2P_STAGE_BYTES;       // one stage slot
constexpr int kP2PSlotsPerWarp = 2;                       // stages in flight per warp
constexpr int kP2PSlots = kP2PSlotsPerWarp * kP2PWarps;   // slot ring per CTA
// dynamic smem of the P2P kernel: stage slots + the chunk buffers + the
// cross-warp reduction + mbarriers
constexpr size_t kP2PSmem = (size_t)kP2PSlots * kP2PStageBytes +
                            (size_t)kP2PWarps * 2 * kP2PChunk * (sizeof(double) * 4 + 8) +
                            (size_t)kP2PWarps * kMaxRows * 8 + (size_t)kP2PSlots * 8 + 16;

// Host-built work lists of the P2P engine (from the Task/Term schedule):
struct P2PTask {       // 40 bytes
  int64_t y_off;       // arena slot of y[0]
  int32_t m;           // rows (<= kMaxRows)
  int32_t row_rec;     // record of row 0
  int32_t t_begin;     // stored GEMV terms [t_begin, t_end) of the Term table (direct loads)
  int32_t t_end;
  int32_t k_begin;     // evaluated chunks [k_begin, k_end) of the chunk table
  int32_t k_end;
  int32_t s_begin;     // TMA-staged stored columns [s_begin, s_end) of the stage table
  int32_t s_end;
};

// STAGED stored data: the stored blocks of a task with contiguous columns
// (lda == m: stored M2L blocks, L2L, L2P, BLR U, near) are cut into stages of
// <= kP2PStageBytes, each ONE cp.async.bulk into a per-warp smem slot, issued
// ahead and consumed between the warp's evaluated chunks -- so HBM streams
// while the fp64 pipe evaluates (m2l_recompute_share < 1: a share of every
// target's M2L blocks is read, the rest evaluated).
struct P2PStage {      // 24 bytes
  uint64_t src;        // 16-byte aligned global address of the copy
  int64_t x_off;       // arena slot of x for column 0
  uint32_t bytes;      // copy bytes (multiple of 16)
  int16_t ncols;       // columns (of m rows, column-major, contiguous)
  int16_t shift;       // A(0, 0) at slot + shift doubles
};

struct P2PChunk {      // 16 bytes: <= 32 columns of one evaluated block
  int64_t x_off;       // arena slot of x for column 0
  int32_t rec;         // record of column 0
  int32_t n_self;      // columns | kSelfBit (row and column runs share points)
};

__device__ __forceinline__ void issue_stage(const P2PStage& st, double* slot, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot done
  mbar_arrive_expect_tx(bar, st.bytes);
  bulk_g2s(slot, reinterpret_cast<const void*>(st.src), st.bytes, bar);
}

// FULL: the phase has self blocks (near diagonal) or coincident points (the
// r == 0 test in every entry); M2L phases of distinct points run the plain
// evaluation loop only -- a third of the code (the dispatch instantiates
// every L x J layout, and instruction fetch was a top stall at the leaf level).
template <int KT, int DIM, int L, int J, bool FULL>
__device__ __forceinline__ void p2p_task(const P2PTask& tk, const Term* __restrict__ terms,
                                         const P2PChunk* __restrict__ chunks,
                                         const P2PStage* __restrict__ stages,
                                         const double4* __restrict__ recs,
                                         const double* __restrict__ blob, double* arena,
                                         const P2PKernel& kp, double4 (*srec)[kP2PChunk],
                                         double (*sx)[kP2PChunk], double* red, double* slots,
                                         uint64_t* sbar, uint32_t& sphase, int lane, int warp) {
  constexpr int G = 32 / L;
  const int g = lane / L, rl = lane % L;
  const int m = tk.m;
  // stages of this warp: s = s_begin + warp + kP2PWarps i, in slot
  // warp + kP2PWarps (i % kP2PSlotsPerWarp); the first ones go out now
  const int n_st = tk.s_end - tk.s_begin;
  if (lane == 0)
    for (int i = 0; i < kP2PSlotsPerWarp; ++i) {
      const int si = warp + kP2PWarps * i;
      if (si < n_st) {
        const int sl = warp + kP2PWarps * i;
        issue_stage(stages[tk.s_begin + si], slots + (size_t)sl * (kP2PStageBytes / 8), &sbar[sl]);
      }
    }
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
  int my_si = warp;  // next stage of this warp (index into the task's stages)
  int my_i = 0;      // its ordinal among the warp's stages (slot = my_i % kP2PSlotsPerWarp)
  // one staged stored block: columns dealt over the lane groups, rows over
  // the lanes of a group (the layout of the evaluated chunks)
  auto consume_stage = [&]() {
    const int sl = warp + kP2PWarps * (my_i % kP2PSlotsPerWarp);
    const P2PStage st = stages[tk.s_begin + my_si];
    mbar_wait(&sbar[sl], (sphase >> sl) & 1u);
    sphase ^= 1u << sl;
    const double* A = slots + (size_t)sl * (kP2PStageBytes / 8) + st.shift;
    const double* x = arena + st.x_off;
    const int nc = st.ncols;
#pragma unroll 2
    for (int c = g; c < nc; c += G) {
      const double xv = x[c];
      const double* col = A + c * m;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int r = rl + L * j;
        if (r < m) acc[j] = fma(col[r], xv, acc[j]);
      }
    }
    __syncwarp();
    const int nxt = my_si + kP2PWarps * kP2PSlotsPerWarp;
    if (lane == 0 && nxt < n_st)
      issue_stage(stages[tk.s_begin + nxt], slots + (size_t)sl * (kP2PStageBytes / 8), &sbar[sl]);
    my_si += kP2PWarps;
    ++my_i;
  };
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
    if (FULL && self) {
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
    } else if (FULL && kp.check) {
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
    if (my_si < n_st) consume_stage();  // one staged block between evaluated chunks
  }
  while (my_si < n_st) consume_stage();
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

template <int KT, int DIM, bool FULL>
__device__ __forceinline__ void p2p_dispatch(const P2PTask& tk, const Term* __restrict__ terms,
                                             const P2PChunk* __restrict__ chunks,
                                             const P2PStage* __restrict__ stages,
                                             const double4* __restrict__ recs,
                                             const double* __restrict__ blob, double* arena,
                                             const P2PKernel& kp, double4 (*srec)[kP2PChunk],
                                             double (*sx)[kP2PChunk], double* red, double* slots,
                                             uint64_t* sbar, uint32_t& sphase, int lane,
                                             int warp) {
  const int m = tk.m;
  constexpr int JT = kP2PRowsPerLane;
  int L = 4;
  while (L < 32 && L * JT < m) L <<= 1;
  const int J = (m + L - 1) / L;
#define H2G_P2P(Lv, Jv)                                                                     \
  p2p_task<KT, DIM, Lv, Jv, FULL>(tk, terms, chunks, stages, recs, blob, arena, kp, srec, sx, red, \
                            slots, sbar, sphase, lane, warp)
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
template <int KT, int DIM, bool FULL>
__global__ void __launch_bounds__(kP2PThreads, kP2PCtasPerSm)
p2p_tasks_kernel(const P2PTask* __restrict__ tasks, int n_tasks, const Term* __restrict__ terms,
                 const P2PChunk* __restrict__ chunks, const P2PStage* __restrict__ stages,
                 const double4* __restrict__ recs, const double* __restrict__ blob,
                 double* arena, P2PKernel kp, int* ctr) {
  extern __shared__ __align__(128) double p2p_smem[];
  double* slots = p2p_smem;  // kP2PSlots x kP2PStageBytes
  auto srec = reinterpret_cast<double4 (*)[2][kP2PChunk]>(slots + kP2PSlots * (kP2PStageBytes / 8));
  auto sx = reinterpret_cast<double (*)[2][kP2PChunk]>(srec + kP2PWarps);
  double* red = reinterpret_cast<double*>(sx + kP2PWarps);
  uint64_t* sbar = reinterpret_cast<uint64_t*>(red + kP2PWarps * kMaxRows);
  int* s_task = reinterpret_cast<int*>(sbar + kP2PSlots);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kP2PSlots; ++i) mbar_init(&sbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t sphase = 0;  // parity of every slot's barrier (bit per slot; a warp touches its own)
  griddep_launch_dependents();
  griddep_wait();  // x (and the counters' reset) come from earlier phases
  for (;;) {
    if (threadIdx.x == 0) *s_task = atomicAdd(ctr, 1);
    __syncthreads();
    const int t = *s_task;
    if (t >= n_tasks) break;
    const P2PTask tk = tasks[t];
    p2p_dispatch<KT, DIM, FULL>(tk, terms, chunks, stages, recs, blob, arena, kp, srec[warp], sx[warp],
                          red, slots, sbar, sphase, lane, warp);
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
