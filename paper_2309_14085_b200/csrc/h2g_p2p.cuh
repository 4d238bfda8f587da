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
// Mapping: one CTA per task, fetched dynamically from a per-launch counter;
// kP2PWarps EVALUATION warps (chunk k of a task belongs to warp k %
// kP2PWarps) and, in phases whose tasks also read stored blocks through TMA
// stages, one STREAMING warp that owns the CTA's stage slots and multiplies
// the staged blocks while the evaluation warps keep the fp64 pipe busy.
// Inside a warp, lanes form G = 32 / L groups of L; lane (g, l) owns rows
// l + L j (j < J) and the chunk's columns g, g + G, ...  Groups are combined
// by a fixed xor-shuffle tree, warps in warp order through smem: the
// summation order is fixed (deterministic, no atomics on data).  Column
// records + x values are staged through a per-warp smem double buffer (the
// warp's next chunk in flight while the current one is evaluated).
#pragma once
#include <algorithm>
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
#ifndef H2G_P2P_WARPS_SW
#define H2G_P2P_WARPS_SW 3
#endif
#ifndef H2G_P2P_CTAS_SW
#define H2G_P2P_CTAS_SW 4
#endif
constexpr int kP2PWarps = H2G_P2P_WARPS;      // evaluation warps per CTA (one task per CTA)
constexpr int kP2PCtasPerSm = H2G_P2P_CTAS;   // CTAs per SM without a streaming warp
constexpr int kP2PWarpsSW = H2G_P2P_WARPS_SW; // evaluation warps beside a streaming warp
constexpr int kP2PCtasSW = H2G_P2P_CTAS_SW;   // CTAs per SM of that shape
#ifndef H2G_P2P_HYBRID_CTAS
#define H2G_P2P_HYBRID_CTAS 2
#endif
// P2P CTAs per SM beside one streaming-engine CTA (hybrid phases): 2 x 128
// threads x 128 registers + 160 x 168 fit the 64K-register file
constexpr int kP2PHybridCtas = H2G_P2P_HYBRID_CTAS;
constexpr int kP2PThreads = 32 * kP2PWarps;
constexpr int kP2PThreadsSW = 32 * (kP2PWarpsSW + 1);
constexpr int kP2PChunk = 32;
constexpr int kRecompute = 2;  // Term.a_space of a kernel-evaluated block (host schedule)
constexpr int kSelfBit = 1 << 16;
#ifndef H2G_P2P_STAGE_BYTES
#define H2G_P2P_STAGE_BYTES 8192
#endif
#ifndef H2G_P2P_ASYNC
#define H2G_P2P_ASYNC 0  // measured slower (cfg 3: 10.23 vs 9.95 ms), kept for the record
#endif
#ifndef H2G_P2P_SLOTS
#define H2G_P2P_SLOTS (H2G_P2P_ASYNC ? 3 : 4)
#endif
#ifndef H2G_P2P_UNROLL
#define H2G_P2P_UNROLL 1
#endif
#ifndef H2G_P2P_UNROLL_SW
#define H2G_P2P_UNROLL_SW 1
#endif
// columns in flight per lane group in the evaluation loop (measured: one
// column at a time is 2-3 % faster than two, with and without a streaming
// warp -- the 8 rows per lane already give the chains to overlap)
constexpr int kP2PUnroll = H2G_P2P_UNROLL;
constexpr int kP2PUnrollSW = H2G_P2P_UNROLL_SW;
constexpr int kP2PStageBytes = H2G_P2P_STAGE_BYTES;       // operator data of one stage
constexpr int kP2PStageCols = 64;                         // columns of one stage at most
// one stage slot: the stage's x values (TMA-copied from the arena, 16-byte
// aligned start: + 1 double of shift), then its operator data (+ shift)
constexpr int kP2PSlotX = 8 * (kP2PStageCols + 2);
constexpr int kP2PSlotBytes = kP2PSlotX + kP2PStageBytes + 16;
constexpr int kP2PSlots = H2G_P2P_SLOTS;                  // stages in flight per CTA
// a phase gets streaming warps only if at least this share of its entries is
// stored (measured: cfg 5's all-evaluated phases lose 12 % with them)
constexpr double kP2PMinStagedShare = 0.15;
static_assert(kP2PSlots <= 32, "slot parity bits; first fill by one lane per slot");
// dynamic smem: [stage slots] + the evaluation warps' chunk buffers + the
// cross-warp reduction rows + [slot mbarriers, infos] + the task index
// kP2PAsync (off): the warps of a CTA run up to one task apart (two sets of
// reduction rows; the last warp to finish a task adds them up and fetches the
// set's next task) instead of meeting at a task-end barrier.  Measured: the
// M2L phases gain 2 % with streaming warps, but warps spinning on the set's
// mbarrier take issue slots from the fp64-bound ones (all-evaluated phases
// lose 4 %) and two reserved tasks per CTA lengthen the phase tails.
constexpr bool kP2PAsync = H2G_P2P_ASYNC != 0;
constexpr size_t p2p_smem_bytes(bool sw) {
  return (sw ? (size_t)kP2PSlots * kP2PSlotBytes + (size_t)kP2PSlots * 16 : 0) +
         (size_t)(sw ? kP2PWarpsSW : kP2PWarps) * 2 * kP2PChunk * (sizeof(double) * 4 + 8) +
         (size_t)(kP2PAsync ? 2 : 1) * (sw ? kP2PWarpsSW + 1 : kP2PWarps) * kMaxRows * 8 + 48;
}
static_assert(kP2PCtasSW * (p2p_smem_bytes(true) + 1024) <= 228 * 1024, "P2P smem per SM");
static_assert(kP2PCtasPerSm * (p2p_smem_bytes(false) + 1024) <= 228 * 1024, "P2P smem per SM");

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
// <= kP2PStageBytes / <= kP2PStageCols columns; a stage is TWO cp.async.bulk
// into a smem slot (its columns, and the x values they multiply), issued
// kP2PSlots ahead by the CTA's streaming warp and multiplied by it -- so HBM
// streams while the evaluation warps keep the fp64 pipe busy
// (m2l_recompute_share < 1: a share of every target's M2L blocks is read,
// the rest evaluated).
struct P2PStage {      // 32 bytes, everything the issuing lane needs precomputed
  uint64_t src;        // 16-byte aligned global address of the operator copy
  int64_t x_slot;      // even arena slot the x copy starts at
  uint32_t a_bytes;    // operator copy bytes (multiple of 16)
  uint32_t x_bytes;    // x copy bytes (multiple of 16)
  uint32_t info;       // columns | A shift << 16 | x shift << 17 (doubles past the copy starts)
  uint32_t pad;
};
static_assert(sizeof(P2PStage) == 32, "stage descriptor");

// Host: cut one stored block (m x ncols at A, contiguous columns) into
// equal-sized stages.
template <class Vec>
inline void p2p_cut_stages(const double* A, int64_t m, int64_t ncols, int64_t x_off, Vec& out) {
  const int64_t cap = std::max<int64_t>(
      1, std::min<int64_t>(kP2PStageCols, (kP2PStageBytes / 8) / std::max<int64_t>(1, m)));
  const int64_t n_st = (ncols + cap - 1) / cap;
  int64_t c0 = 0;
  for (int64_t i = 0; i < n_st; ++i) {
    const int64_t nc = (ncols - c0 + (n_st - i) - 1) / (n_st - i);
    const uint64_t src = reinterpret_cast<uint64_t>(A + c0 * m);
    const uint64_t a = src & ~uint64_t(15);
    const uint64_t e = (src + 8ull * (uint64_t)(m * nc) + 15) & ~uint64_t(15);
    const int64_t xo = x_off + c0, xs = xo & 1;
    P2PStage st{};
    st.src = a;
    st.x_slot = xo - xs;
    st.a_bytes = (uint32_t)(e - a);
    st.x_bytes = 8u * (uint32_t)((xs + nc + 1) & ~int64_t(1));
    st.info = (uint32_t)nc | ((uint32_t)((src - a) / 8) << 16) | ((uint32_t)xs << 17);
    out.push_back(st);
    c0 += nc;
  }
}

struct P2PChunk {      // 16 bytes: <= 32 columns of one evaluated block
  int64_t x_off;       // arena slot of x for column 0
  int32_t rec;         // record of column 0
  int32_t n_self;      // columns | kSelfBit (row and column runs share points)
};

// A stage descriptor held in registers (the two 16-byte loads as they come,
// unpacked only at the issue) many stages ahead of its use.
struct P2PStageRaw {
  ulonglong2 a;  // src, x_slot
  uint4 b;       // a_bytes, x_bytes, info, pad
};
__device__ __forceinline__ void load_stage_raw(P2PStageRaw& r, const P2PStage* p) {
  asm volatile("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(r.a.x), "=l"(r.a.y) : "l"(p));
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.b.x), "=r"(r.b.y), "=r"(r.b.z), "=r"(r.b.w)
               : "l"(reinterpret_cast<const char*>(p) + 16));
}

// One lane: post the slot's info word and the two bulk copies of a stage.
// (Slot reuse is a read-then-overwrite hazard only: the streaming warp's
// loads of the previous stage have all returned -- its sums depend on them --
// before this is issued, so no proxy fence is needed, as in the streaming
// engine's ring.)
__device__ __forceinline__ void issue_stage(const P2PStageRaw& st, const double* arena, char* slot,
                                            uint64_t* bar, int* info) {
  *info = (int)st.b.z;
  mbar_arrive_expect_tx(bar, st.b.x + st.b.y);
  bulk_g2s(slot + kP2PSlotX, reinterpret_cast<const void*>(st.a.x), st.b.x, bar);
  bulk_g2s(slot, arena + (int64_t)st.a.y, st.b.y, bar);
}

// One staged block for the streaming warp: lanes own rows lane + 32 jj (whole
// columns per warp request: conflict-free smem reads for any m), two columns
// per iteration into two partial sums per row.  Rows >= m read whatever
// follows in shared memory; their sums are never stored.
template <int JSC>
__device__ __forceinline__ void consume_staged(const double* __restrict__ col,
                                               const double* __restrict__ x, int nc, int m,
                                               double (&acc)[JSC]) {
  double p0[JSC], p1[JSC];
#pragma unroll
  for (int jj = 0; jj < JSC; ++jj) p0[jj] = p1[jj] = 0.0;
  const double* xe = x + (nc & ~1);
#pragma unroll 2
  for (; x < xe; x += 2, col += 2 * m) {
    const double x0 = x[0], x1 = x[1];
    double a0[JSC], a1[JSC];
#pragma unroll
    for (int jj = 0; jj < JSC; ++jj) {
      a0[jj] = col[32 * jj];
      a1[jj] = col[m + 32 * jj];
    }
#pragma unroll
    for (int jj = 0; jj < JSC; ++jj) {
      p0[jj] = fma(a0[jj], x0, p0[jj]);
      p1[jj] = fma(a1[jj], x1, p1[jj]);
    }
  }
  if (nc & 1) {
    const double x0 = x[0];
#pragma unroll
    for (int jj = 0; jj < JSC; ++jj) p0[jj] = fma(col[32 * jj], x0, p0[jj]);
  }
#pragma unroll
  for (int jj = 0; jj < JSC; ++jj) acc[jj] += p0[jj] + p1[jj];
}

// The streaming warp's share of one task: all its stages, in order, through
// the CTA's slot ring (stage i in slot i % kP2PSlots, kP2PSlots in flight);
// the sums of rows lane + 32 jj land in the warp's reduction row.
template <int JSC>
__device__ __forceinline__ void p2p_stream_task(const P2PTask& tk,
                                                const P2PStage* __restrict__ stages,
                                                const double* arena, char* slots, uint64_t* sbar,
                                                int* sinfo, uint32_t& sphase, double* myred,
                                                int lane) {
  const int m = tk.m;
  const int n_st = tk.s_end - tk.s_begin;
  const P2PStage* st = stages + tk.s_begin;
  // stage i is issued by lane i % 32 from `mine` (the descriptors of stages
  // [32 w, 32 w + 32), one per lane); the next window loads while this one is
  // worked through, so no load latency sits on the issue path
  P2PStageRaw mine{}, next{};
  if (lane < n_st) load_stage_raw(mine, st + lane);
  if (lane + 32 < n_st) load_stage_raw(next, st + lane + 32);
  if (lane < kP2PSlots && lane < n_st)  // first fill: one stage per lane
    issue_stage(mine, arena, slots + (size_t)lane * kP2PSlotBytes, &sbar[lane], &sinfo[lane]);
  __syncwarp();
  double acc[JSC];
#pragma unroll
  for (int jj = 0; jj < JSC; ++jj) acc[jj] = 0.0;
  int sl = 0;
  for (int i = 0; i < n_st; ++i) {
    mbar_wait(&sbar[sl], (sphase >> sl) & 1u);
    sphase ^= 1u << sl;
    const int info = sinfo[sl];
    char* slot = slots + (size_t)sl * kP2PSlotBytes;
    const double* sd = reinterpret_cast<const double*>(slot);
    consume_staged<JSC>(sd + kP2PSlotX / 8 + ((info >> 16) & 1) + lane, sd + ((info >> 17) & 1),
                        info & 0xffff, m, acc);
    __syncwarp();
    const int ni = i + kP2PSlots;
    if ((ni & 31) == 0) {  // warp-uniform: next window of descriptors
      mine = next;
      if (ni + 32 + lane < n_st) load_stage_raw(next, st + ni + 32 + lane);
    }
    if (lane == (ni & 31) && ni < n_st) issue_stage(mine, arena, slot, &sbar[sl], &sinfo[sl]);
    sl = sl + 1 == kP2PSlots ? 0 : sl + 1;
  }
#pragma unroll
  for (int jj = 0; jj < JSC; ++jj)
    if (lane + 32 * jj < m) myred[lane + 32 * jj] = acc[jj];
}

// FULL: the phase has self blocks (near diagonal) or coincident points (the
// r == 0 test in every entry); M2L phases of distinct points run the plain
// evaluation loop only -- a third of the code (the dispatch instantiates
// every L x J layout, and instruction fetch was a top stall at the leaf level).
template <int KT, int DIM, int L, int J, bool FULL, int W, int U>
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
  // ---- evaluated chunks k = k_begin + warp, + W, ...: the next
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
    k += W;
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
#pragma unroll U
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
#pragma unroll U
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
    for (int c = warp * G + g; c < tm.ncols; c += W * G) {
      const double xv = x[c];
      const double* col = A + (int64_t)c * tm.lda;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int r = rl + L * j;
        if (r < m) acc[j] = fma(ld_stream(col + r), xv, acc[j]);
      }
    }
  }
  // ---- combine: lane groups by a fixed xor tree into the warp's reduction
  // row (the kernel adds the rows of all warps in warp order)
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
}

// rows-per-lane layout for m rows: J ~ kP2PRowsPerLane independent row
// chains per lane, L = clamp(pow2ceil(ceil(m / JT)), 4, 32) lanes per column
// group, J = ceil(m / L) (<= 8 since m <= kMaxRows = 256)
#ifndef H2G_P2P_JT
#define H2G_P2P_JT 8
#endif
constexpr int kP2PRowsPerLane = H2G_P2P_JT;

template <int KT, int DIM, bool FULL, int W, int U>
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
  p2p_task<KT, DIM, Lv, Jv, FULL, W, U>(tk, terms, chunks, recs, blob, arena, kp, srec, sx, red, lane, warp)
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
// output is written once, in a fixed summation order (evaluation warps in
// warp order, then the streaming warp).  SW: the CTA has a streaming warp
// (phases with TMA stages).
template <int KT, int DIM, bool FULL, bool SW>
__global__ void __launch_bounds__(SW ? kP2PThreadsSW : kP2PThreads, SW ? kP2PCtasSW : kP2PCtasPerSm)
p2p_tasks_kernel(const P2PTask* __restrict__ tasks, int n_tasks, const Term* __restrict__ terms,
                 const P2PChunk* __restrict__ chunks, const P2PStage* __restrict__ stages,
                 const double4* __restrict__ recs, const double* __restrict__ blob,
                 double* arena, P2PKernel kp, int* ctr) {
  constexpr int W = SW ? kP2PWarpsSW : kP2PWarps;  // evaluation warps
  constexpr int NW = W + (SW ? 1 : 0);
  extern __shared__ __align__(128) double p2p_smem[];
  char* slots = reinterpret_cast<char*>(p2p_smem);  // SW: kP2PSlots x kP2PSlotBytes
  auto srec = reinterpret_cast<double4 (*)[2][kP2PChunk]>(
      slots + (SW ? (size_t)kP2PSlots * kP2PSlotBytes : 0));
  auto sx = reinterpret_cast<double (*)[2][kP2PChunk]>(srec + W);
  double* red = reinterpret_cast<double*>(sx + W);
  constexpr int NSET = kP2PAsync ? 2 : 1;  // sets of reduction rows
  uint64_t* sbar = reinterpret_cast<uint64_t*>(red + NSET * NW * kMaxRows);
  int* sinfo = reinterpret_cast<int*>(sbar + (SW ? kP2PSlots : 0));
  uint64_t* tbar = reinterpret_cast<uint64_t*>(sinfo + (SW ? 2 * kP2PSlots : 0));  // [2]
  int* s_task = reinterpret_cast<int*>(tbar + 2);                                  // [2]
  int* s_cnt = s_task + 2;                                                         // [2]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    if (SW)
      for (int i = 0; i < kP2PSlots; ++i) mbar_init(&sbar[i], 1);
    mbar_init(&tbar[0], 1);
    mbar_init(&tbar[1], 1);
    s_cnt[0] = s_cnt[1] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t sphase = 0;  // parity of every slot's barrier (streaming warp)
  griddep_launch_dependents();
  griddep_wait();  // x (and the counters' reset) come from earlier phases
  // this warp's share of task tk into the reduction rows at `rd`
  auto run_task = [&](const P2PTask& tk, double* rd) {
    if (!SW || warp < W)
      p2p_dispatch<KT, DIM, FULL, W, SW ? kP2PUnrollSW : kP2PUnroll>(
          tk, terms, chunks, recs, blob, arena, kp, srec[warp], sx[warp], rd, lane, warp);
    else {  // streaming warp: rows lane + 32 jj, jj < ceil(m / 32)
      double* myred = rd + W * kMaxRows;
      const int js = (tk.m + 31) >> 5;
      if (js == 1)
        p2p_stream_task<1>(tk, stages, arena, slots, sbar, sinfo, sphase, myred, lane);
      else if (js == 2)
        p2p_stream_task<2>(tk, stages, arena, slots, sbar, sinfo, sphase, myred, lane);
      else if (js <= 4)
        p2p_stream_task<4>(tk, stages, arena, slots, sbar, sinfo, sphase, myred, lane);
      else
        p2p_stream_task<8>(tk, stages, arena, slots, sbar, sinfo, sphase, myred, lane);
    }
  };
  if constexpr (kP2PAsync) {
    // Task n of the CTA lives in set n % 2.  A warp finishing its share of a
    // task counts itself in; the last one adds the warps' rows up in warp
    // order, stores y, fetches the set's next task and opens it (mbarrier):
    // warps run up to one task apart, the summation order stays fixed.
    if (threadIdx.x == 0)
      for (int b = 0; b < 2; ++b) {
        s_task[b] = atomicAdd(ctr, 1);
        mbar_arrive(&tbar[b]);
      }
    for (int n = 0;; ++n) {
      const int b = n & 1;
      mbar_wait(&tbar[b], (uint32_t)(n >> 1) & 1u);
      const int t = *reinterpret_cast<volatile int*>(&s_task[b]);
      if (t >= n_tasks) break;
      const P2PTask tk = tasks[t];
      double* rd = red + b * NW * kMaxRows;
      run_task(tk, rd);
      __syncwarp();
      int last = 0;
      if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&s_cnt[b], 1) == NW - 1;
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __threadfence_block();
        double* y = arena + tk.y_off;
        for (int r = lane; r < tk.m; r += 32) {
          double sum = rd[r];
#pragma unroll
          for (int w = 1; w < NW; ++w) sum += rd[w * kMaxRows + r];
          y[r] = sum;
        }
        __syncwarp();
        if (lane == 0) {
          s_cnt[b] = 0;
          *reinterpret_cast<volatile int*>(&s_task[b]) = atomicAdd(ctr, 1);
          __threadfence_block();
          mbar_arrive(&tbar[b]);
        }
      }
    }
    __syncthreads();  // every warp is done before the CTA reports out
  } else {
    for (;;) {
      if (threadIdx.x == 0) s_task[0] = atomicAdd(ctr, 1);
      __syncthreads();
      const int t = s_task[0];
      if (t >= n_tasks) break;
      const P2PTask tk = tasks[t];
      run_task(tk, red);
      __syncthreads();
      double* y = arena + tk.y_off;
      for (int r = threadIdx.x; r < tk.m; r += 32 * NW) {
        double sum = red[r];
#pragma unroll
        for (int w = 1; w < NW; ++w) sum += red[w * kMaxRows + r];
        y[r] = sum;
      }
      __syncthreads();  // red / s_task reuse
    }
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

// Launch interface (h2g_p2p_launch.cu: the kernels are their own translation
// unit): kt = 0 log r, 1 1/r, 2 Gaussian; full = self blocks / coincident
// points in the phase; sw = the phase has TMA stages.
cudaError_t p2p_configure();
int p2p_ctas_per_sm(bool sw);
cudaError_t p2p_launch(int kt, int dim, bool full, bool sw, bool pdl, unsigned grid,
                       cudaStream_t s, const P2PTask* tasks, int n_tasks, const Term* terms,
                       const P2PChunk* chunks, const P2PStage* stages, const double4* recs,
                       const double* blob, double* arena, const P2PKernel& kp, int* ctr);

}  // namespace h2g
