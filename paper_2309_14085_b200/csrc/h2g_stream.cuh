// h2g_stream.cuh — persistent TMA-bulk streaming GEMV engine (sm_100a).
//
// The matvec is HBM-bound: every stored operator scalar is used in exactly
// one multiply-add (0.25 flop/B).  The engine keeps many
// bytes in flight per SM without spending registers or issue slots on them:
//
//   * the host cuts every task (one output slice y[0:m), see h2g_kernels.cuh)
//     into CHUNKS of <= kChunkA doubles of operator data -- a run of whole
//     columns contiguous in the blob (possibly spanning several terms of the
//     task, e.g. the whole M2L row of a target) -- plus, per term, the slice of
//     the input vector x it multiplies (a "segment"; adjacent slices merge);
//   * every chunk is pre-decoded on the host into a 256-byte RECORD: the
//     consumer header (rows, columns, smem stride, alignment shift, segment
//     table) and the exact list of TMA bulk copies (absolute global source,
//     ring destination, bytes) that stage its operator data;
//   * one persistent CTA per SM-slot owns a contiguous range of tasks
//     (balanced by bytes on the host); kCtasPerSm pipelines per SM.  Inside a
//     CTA every task is OWNED by one consumer warp; the host interleaves the
//     chunk stream so that chunk i belongs to warp i % kConsumers (null chunks
//     pad uneven queues);
//   * warp 0 is the producer: lane 0 bulk-copies records kRecAhead chunks
//     ahead into a record ring, allocates each chunk a 16-byte aligned extent
//     of a byte-addressed data ring (freeing the oldest released chunks), arms
//     the slot's mbarrier (arrive.expect_tx) and lane k issues the record's
//     k-th cp.async.bulk (SASS UBLKCP);
//   * each consumer warp prefetches the x values of its next chunk from L2
//     into registers while the current one streams in, parks them in its smem
//     strip, waits for the slot, and runs a regular loop over the chunk's
//     columns: LDS.128 broadcast of two x values, one LDS.64 of A per 32 rows
//     per column, DFMA into per-lane row accumulators.  At a task's last chunk
//     the lanes store y directly: no cross-lane or cross-warp reduction.
//
// Narrow phases (few tasks: the coarse tree levels) run in SPLIT mode
// instead: all consumer warps work on every chunk (warp cw takes columns
// cw + kConsumers*t) and a task's partial sums are combined across warps in
// fixed order through shared memory at its last chunk.
//
// Determinism: a task is computed by one warp (or by all warps combined in
// warp order) in a fixed order.  No atomics.
#pragma once
#include <cstdint>

namespace h2g {

// Tunables (macro overrides exist for diagnostic builds only).
#ifndef H2G_CONSUMERS
#define H2G_CONSUMERS 4
#endif
#ifndef H2G_CTAS_PER_SM
#define H2G_CTAS_PER_SM 2
#endif
#ifndef H2G_RING_DOUBLES
#define H2G_RING_DOUBLES 12288   // 96 KB data ring per CTA
#endif
#ifndef H2G_SLOTS
#define H2G_SLOTS 16
#endif
#ifndef H2G_CHUNK_A
#define H2G_CHUNK_A 4096
#endif
constexpr int kLastOfTask = 1;
constexpr int kStridedRun = 2;                // record flag: one bulk copy per column
constexpr int kArenaA = 4;                    // record flag: operator data lives in the arena
                                              // (split-K partials written by the previous phase)
constexpr int kConsumers = H2G_CONSUMERS;     // consumer warps per CTA
constexpr int kStreamThreads = 32 * (1 + kConsumers);
constexpr int kCtasPerSm = H2G_CTAS_PER_SM;   // independent pipelines per SM
constexpr int kRing = H2G_RING_DOUBLES;       // byte-addressed data ring (doubles, per CTA)
constexpr int kSlots = H2G_SLOTS;             // max chunks in flight per CTA
constexpr int kRecRing = 28;                  // record ring depth
constexpr int kRecAhead = 8;                  // records prefetched ahead of the producer
constexpr int kChunkA = H2G_CHUNK_A;          // doubles of operator data per chunk (32 KB)
constexpr int kChunkCols = 256;               // max columns per chunk
constexpr int kMaxCopies = 6;                 // operator bulk copies per chunk (record capacity)
constexpr int kMaxSeg = 9;                    // x segments per chunk
constexpr int kStreamMaxRows = 256;
constexpr int kXStrip = kChunkCols + 8;       // per-warp x strip (doubles)
constexpr int kXPerLane = kChunkCols / 32;    // x values a lane prefetches
static_assert(kRecRing >= kSlots + kRecAhead, "record ring too shallow");
static_assert(kRing >= kChunkA + 8, "ring smaller than one chunk");

struct CopyDesc {       // 16 bytes
  uint64_t src;         // absolute global address (16-byte aligned)
  uint32_t dst;         // byte offset inside the data stage (16-byte aligned)
  uint32_t bytes;       // multiple of 16
};

struct ChunkRec {       // 256 bytes, host-built, TMA-copied into the record ring
  int64_t y_off;        // arena slot of y[0] of the owning task
  int32_t m;            // rows of the task (<= kStreamMaxRows)
  int32_t ncols;        // columns in this chunk
  int32_t flags;        // kLastOfTask
  int32_t n_seg;        // x segments
  int32_t ldas;         // column stride of A in smem (doubles)
  int32_t a_shift;      // A(0, 0) at sA + a_shift (odd_lda: shift of column 0)
  int32_t odd_lda;      // per-column copies whose alignment shift alternates
  int32_t n_copies;     // operator bulk copies
  uint32_t bytes_a;     // sum of operator copy bytes (expect_tx)
  int32_t extent;       // ring space the chunk occupies (doubles, even)
  int16_t seg_c0[kMaxSeg + 1];  // first chunk column of segment k (+ end sentinel)
  int32_t x_base;               // batched RHS: X (ncols x KB) at chunk + x_base doubles
  uint32_t bytes_x;             // batched RHS: bytes of the X copies (expect_tx)
  int16_t pad1[kMaxSeg + 1 - 4];
  uint64_t seg_src[kMaxSeg];    // absolute address of x for segment k's first column
  CopyDesc copies[kMaxCopies];
};
static_assert(sizeof(ChunkRec) == 256, "record layout");

constexpr size_t kStreamSmem = (size_t)kRing * 8 + (size_t)kConsumers * kXStrip * 8 +
                               (size_t)kRecRing * 256 +
                               (size_t)(2 * kSlots + kRecRing) * 8 + (size_t)kSlots * 4;

// ---------------------------------------------------------------- PTX helpers
// Programmatic dependent launch (phases launched with the programmatic
// stream-serialization attribute): a phase's grid may start while the
// previous one drains.  Everything a phase reads that the previous phase
// wrote (coefficients in the arena) is read only after griddep_wait(); the
// operator blob and the host-built records are read-only, so the producer
// streams them ahead.  Without the attribute both are no-ops.
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// TMA bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Same, with an L2 cache-policy hint (createpolicy): operator data is read
// exactly once per pass, so it is streamed evict_first and leaves L2 to the
// reused vectors (the batched engine's X arena is ~L2-sized).
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// Stage a chunk's operator data: either the record's explicit copy list
// (lane k issues copy k) or, for a STRIDED RUN (columns of a larger matrix,
// lda != m), one bulk copy per column: lane k copies column k (16-byte
// aligned start, so odd offsets carry a one-double shift) to k * ldas.
// copies[0] then holds {address of A(0, 0), lda, m}.
template <bool HINT = false>
__device__ __forceinline__ void issue_operator_copies(const ChunkRec& h, char* st, uint64_t* bar,
                                                      int lane, uint64_t pol = 0) {
  if (h.flags & kStridedRun) {
    if (lane < h.ncols) {
      const CopyDesc cd = h.copies[0];
      const int64_t lda = cd.dst;
      const int64_t col = (int64_t)lane * lda;
      const int sh = (int)((h.a_shift + col) & 1);
      const char* src = reinterpret_cast<const char*>(cd.src) + 8 * (col - sh);
      const uint32_t nb = (uint32_t)((8 * (sh + (int)cd.bytes) + 15) & ~15);
      if constexpr (HINT)
        bulk_g2s_hint(st + 8 * (int64_t)lane * h.ldas, src, nb, bar, pol);
      else
        bulk_g2s(st + 8 * (int64_t)lane * h.ldas, src, nb, bar);
    }
  } else if (lane < h.n_copies) {
    const CopyDesc cd = h.copies[lane];
    if constexpr (HINT)
      bulk_g2s_hint(st + cd.dst, reinterpret_cast<const void*>(cd.src), cd.bytes, bar, pol);
    else
      bulk_g2s(st + cd.dst, reinterpret_cast<const void*>(cd.src), cd.bytes, bar);
  }
}

// ---------------------------------------------------------------- consumer
// x of chunk columns c = lane + 32 q (q < kXPerLane), loaded from global (L2);
// 0 past the chunk.
__device__ __forceinline__ void fetch_x(const ChunkRec& h, int lane, double* xr) {
  const int ncols = h.ncols, n_seg = h.n_seg;
  int c0[kMaxSeg];
#pragma unroll
  for (int k = 0; k < kMaxSeg; ++k) c0[k] = h.seg_c0[k];
#pragma unroll
  for (int q = 0; q < kXPerLane; ++q) {
    const int c = lane + 32 * q;
    xr[q] = 0.0;
    if (32 * q < ncols) {  // warp-uniform skip of empty groups
      int k = 0, start = c0[0];
#pragma unroll
      for (int j = 1; j < kMaxSeg; ++j)
        if (j < n_seg && c >= c0[j]) {  // segments are ascending: the last hit wins
          k = j;
          start = c0[j];
        }
      if (c < ncols) xr[q] = __ldg(reinterpret_cast<const double*>(h.seg_src[k]) + (c - start));
    }
  }
}

// SPLIT mode: x of the warp's columns c = cw + kConsumers * (lane + 32 q), q < 2.
__device__ __forceinline__ void fetch_x_split(const ChunkRec& h, int lane, int cw, double* xr) {
  const int ncols = h.ncols, n_seg = h.n_seg;
  int c0[kMaxSeg];
#pragma unroll
  for (int k = 0; k < kMaxSeg; ++k) c0[k] = h.seg_c0[k];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int c = cw + kConsumers * (lane + 32 * q);
    int k = 0, start = c0[0];
#pragma unroll
    for (int j = 1; j < kMaxSeg; ++j)
      if (j < n_seg && c >= c0[j]) {
        k = j;
        start = c0[j];
      }
    xr[q] = c < ncols ? __ldg(reinterpret_cast<const double*>(h.seg_src[k]) + (c - start)) : 0.0;
  }
}

// One chunk: T columns of one warp, column t at As + t * step, x at xs[t]
// (owned mode: step = ldas, all columns; split mode: step = kConsumers*ldas).
// Rows >= m are computed from whatever lies in shared memory and discarded.
template <int J>
__device__ __forceinline__ void consume_stage(const double* __restrict__ As, int step, int T,
                                              const double* __restrict__ xs, int lane,
                                              double* acc) {
  constexpr int U = J == 1 ? 8 : (J == 2 ? 4 : 2);  // columns in flight per iteration
  double r[U][J];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int j = 0; j < J; ++j) r[u][j] = 0.0;
  const double* base = As + lane;
  int t = 0;
  for (; t + U <= T; t += U) {
    double xv[U], a[U][J];
#pragma unroll
    for (int u = 0; u < U; u += 2) {
      const double2 x2 = *reinterpret_cast<const double2*>(xs + t + u);
      xv[u] = x2.x;
      xv[u + 1] = x2.y;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double* col = base + (t + u) * step;
#pragma unroll
      for (int j = 0; j < J; ++j) a[u][j] = col[32 * j];
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < J; ++j) r[u][j] = fma(a[u][j], xv[u], r[u][j]);
  }
  for (; t < T; ++t) {
    const double x0 = xs[t];
    const double* col = base + t * step;
#pragma unroll
    for (int j = 0; j < J; ++j) r[0][j] = fma(col[32 * j], x0, r[0][j]);
  }
#pragma unroll
  for (int j = 0; j < J; ++j) {
    double tsum = r[0][j];
#pragma unroll
    for (int u = 1; u < U; ++u) tsum += r[u][j];
    acc[j] += tsum;
  }
}

// ------------------------------------------------------------------------
// Batched-RHS engine on the fp64 tensor pipe (DMMA, mma.sync m8n8k4 f64).
//
// Y (m x KB) += A (m x ncols) X (ncols x KB) per chunk: 8-row tiles of A by
// 4-column k-steps, NT = KB / 8 column tiles of X.  Fragments (PTX ISA
// m8n8k4 .f64): lane holds A[lane / 4][lane % 4], B[lane % 4][lane / 4] and
// C[lane / 4][2 (lane % 4) + {0, 1}].  Every chunk is SHARED by the four
// consumer warps, split 2-D by the task's row count: wr row groups (8-row
// tiles dealt round-robin) x wk column groups (k-steps dealt round-robin),
// wr * wk = 4:
//   m <= 32: 1 x 4,   m <= 64: 2 x 2,   m <= 256: 4 x 1,
// so a warp holds at most 8 tiles x NT accumulators (32 doubles at KB = 16)
// and column groups are combined at the task's last chunk in fixed warp order
// through shared memory.  Garbage rows (>= m) are computed and discarded; the
// k tail of a chunk is zeroed in both operands.  Deterministic, no atomics.
#ifndef H2G_MMA_CONSUMERS
#define H2G_MMA_CONSUMERS 4
#endif
#ifndef H2G_MMA_CTAS
#define H2G_MMA_CTAS 2
#endif
#ifndef H2G_MMA_RING
#define H2G_MMA_RING 11264        // 88 KB data ring per CTA
#endif
#ifndef H2G_MMA_CHUNK_A
#define H2G_MMA_CHUNK_A 4096
#endif
constexpr int kMmaConsumers = H2G_MMA_CONSUMERS;   // consumer warps sharing every chunk
constexpr int kMmaThreads = 32 * (1 + kMmaConsumers);
constexpr int kMmaCtasPerSm = H2G_MMA_CTAS;
constexpr int kRingMma = H2G_MMA_RING;
constexpr int kChunkAMma = H2G_MMA_CHUNK_A;        // operator + X doubles per chunk
#ifndef H2G_MMA_MIN_COLS
#define H2G_MMA_MIN_COLS 16
#endif
constexpr int kMmaMinCols = H2G_MMA_MIN_COLS;      // columns per chunk at least (tall tasks)
#ifndef H2G_MMA_GROUP
#define H2G_MMA_GROUP 1
#endif
#ifndef H2G_MMA_CHUNK_TALL
#define H2G_MMA_CHUNK_TALL 3072
#endif
#ifndef H2G_MMA_L2HINT
#define H2G_MMA_L2HINT 1   // operator copies evict_first (X stays in L2)
#endif
#ifndef H2G_MMA_GROUP_MIN
#define H2G_MMA_GROUP_MIN 2
#endif
constexpr bool kMmaGroupMode = H2G_MMA_GROUP != 0;  // wide phases in group mode
#ifndef H2G_MMA_DUAL
#define H2G_MMA_DUAL 0  // measured: no gain at cfg 2 (1.958 -> 1.973 ms per 16 RHS)
#endif
#ifndef H2G_MMA_PAD
#define H2G_MMA_PAD 0      // contiguous chunks of tall tasks staged column by column, padded stride
#endif
#ifndef H2G_MMA_PAD_MIN_M
#define H2G_MMA_PAD_MIN_M 48
#endif
constexpr bool kMmaPad = H2G_MMA_PAD != 0;
constexpr int kMmaPadMinM = H2G_MMA_PAD_MIN_M;
#ifndef H2G_MMA_PIPE
#define H2G_MMA_PIPE 1  // software-pipelined fragment loads in consume_mma (cfg 2 leaf pass 644 -> 628 us)
#endif
constexpr bool kMmaDualAcc = H2G_MMA_DUAL != 0;     // two accumulator sets for short row groups
constexpr int kMmaGroupMin = H2G_MMA_GROUP_MIN;     // smallest group (warps per chunk stream)
constexpr int kChunkAMmaTall = H2G_MMA_CHUNK_TALL;  // chunk of group-mode phases with tasks
                                                     // taller than 64 rows
static_assert(kMmaConsumers == 4 || kMmaConsumers == 8 || kMmaConsumers == 12, "mma consumers");
// row groups per size class (rt = 8-row tiles: <= 4, <= 8, <= 16, <= 32)
constexpr int kMmaWr3 = kMmaConsumers;             // widest class: all warps split rows
constexpr int kMaxTpw = kMmaConsumers == 4 ? 8 : 4; // tiles per warp (accumulator sets)
constexpr int kRedPerWarp = 4 * 2 * 64;            // partial tiles of one warp (doubles)
constexpr size_t kMmaSmem = (size_t)kRingMma * 8 + (size_t)kMmaConsumers * kRedPerWarp * 8 +
                            (size_t)kRecRing * 256 + (size_t)(2 * kSlots + kRecRing) * 8 +
                            (size_t)kSlots * 4;
static_assert(kRingMma >= kChunkAMma + 16 * 8 + 64, "mma ring smaller than one chunk");
static_assert(kMmaSmem <= 227 * 1024, "mma smem");

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Batched arena layout ("planes"): right-hand side b of slot s lives at
// (b >> 3) * ps + 8 s + (b & 7), i.e. KB / 8 planes of 8 doubles per slot.
// A chunk's X is staged plane by plane ([plane][column][8] in smem): the B
// fragment (column k = lane & 3, RHS n = lane >> 2) then spreads its four
// columns over both halves of the banks (16-wide rows put all four on the
// same banks).  Measured (cfg 2 leaf launch, 16 RHS): shared-memory
// wavefronts 142 M -> 104 M, 1004 -> 775 us.  (Re-pairing the columns of a
// k-step to de-conflict the A fragments did not reduce the wavefronts and
// cost time.)
template <int TPW, int NT>
__device__ __forceinline__ void mma_step(const double (&a)[TPW], const double (&b)[NT],
                                         double (&c)[8][2][2]) {
#pragma unroll
  for (int i = 0; i < TPW; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) dmma(c[i][nt], a[i], b[nt]);
}

// One chunk for one warp: tiles i < TPW at rows 8 (w_r + wr i), k-steps
// w_k, w_k + wk, ...  Ab: lane's A element of (tile 0, k-step 0); Bb: lane's
// X element of (k-step 0, plane 0); xps: smem plane stride.
// Short row groups (TPW <= 4 tiles: TPW x NT <= 8 accumulator chains) leave
// the DMMA pipe waiting on its own results (ncu: "wait" stalls); they
// alternate k-steps between two accumulator sets (c: even, c2: odd), summed
// in that fixed order at the task's end.
template <int TPW, int NT>
__device__ __forceinline__ void consume_mma(const double* __restrict__ Ab, int ldas, int tstride,
                                            const double* __restrict__ Bb, int xps, int ncols,
                                            int kq, int w_k, int wk, double (&c)[8][2][2],
                                            double (&c2)[4][2][2]) {
  const int full = ncols >> 2;                 // whole k-steps
  const int n_my = full > w_k ? (full - w_k + wk - 1) / wk : 0;
  const int adv_a = 4 * ldas * wk, adv_b = 4 * 8 * wk;
  const double* Ap = Ab + 4 * ldas * w_k;
  const double* Bp = Bb + 4 * 8 * w_k;
  int t = 0;
  if constexpr (TPW <= 4 && kMmaDualAcc) {
    for (; t + 2 <= n_my; t += 2) {
      double a[TPW], b[NT], a2[TPW], b2[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        b[nt] = Bp[nt * xps];
        b2[nt] = Bp[adv_b + nt * xps];
      }
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        a[i] = Ap[i * tstride];
        a2[i] = Ap[adv_a + i * tstride];
      }
#pragma unroll
      for (int i = 0; i < TPW; ++i)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma(c[i][nt], a[i], b[nt]);
          dmma(c2[i][nt], a2[i], b2[nt]);
        }
      Ap += 2 * adv_a;
      Bp += 2 * adv_b;
    }
  }
#if H2G_MMA_PIPE
  // software-pipelined: the fragments of k-step t + 1 are loaded before the
  // DMMAs of k-step t issue, so the LDS latency hides behind the tensor pipe
  if (t < n_my) {
    double a[TPW], b[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) b[nt] = Bp[nt * xps];
#pragma unroll
    for (int i = 0; i < TPW; ++i) a[i] = Ap[i * tstride];
#pragma unroll 2
    for (++t; t < n_my; ++t) {
      Ap += adv_a;
      Bp += adv_b;
      double an[TPW], bn[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) bn[nt] = Bp[nt * xps];
#pragma unroll
      for (int i = 0; i < TPW; ++i) an[i] = Ap[i * tstride];
      mma_step<TPW, NT>(a, b, c);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) b[nt] = bn[nt];
#pragma unroll
      for (int i = 0; i < TPW; ++i) a[i] = an[i];
    }
    mma_step<TPW, NT>(a, b, c);
  }
#else
#pragma unroll 2
  for (; t < n_my; ++t) {
    double a[TPW], b[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) b[nt] = Bp[nt * xps];
#pragma unroll
    for (int i = 0; i < TPW; ++i) a[i] = Ap[i * tstride];
    mma_step<TPW, NT>(a, b, c);
    Ap += adv_a;
    Bp += adv_b;
  }
#endif
  // k tail (ncols % 4 columns): the column group holding k-step `full`
  if ((ncols & 3) && (full % wk) == w_k) {
    const bool ok = 4 * full + kq < ncols;
    const double* At = Ab + 4 * ldas * full;
    const double* Bt = Bb + 4 * 8 * full;
    double a[TPW], b[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) b[nt] = ok ? Bt[nt * xps] : 0.0;
#pragma unroll
    for (int i = 0; i < TPW; ++i) a[i] = ok ? At[i * tstride] : 0.0;
    mma_step<TPW, NT>(a, b, c);
  }
}

template <int KB>
__global__ void __launch_bounds__(kMmaThreads, kMmaCtasPerSm)
stream_mma_kernel(const ChunkRec* __restrict__ recs, const int64_t* __restrict__ cta_begin,
                  double* arena, int64_t ps, int group) {
  constexpr int NT = KB / 8;
  static_assert(KB == 8 || KB == 16, "KB");
  extern __shared__ __align__(128) double smem[];
  double* ring = smem;
  double* red = smem + kRingMma;
  ChunkRec* rring = reinterpret_cast<ChunkRec*>(red + kMmaConsumers * kRedPerWarp);
  uint64_t* full = reinterpret_cast<uint64_t*>(rring + kRecRing);
  uint64_t* empty = full + kSlots;
  uint64_t* recbar = empty + kSlots;
  int* slot_off = reinterpret_cast<int*>(recbar + kRecRing);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t cb = cta_begin[blockIdx.x];
  const int n = (int)(cta_begin[blockIdx.x + 1] - cb);
  const ChunkRec* my = recs + cb;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], group > 0 ? group : kMmaConsumers);
    }
    for (int r = 0; r < kRecRing; ++r) mbar_init(&recbar[r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {  // producer: as stream_gemv_kernel, plus the chunk's X by TMA
    // group mode never reduces across warps: the reduction area (right behind
    // the ring) extends the ring
    const int ring_cap = group > 0 ? kRingMma + kMmaConsumers * kRedPerWarp : kRingMma;
#if H2G_MMA_L2HINT
    const uint64_t pol_a = l2_policy_evict_first();
#endif
    int oldest = 0, head = 0, tail = 0;
    if (lane == 0)
      for (int j = 0; j < kRecAhead && j < n; ++j) {
        mbar_arrive_expect_tx(&recbar[j], sizeof(ChunkRec));
        bulk_g2s(&rring[j], my + j, sizeof(ChunkRec), &recbar[j]);
      }
    for (int i = 0; i < n; ++i) {
      const int s = i % kSlots;
      const int r = i % kRecRing;
      mbar_wait(&recbar[r], (uint32_t)(i / kRecRing) & 1u);
      const ChunkRec& h = rring[r];
      int off = 0;
      if (lane == 0) {
        const int need = h.extent;
        auto release_oldest = [&]() {
          mbar_wait(&empty[oldest % kSlots], (uint32_t)(oldest / kSlots) & 1u);
          ++oldest;
          tail = oldest < i ? slot_off[oldest % kSlots] : head;
        };
        while (i - oldest >= kSlots) release_oldest();
        while (true) {
          if (oldest == i) {
            head = tail = 0;
            off = 0;
            break;
          }
          if (head >= tail) {
            if (ring_cap - head >= need) { off = head; break; }
            if (tail > need) { off = 0; break; }
          } else if (tail - head > need) {
            off = head;
            break;
          }
          release_oldest();
        }
        head = off + need;
        slot_off[s] = off;
        const int j = i + kRecAhead;
        if (j < n) {
          const int rj = j % kRecRing;
          mbar_arrive_expect_tx(&recbar[rj], sizeof(ChunkRec));
          bulk_g2s(&rring[rj], my + j, sizeof(ChunkRec), &recbar[rj]);
        }
        mbar_arrive_expect_tx(&full[s], h.bytes_a + h.bytes_x);
      }
      off = __shfl_sync(0xffffffffu, off, 0);
      char* st = reinterpret_cast<char*>(ring + off);
#if H2G_MMA_L2HINT
      issue_operator_copies<true>(h, st, &full[s], lane, pol_a);
#else
      issue_operator_copies(h, st, &full[s], lane);
#endif
      // X plane by plane: [plane][column][8] behind the operator data
      for (int k = lane; k < h.n_seg * NT; k += 32) {
        const int sg = k % h.n_seg, pl = k / h.n_seg;
        const int c0 = h.seg_c0[sg], c1 = h.seg_c0[sg + 1];
        bulk_g2s(st + 8 * (h.x_base + pl * 8 * h.ncols + 8 * c0),
                 reinterpret_cast<const char*>(h.seg_src[sg]) + 8 * (uint64_t)pl * ps,
                 (uint32_t)(64 * (c1 - c0)), &full[s]);
      }
      __syncwarp();
    }
    return;
  }

  const int cw = warp - 1;
  const int kq = lane & 3, rq = lane >> 2;
  // this warp's (row group, column group) in each size class
  int cls_wr[4], cls_wk[4], cls_r[4], cls_k[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int wr = k == 3 ? kMmaWr3 : (1 << k);
    cls_wr[k] = wr;
    cls_wk[k] = kMmaConsumers / wr;
    cls_r[k] = cw % wr;
    cls_k[k] = cw / wr;
  }
  double c[8][2][2];
  double c2[4][2][2];  // odd k-steps of short row groups (consume_mma)
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) c[i][nt][0] = c[i][nt][1] = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) c2[i][nt][0] = c2[i][nt][1] = 0.0;
  // fold the odd-k-step accumulators into c (fixed order) and clear them
  auto fold_c2 = [&]() {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        c[i][nt][0] += c2[i][nt][0];
        c[i][nt][1] += c2[i][nt][1];
        c2[i][nt][0] = c2[i][nt][1] = 0.0;
      }
  };
  if (group > 0) {
    // GROUP mode: warps [G st, G st + G) own chunk stream st (chunks i = st
    // mod S); warp g of the group takes row tiles g, g + G, ... (<= 8, the
    // host picks G by the phase's largest task) and every k-step, so it
    // stores its rows at the task's last chunk -- no cross-warp reduction.
    const int G = group, S = kMmaConsumers / group;
    const int st = cw / G, g = cw - st * G;
    for (int i = st; i < n; i += S) {
      const int s = i % kSlots;
      mbar_wait(&recbar[i % kRecRing], (uint32_t)(i / kRecRing) & 1u);
      const ChunkRec& h = rring[i % kRecRing];
      const int m = h.m;
      const int ncols = h.ncols;
      const int flags = h.flags;
      const int ldas = h.ldas;
      const int a_shift = h.a_shift;
      const int odd = h.odd_lda;
      const int x_base = h.x_base;
      const int64_t y_off = h.y_off;
      const int rt = (m + 7) >> 3;
      const int tpw = g < rt ? (rt - g + G - 1) / G : 0;
      mbar_wait(&full[s], (uint32_t)(i / kSlots) & 1u);
      if (ncols > 0 && tpw > 0) {
        const double* sA = ring + slot_off[s];
        const int lane_shift = odd ? ((a_shift + kq) & 1) : a_shift;
        const double* Ab = sA + kq * ldas + lane_shift + rq + 8 * g;
        const double* Bb = sA + x_base + kq * 8 + rq;
        const int xps = 8 * ncols;
        const int ts = 8 * G;
        switch (tpw) {
          case 1: consume_mma<1, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, 0, 1, c, c2); break;
          case 2: consume_mma<2, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, 0, 1, c, c2); break;
          case 3: consume_mma<3, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, 0, 1, c, c2); break;
          case 4: consume_mma<4, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, 0, 1, c, c2); break;
          default:
            if constexpr (kMaxTpw > 4) {
              switch (tpw) {
                case 5: consume_mma<5, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, 0, 1, c, c2); break;
                case 6: consume_mma<6, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, 0, 1, c, c2); break;
                case 7: consume_mma<7, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, 0, 1, c, c2); break;
                default: consume_mma<8, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, 0, 1, c, c2); break;
              }
            }
            break;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (flags & kLastOfTask) {
        fold_c2();
        double* y = arena + y_off * 8;
#pragma unroll
        for (int t = 0; t < kMaxTpw; ++t) {
          const int row = 8 * (g + G * t) + rq;
          if (t < tpw && row < m)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              *reinterpret_cast<double2*>(y + nt * ps + (int64_t)row * 8 + 2 * kq) =
                  make_double2(c[t][nt][0], c[t][nt][1]);
        }
#pragma unroll
        for (int t = 0; t < 8; ++t)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) c[t][nt][0] = c[t][nt][1] = 0.0;
      }
    }
    return;
  }
  for (int i = 0; i < n; ++i) {
    const int s = i % kSlots;
    mbar_wait(&recbar[i % kRecRing], (uint32_t)(i / kRecRing) & 1u);
    const ChunkRec& h = rring[i % kRecRing];
    const int m = h.m;
    const int ncols = h.ncols;
    const int flags = h.flags;
    const int ldas = h.ldas;
    const int a_shift = h.a_shift;
    const int odd = h.odd_lda;
    const int x_base = h.x_base;
    const int64_t y_off = h.y_off;
    const int rt = (m + 7) >> 3;                     // 8-row tiles
    const int cls = rt <= 4 ? 0 : (rt <= 8 ? 1 : (rt <= 16 ? 2 : 3));
    int wr = cls_wr[0], wk = cls_wk[0], w_r = cls_r[0], w_k = cls_k[0];
#pragma unroll
    for (int k = 1; k < 4; ++k)
      if (cls == k) {
        wr = cls_wr[k];
        wk = cls_wk[k];
        w_r = cls_r[k];
        w_k = cls_k[k];
      }
    const int tpw = w_r < rt ? (rt - w_r + wr - 1) / wr : 0;  // this warp's tiles
    mbar_wait(&full[s], (uint32_t)(i / kSlots) & 1u);
    if (ncols > 0 && tpw > 0) {
      const double* sA = ring + slot_off[s];
      const int lane_shift = odd ? ((a_shift + kq) & 1) : a_shift;
      const double* Ab = sA + kq * ldas + lane_shift + rq + 8 * w_r;
      const double* Bb = sA + x_base + kq * 8 + rq;
      const int xps = 8 * ncols;
      const int ts = 8 * wr;
      switch (tpw) {
        case 1: consume_mma<1, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, w_k, wk, c, c2); break;
        case 2: consume_mma<2, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, w_k, wk, c, c2); break;
        case 3: consume_mma<3, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, w_k, wk, c, c2); break;
        case 4: consume_mma<4, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, w_k, wk, c, c2); break;
        default:
          if constexpr (kMaxTpw > 4) {
            switch (tpw) {
              case 5: consume_mma<5, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, w_k, wk, c, c2); break;
              case 6: consume_mma<6, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, w_k, wk, c, c2); break;
              case 7: consume_mma<7, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, w_k, wk, c, c2); break;
              default: consume_mma<8, NT>(Ab, ldas, ts, Bb, xps, ncols, kq, w_k, wk, c, c2); break;
            }
          }
          break;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (flags & kLastOfTask) {
      fold_c2();
      double* y = arena + y_off * 8;  // plane 0; plane nt at + nt * ps
      // classes with wk > 1 have at most 4 tiles per warp
      if (wk > 1) {  // park partials of column groups 1.. ; group 0 combines them
        if (w_k > 0) {
          double* rw = red + cw * kRedPerWarp;
#pragma unroll
          for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              *reinterpret_cast<double2*>(rw + (t * 2 + nt) * 64 + 2 * lane) =
                  make_double2(c[t][nt][0], c[t][nt][1]);
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kMmaConsumers * 32) : "memory");
        if (w_k == 0) {
          for (int g = 1; g < wk; ++g) {
            const double* rg = red + (w_r + wr * g) * kRedPerWarp + 2 * lane;
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) {
                const double2 v = *reinterpret_cast<const double2*>(rg + (t * 2 + nt) * 64);
                c[t][nt][0] += v.x;
                c[t][nt][1] += v.y;
              }
          }
        }
      }
      if (w_k == 0) {
#pragma unroll
        for (int t = 0; t < kMaxTpw; ++t) {
          const int row = 8 * (w_r + wr * t) + rq;
          if (t < tpw && row < m)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              *reinterpret_cast<double2*>(y + nt * ps + (int64_t)row * 8 + 2 * kq) =
                  make_double2(c[t][nt][0], c[t][nt][1]);
        }
      }
#pragma unroll
      for (int t = 0; t < 8; ++t)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) c[t][nt][0] = c[t][nt][1] = 0.0;
      if (wk > 1) asm volatile("bar.sync 1, %0;" ::"r"(kMmaConsumers * 32) : "memory");
    }
  }
}

template <bool SPLIT>
__global__ void __launch_bounds__(kStreamThreads, kCtasPerSm)
stream_gemv_kernel(const ChunkRec* __restrict__ recs, const int64_t* __restrict__ cta_begin,
                   double* arena) {
  extern __shared__ __align__(128) double smem[];
  double* ring = smem;
  double* xstrip = smem + kRing;
  ChunkRec* rring = reinterpret_cast<ChunkRec*>(xstrip + kConsumers * kXStrip);
  uint64_t* full = reinterpret_cast<uint64_t*>(rring + kRecRing);
  uint64_t* empty = full + kSlots;
  uint64_t* recbar = empty + kSlots;
  int* slot_off = reinterpret_cast<int*>(recbar + kRecRing);  // ring offset of slot's chunk

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t cb = cta_begin[blockIdx.x];
  const int n = (int)(cta_begin[blockIdx.x + 1] - cb);
  const ChunkRec* my = recs + cb;
  griddep_launch_dependents();  // the next phase may start filling its rings

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SPLIT ? kConsumers : 1);  // owning warp, or all warps
    }
    for (int r = 0; r < kRecRing; ++r) mbar_init(&recbar[r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------ producer warp
    // Chunks occupy variable-size, 16-byte aligned extents of the data ring in
    // issue order; chunk i uses slot i % kSlots.  Lane 0 allocates: it frees
    // the oldest chunks (waiting for their release) until the next extent fits.
    int oldest = 0;        // oldest chunk not yet known to be released
    int head = 0;          // next free ring offset (doubles)
    int tail = 0;          // ring offset of chunk `oldest` (valid if oldest < i)
    bool waited = false;   // griddep_wait() done (needed before arena-sourced copies)
    if (lane == 0)
      for (int j = 0; j < kRecAhead && j < n; ++j) {
        mbar_arrive_expect_tx(&recbar[j], sizeof(ChunkRec));
        bulk_g2s(&rring[j], my + j, sizeof(ChunkRec), &recbar[j]);
      }
    for (int i = 0; i < n; ++i) {
      const int s = i % kSlots;
      const int r = i % kRecRing;
      mbar_wait(&recbar[r], (uint32_t)(i / kRecRing) & 1u);
      const ChunkRec& h = rring[r];
      int off = 0;
      if (lane == 0) {
        const int need = h.extent;
        auto release_oldest = [&]() {
          mbar_wait(&empty[oldest % kSlots], (uint32_t)(oldest / kSlots) & 1u);
          ++oldest;
          tail = oldest < i ? slot_off[oldest % kSlots] : head;
        };
        while (i - oldest >= kSlots) release_oldest();
        while (true) {
          if (oldest == i) {  // ring empty
            head = tail = 0;
            off = 0;
            break;
          }
          // strict inequalities when allocating below `tail` keep head < tail
          // afterwards, so head == tail never means "full"
          if (head >= tail) {  // occupied [tail, head): free [head, kRing) and [0, tail)
            if (kRing - head >= need) { off = head; break; }
            if (tail > need) { off = 0; break; }
          } else if (tail - head > need) {  // occupied wraps: free [head, tail)
            off = head;
            break;
          }
          release_oldest();
        }
        head = off + need;
        slot_off[s] = off;
        // records ahead: slot (i + kRecAhead) % kRecRing last held chunk
        // i + kRecAhead - kRecRing < oldest, which consumers have released
        const int j = i + kRecAhead;
        if (j < n) {
          const int rj = j % kRecRing;
          mbar_arrive_expect_tx(&recbar[rj], sizeof(ChunkRec));
          bulk_g2s(&rring[rj], my + j, sizeof(ChunkRec), &recbar[rj]);
        }
        mbar_arrive_expect_tx(&full[s], h.bytes_a);
      }
      off = __shfl_sync(0xffffffffu, off, 0);
      if ((h.flags & kArenaA) && !waited) {
        griddep_wait();
        waited = true;
      }
      issue_operator_copies(h, reinterpret_cast<char*>(ring + off), &full[s], lane);
      __syncwarp();
    }
    return;
  }
  griddep_wait();  // consumers read x (previous phases' outputs) from here on

  // ---------------------------------------------------- consumers
  const int cw = warp - 1;
  double* xs = xstrip + cw * kXStrip;
  double acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.0;
  if constexpr (SPLIT) {
    // all warps on every chunk; task partials combined across warps in smem
    // (warp w's strip doubles as its reduction row once its chunk is consumed)
    double xn[2] = {0.0, 0.0};
    if (n > 0) {
      mbar_wait(&recbar[0], 0u);
      fetch_x_split(rring[0], lane, cw, xn);
    }
    for (int i = 0; i < n; ++i) {
      const int s = i % kSlots;
      const ChunkRec& h = rring[i % kRecRing];
      const int m = h.m;
      const int ncols = h.ncols;
      const int flags = h.flags;
      const int ldas = h.ldas;
      const int a_shift = h.a_shift;
      const int odd = h.odd_lda;
      const int64_t y_off = h.y_off;
      xs[lane] = xn[0];
      xs[lane + 32] = xn[1];
      if (i + 1 < n) {
        mbar_wait(&recbar[(i + 1) % kRecRing], (uint32_t)((i + 1) / kRecRing) & 1u);
        fetch_x_split(rring[(i + 1) % kRecRing], lane, cw, xn);
      }
      __syncwarp();
      mbar_wait(&full[s], (uint32_t)(i / kSlots) & 1u);
      const double* sA = ring + slot_off[s];
      const int T = ncols > cw ? (ncols - cw + kConsumers - 1) / kConsumers : 0;
#ifndef H2G_DIAG_NOCOMPUTE
      if (!odd) {
        const double* As = sA + a_shift + cw * ldas;
        const int step = kConsumers * ldas;
        const int J = (m + 31) >> 5;
        if (J == 1)
          consume_stage<1>(As, step, T, xs, lane, acc);
        else if (J == 2)
          consume_stage<2>(As, step, T, xs, lane, acc);
        else if (J <= 4)
          consume_stage<4>(As, step, T, xs, lane, acc);
        else
          consume_stage<8>(As, step, T, xs, lane, acc);
      } else {
        for (int t = 0; t < T; ++t) {
          const int c = cw + kConsumers * t;
          const double* col = sA + (size_t)c * ldas + ((a_shift + c) & 1);
          const double xv = xs[t];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int rr = lane + 32 * j;
            if (rr < m) acc[j] = fma(col[rr], xv, acc[j]);
          }
        }
      }
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (flags & kLastOfTask) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int rr = lane + 32 * j;
          if (rr < m) xs[rr] = acc[j];
          acc[j] = 0.0;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
        double* y = arena + y_off;
        for (int rr = threadIdx.x - 32; rr < m; rr += kConsumers * 32) {
          double sum = xstrip[rr];
#pragma unroll
          for (int w = 1; w < kConsumers; ++w) sum += xstrip[w * kXStrip + rr];
          y[rr] = sum;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
      }
    }
  } else {
  // owned mode: chunk i belongs to warp i % kConsumers
  double xn[kXPerLane];
#pragma unroll
  for (int q = 0; q < kXPerLane; ++q) xn[q] = 0.0;
  if (cw < n) {
    mbar_wait(&recbar[cw % kRecRing], (uint32_t)(cw / kRecRing) & 1u);
    fetch_x(rring[cw % kRecRing], lane, xn);
  }
  for (int i = cw; i < n; i += kConsumers) {
    const int s = i % kSlots;
    const ChunkRec& h = rring[i % kRecRing];
    const int m = h.m;
    const int ncols = h.ncols;
    const int flags = h.flags;
    const int ldas = h.ldas;
    const int a_shift = h.a_shift;
    const int odd = h.odd_lda;
    const int64_t y_off = h.y_off;
    // park this chunk's x, then issue the next owned chunk's x loads
#pragma unroll
    for (int q = 0; q < kXPerLane; ++q)
      if (32 * q < ncols) xs[lane + 32 * q] = xn[q];
    const int inext = i + kConsumers;
    if (inext < n) {
      mbar_wait(&recbar[inext % kRecRing], (uint32_t)(inext / kRecRing) & 1u);
      fetch_x(rring[inext % kRecRing], lane, xn);
    }
    __syncwarp();
    mbar_wait(&full[s], (uint32_t)(i / kSlots) & 1u);
    const double* sA = ring + slot_off[s];
#ifndef H2G_DIAG_NOCOMPUTE
    if (!odd) {
      const double* As = sA + a_shift;
      const int J = (m + 31) >> 5;
      if (J == 1)
        consume_stage<1>(As, ldas, ncols, xs, lane, acc);
      else if (J == 2)
        consume_stage<2>(As, ldas, ncols, xs, lane, acc);
      else if (J <= 4)
        consume_stage<4>(As, ldas, ncols, xs, lane, acc);
      else
        consume_stage<8>(As, ldas, ncols, xs, lane, acc);
    } else {
      // per-column copies with odd lda (rare): alignment shift alternates
      for (int c = 0; c < ncols; ++c) {
        const double* col = sA + (size_t)c * ldas + ((a_shift + c) & 1);
        const double xv = xs[c];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int rr = lane + 32 * j;
          if (rr < m) acc[j] = fma(col[rr], xv, acc[j]);
        }
      }
    }
#endif
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (flags & kLastOfTask) {  // this warp owns the task: store y directly
      double* y = arena + y_off;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int rr = lane + 32 * j;
        if (rr < m) y[rr] = acc[j];
        acc[j] = 0.0;
      }
    }
  }
  }  // owned mode
}

}  // namespace h2g
