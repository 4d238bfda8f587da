// h2g_stream.cuh — persistent TMA-bulk streaming GEMV engine (sm_100a).
//
// The matvec is HBM-bound: every stored operator scalar is used in exactly
// one multiply-add (0.25 flop/B).  The engine keeps many
// bytes in flight per SM without spending registers on them:
//
//   * the host cuts every task (one output slice y[0:m), see h2g_kernels.cuh)
//     into CHUNKS of <= kChunkA doubles of operator data: a run of whole
//     columns that is contiguous in the blob (possibly spanning several terms
//     of the task, e.g. all M2L blocks of one target) plus, per term, the
//     matching slice of the input vector x (a "segment");
//   * one persistent CTA per SM owns a contiguous range of chunks (whole
//     tasks, balanced by bytes on the host);
//   * warp 0 is the producer: its lanes fetch 32 chunk headers at a time
//     (coalesced, prefetched one batch ahead), then one elected lane waits for
//     a free ring stage, writes the chunk's decoded header into shared memory
//     and issues cp.async.bulk copies (TMA bulk, SASS UBLKCP) of the operator
//     columns and of every x segment, completing on the stage's mbarrier
//     (arrive.expect_tx);
//   * warps 1..kConsumers are consumers: they wait on the stage's mbarrier,
//     read the column-major chunk from shared memory (lane = row,
//     conflict-free), accumulate in registers, release the stage, and at the
//     end of a task reduce the warps' partial sums in a fixed order and store
//     y once.
//
// Determinism: a task lives in one CTA; each warp accumulates its columns in
// a fixed order; warps are combined in warp order.  No atomics.
#pragma once
#include <cstdint>

namespace h2g {

struct Chunk {          // 40 bytes, host-built
  int64_t a_off;        // blob offset (doubles) of the first operator entry
  int64_t y_off;        // arena slot of y[0] of the owning task
  int32_t lda;          // == m: contiguous run (one copy); else per-column copies
  int32_t m;            // rows of the task (<= kStreamMaxRows)
  int32_t ncols;        // columns in this chunk
  int32_t flags;        // kLastOfTask
  int32_t seg_begin;    // x segments [seg_begin, seg_begin + n_seg) in Seg[]
  int32_t n_seg;
};

struct Seg {            // 16 bytes: x slice of consecutive chunk columns
  int64_t x_off;        // arena slot of x for the segment's first column
  int32_t ncols;
  int32_t pad;
};

constexpr int kLastOfTask = 1;
constexpr int kConsumers = 4;                 // consumer warps per CTA
constexpr int kStreamThreads = 32 * (1 + kConsumers);
constexpr int kStages = 8;                    // ring depth
constexpr int kChunkA = 2048;                 // doubles of operator data per chunk (16 KB)
constexpr int kChunkCols = 256;               // max columns per chunk
constexpr int kMaxSeg = 16;                   // max x segments per chunk
constexpr int kStageX = kChunkCols + 2 * kMaxSeg + 4;  // x slots incl. alignment slack
constexpr int kStageA = kChunkA + 8;
constexpr int kStageDoubles = kStageA + kStageX;
constexpr int kStreamMaxRows = 256;

struct StageHdr {       // decoded by the producer, read by consumers (smem)
  int64_t y_off;
  int32_t m, ncols, flags, n_seg;
  int32_t ldas;         // column stride in smem
  int32_t a_shift;      // first operator entry at sA + a_shift (contiguous runs)
  int32_t strided;      // 1: per-column copies, column c at sA + c*ldas + shift_c
  int32_t odd_lda;      // strided with odd lda: per-column shift alternates
  int32_t a_shift0;     // shift of column 0 (strided)
  int32_t pad;
  int16_t seg_c0[kMaxSeg];   // first chunk column of segment k
  int16_t seg_x[kMaxSeg];    // smem x index of segment k's first value
};

constexpr size_t kHdrBytes = ((sizeof(StageHdr) + 15) / 16) * 16;
constexpr size_t kStreamSmem = (size_t)kStages * kStageDoubles * 8 +
                               (size_t)kConsumers * kStreamMaxRows * 8 +
                               (size_t)kStages * kHdrBytes + 2 * kStages * 8 +
                               (size_t)32 * kMaxSeg * sizeof(Seg);

// ---------------------------------------------------------------- PTX helpers
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

__device__ __forceinline__ int dshift(const double* p) {
  return (int)((((uintptr_t)p) & 15) >> 3);
}

// bytes of an aligned-down copy of n doubles starting at p
__device__ __forceinline__ uint32_t span_bytes(const double* p, int n) {
  return (uint32_t)(((dshift(p) + n) * 8 + 15) & ~15);
}

__device__ __forceinline__ const double* align_down(const double* p) {
  return (const double*)(((uintptr_t)p) & ~(uintptr_t)15);
}

__device__ __forceinline__ Chunk shfl_chunk(const Chunk& c, int src) {
  Chunk o;
  o.a_off = __shfl_sync(0xffffffffu, c.a_off, src);
  o.y_off = __shfl_sync(0xffffffffu, c.y_off, src);
  o.lda = __shfl_sync(0xffffffffu, c.lda, src);
  o.m = __shfl_sync(0xffffffffu, c.m, src);
  o.ncols = __shfl_sync(0xffffffffu, c.ncols, src);
  o.flags = __shfl_sync(0xffffffffu, c.flags, src);
  o.seg_begin = __shfl_sync(0xffffffffu, c.seg_begin, src);
  o.n_seg = __shfl_sync(0xffffffffu, c.n_seg, src);
  return o;
}

// ---------------------------------------------------------------- consumer
// columns [c_begin, c_end) of a chunk whose column c is at As + c*ldas and
// whose x value is xs[c - c_begin]; warp cw takes c_begin+cw, +kConsumers, ...
template <int J>
__device__ __forceinline__ void consume_cols(const double* __restrict__ As, int ldas,
                                             const double* __restrict__ xs, int c_begin,
                                             int c_end, int m, int lane, int cw, double* acc) {
  double r0[J], r1[J];
#pragma unroll
  for (int j = 0; j < J; ++j) r0[j] = r1[j] = 0.0;
  int c = c_begin + cw;
  for (; c + kConsumers < c_end; c += 2 * kConsumers) {
    const double x0 = xs[c - c_begin];
    const double x1 = xs[c + kConsumers - c_begin];
    const double* col0 = As + c * ldas;
    const double* col1 = col0 + kConsumers * ldas;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int rr = lane + 32 * j;
      if (rr < m) {
        r0[j] = fma(col0[rr], x0, r0[j]);
        r1[j] = fma(col1[rr], x1, r1[j]);
      }
    }
  }
  if (c < c_end) {
    const double x0 = xs[c - c_begin];
    const double* col0 = As + c * ldas;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int rr = lane + 32 * j;
      if (rr < m) r0[j] = fma(col0[rr], x0, r0[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < J; ++j) acc[j] += r0[j] + r1[j];
}

template <int J>
__device__ __forceinline__ void consume_stage(const StageHdr& h, const double* sA,
                                              const double* sX, int lane, int cw, double* acc) {
  const double* As = sA + h.a_shift;
  for (int k = 0; k < h.n_seg; ++k) {
    const int c0 = h.seg_c0[k];
    const int c1 = (k + 1 < h.n_seg) ? h.seg_c0[k + 1] : h.ncols;
    consume_cols<J>(As, h.ldas, sX + h.seg_x[k], c0, c1, h.m, lane, cw, acc);
  }
}

__global__ void __launch_bounds__(kStreamThreads, 1)
stream_gemv_kernel(const Chunk* __restrict__ chunks, const Seg* __restrict__ segs,
                   const int64_t* __restrict__ cta_begin, const double* __restrict__ blob,
                   double* arena) {
  extern __shared__ __align__(128) double smem[];
  double* stage_buf = smem;
  double* red = smem + (size_t)kStages * kStageDoubles;
  StageHdr* hdr = reinterpret_cast<StageHdr*>(red + kConsumers * kStreamMaxRows);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(hdr) + kStages * kHdrBytes);
  uint64_t* empty = full + kStages;
  Seg* seg_scratch = reinterpret_cast<Seg*>(empty + kStages);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t cb = cta_begin[blockIdx.x];
  const int64_t ce = cta_begin[blockIdx.x + 1];

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------ producer warp
    Chunk cur{}, nxt{};
    if (cb + lane < ce) cur = chunks[cb + lane];
    if (cb + 32 + lane < ce) nxt = chunks[cb + 32 + lane];
    for (int64_t base = cb; base < ce; base += 32) {
      const int nb = (int)(ce - base < 32 ? ce - base : 32);
      // stage this batch's segment descriptors (consecutive in segs[]) in smem
      const int seg_base = __shfl_sync(0xffffffffu, cur.seg_begin, 0);
      const int seg_end = __shfl_sync(0xffffffffu, cur.seg_begin + cur.n_seg, nb - 1);
      for (int e = lane; e < seg_end - seg_base; e += 32) seg_scratch[e] = segs[seg_base + e];
      __syncwarp();
      for (int k = 0; k < nb; ++k) {
        const Chunk ch = shfl_chunk(cur, k);
        // lanes < n_seg take the segment descriptors of this chunk (smem copy)
        Seg sg{};
        if (lane < ch.n_seg) sg = seg_scratch[ch.seg_begin - seg_base + lane];
        const int it = (int)(base + k - cb);
        const int s = it % kStages;
        const uint32_t ph = (uint32_t)(it / kStages) & 1u;
        // per-segment x placement (prefix over lanes)
        const double* xsrc = arena + sg.x_off;
        const uint32_t xb = lane < ch.n_seg ? span_bytes(xsrc, sg.ncols) : 0u;
        uint32_t xpos = xb;  // inclusive scan of bytes
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(0xffffffffu, xpos, o);
          if (lane >= o) xpos += v;
        }
        const uint32_t x_total = __shfl_sync(0xffffffffu, xpos, 31);
        xpos -= xb;  // exclusive
        int ccol = sg.ncols;  // column prefix
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, ccol, o);
          if (lane >= o) ccol += v;
        }
        ccol -= sg.ncols;
        double* sA = stage_buf + (size_t)s * kStageDoubles;
        double* sX = sA + kStageA;
        StageHdr* h = reinterpret_cast<StageHdr*>(reinterpret_cast<char*>(hdr) + s * kHdrBytes);
        if (lane == 0) mbar_wait(&empty[s], ph ^ 1u);
        __syncwarp();
        if (lane < ch.n_seg) {
          h->seg_c0[lane] = (int16_t)ccol;
          h->seg_x[lane] = (int16_t)(xpos / 8 + dshift(xsrc));
        }
        __syncwarp();  // segment table before lane 0's release (arrive) below
        const bool strided = ch.lda != ch.m;
        const double* a0 = blob + ch.a_off;
        uint32_t a_total = 0;
        if (!strided) {
          a_total = ch.ncols > 0 ? span_bytes(a0, ch.m * ch.ncols) : 0u;
        } else {
          for (int c = lane; c < ch.ncols; c += 32)
            a_total += span_bytes(a0 + (int64_t)c * ch.lda, ch.m);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) a_total += __shfl_xor_sync(0xffffffffu, a_total, o);
        }
        const int ldas = strided ? ((ch.m + 1) & ~1) + 2 : ch.m;
        if (lane == 0) {
          h->y_off = ch.y_off;
          h->m = ch.m;
          h->ncols = ch.ncols;
          h->flags = ch.flags;
          h->n_seg = ch.n_seg;
          h->ldas = ldas;
          h->strided = strided;
          h->odd_lda = strided && (ch.lda & 1);
          h->a_shift = dshift(a0);
          h->a_shift0 = dshift(a0);
          mbar_arrive_expect_tx(&full[s], a_total + x_total);
        }
        __syncwarp();
        // issue the copies: x segments by their lanes, operator data by lane 0
        // (contiguous) or by column-strided lanes (strided)
        if (lane < ch.n_seg && sg.ncols > 0)
          bulk_g2s(reinterpret_cast<char*>(sX) + xpos, align_down(xsrc), xb, &full[s]);
        if (!strided) {
          if (lane == 0 && a_total) bulk_g2s(sA, align_down(a0), a_total, &full[s]);
        } else {
          for (int c = lane; c < ch.ncols; c += 32) {
            const double* src = a0 + (int64_t)c * ch.lda;
            bulk_g2s(sA + (size_t)c * ldas, align_down(src), span_bytes(src, ch.m), &full[s]);
          }
        }
        __syncwarp();
      }
      cur = nxt;
      if (base + 64 + lane < ce) nxt = chunks[base + 64 + lane];
    }
    return;
  }

  // ---------------------------------------------------- consumers
  const int cw = warp - 1;
  double acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.0;
  for (int64_t i = cb; i < ce; ++i) {
    const int it = (int)(i - cb);
    const int s = it % kStages;
    const uint32_t ph = (uint32_t)(it / kStages) & 1u;
    mbar_wait(&full[s], ph);
    const StageHdr& h = *reinterpret_cast<const StageHdr*>(reinterpret_cast<const char*>(hdr) +
                                                           s * kHdrBytes);
    const double* sA = stage_buf + (size_t)s * kStageDoubles;
    const double* sX = sA + kStageA;
    const int m = h.m;
    if (h.ncols > 0) {
      if (!h.odd_lda) {
        const int J = (m + 31) >> 5;
        switch (J) {
          case 1: consume_stage<1>(h, sA, sX, lane, cw, acc); break;
          case 2: consume_stage<2>(h, sA, sX, lane, cw, acc); break;
          case 3: consume_stage<3>(h, sA, sX, lane, cw, acc); break;
          case 4: consume_stage<4>(h, sA, sX, lane, cw, acc); break;
          default: consume_stage<8>(h, sA, sX, lane, cw, acc); break;
        }
      } else {
        // strided run with odd lda (rare): the alignment shift alternates per column
        const double* xs = sX + h.seg_x[0];
        for (int c = cw; c < h.ncols; c += kConsumers) {
          const int sh = (h.a_shift0 + c) & 1;
          const double* col = sA + (size_t)c * h.ldas + sh;
          const double xv = xs[c];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int rr = lane + 32 * j;
            if (rr < m) acc[j] = fma(col[rr], xv, acc[j]);
          }
        }
      }
    }
    const int flags = h.flags;
    const int64_t y_off = h.y_off;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (flags & kLastOfTask) {
      // fixed-order cross-warp reduction, one store per output
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int rr = lane + 32 * j;
        if (rr < m) red[cw * kStreamMaxRows + rr] = acc[j];
        acc[j] = 0.0;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
      double* y = arena + y_off;
      for (int rr = threadIdx.x - 32; rr < m; rr += kConsumers * 32) {
        double sum = red[rr];
#pragma unroll
        for (int w = 1; w < kConsumers; ++w) sum += red[w * kStreamMaxRows + rr];
        y[rr] = sum;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
    }
  }
}

}  // namespace h2g
