// h2g_kernels.cuh — device code of the H2* / (H2+H)* matvec (sm_100a).
//
// Every phase of the reference MVP (engine.py:190-269) is a batch of
// gather-by-target GEMV *tasks*: task t owns a disjoint output slice
// y[0:m) of the coefficient arena and computes
//
//     y = sum_{terms k of t}  A_k (m x ncols_k, column-major, leading dim lda_k)
//                               * x_k (ncols_k contiguous arena slots)
//
// P2M, M2M, M2L(+L2L), L2P, the BLR leg and the near field are all instances
// (see h2g_plan.cu for the mapping).  One CTA runs one task; its warps split
// each term's columns in groups of kUnroll, every lane owns rows lane+32j, so
// each column is read with one coalesced request per 32 rows and no
// cross-lane reduction is needed.  Warps are combined through shared memory
// in a fixed order and the result is stored once: no atomics, deterministic
// summation order (SURVEY.md §7 hard part 2).
#pragma once
#include <cstdint>

namespace h2g {

struct Task {          // 24 bytes
  int64_t y_off;       // arena slot of y[0]
  int32_t m;           // rows (<= kMaxRows)
  int32_t t_begin;     // term range [t_begin, t_end) -- int32 is enough per phase
  int32_t t_end;
  int32_t pad;
};

struct Term {          // 32 bytes
  int64_t a_off;       // offset (doubles) of A(0, 0) in the blob (a_space 0) or arena (1)
  int64_t x_off;       // arena slot of x[0]
  int32_t lda;         // column stride of A in doubles
  int32_t ncols;
  int32_t a_space;     // 0: operator blob, 1: coefficient arena (split-K partials)
  int32_t pad;
};

constexpr int kMaxJ = 8;         // rows per lane -> m <= 256 per task
constexpr int kMaxRows = 32 * kMaxJ;
constexpr int kWarps = 4;        // warps per CTA (one task per CTA)
constexpr int kUnroll = 4;       // columns in flight per warp iteration

__device__ __forceinline__ double ld_stream(const double* p) {
  // operator entries are touched exactly once per matvec: evict-first
  return __ldcs(p);
}

template <int J>
__device__ __forceinline__ void term_accumulate(const double* __restrict__ A, int lda,
                                                int ncols, const double* __restrict__ x,
                                                int m, int lane, int warp, double (&acc)[J]) {
  // warp w takes column groups [g*kUnroll, g*kUnroll + kUnroll) with g = w, w+kWarps, ...
  for (int c0 = warp * kUnroll; c0 < ncols; c0 += kWarps * kUnroll) {
    double a[kUnroll][J];
    double xv[kUnroll];
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
      const int c = c0 + k;
      const bool cv = c < ncols;
      xv[k] = cv ? __ldg(x + c) : 0.0;
      const double* col = A + (int64_t)c * lda;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int r = lane + 32 * j;
        a[k][j] = (cv && r < m) ? ld_stream(col + r) : 0.0;
      }
    }
#pragma unroll
    for (int k = 0; k < kUnroll; ++k)
#pragma unroll
      for (int j = 0; j < J; ++j) acc[j] = fma(a[k][j], xv[k], acc[j]);
  }
}

template <int J>
__device__ __forceinline__ void run_task(const Task& tk, const Term* __restrict__ terms,
                                         const double* __restrict__ blob, double* arena,
                                         double* red /* smem [kWarps][32*J] */) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double acc[J];
#pragma unroll
  for (int j = 0; j < J; ++j) acc[j] = 0.0;
  for (int t = tk.t_begin; t < tk.t_end; ++t) {
    const Term tm = terms[t];
    term_accumulate<J>((tm.a_space ? arena : blob) + tm.a_off, tm.lda, tm.ncols, arena + tm.x_off,
                       tk.m, lane, warp, acc);
  }
#pragma unroll
  for (int j = 0; j < J; ++j) red[warp * (32 * J) + lane + 32 * j] = acc[j];
  __syncthreads();
  double* y = arena + tk.y_off;
  for (int r = threadIdx.x; r < tk.m; r += blockDim.x) {
    double s = red[r];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) s += red[w * (32 * J) + r];
    y[r] = s;
  }
}

// One CTA per task.  Rows-per-lane J is chosen per task at run time and
// dispatched to a compile-time instance so accumulators stay in registers.
static __global__ void __launch_bounds__(kWarps * 32)
gemv_tasks_kernel(const Task* __restrict__ tasks, const Term* __restrict__ terms,
                  const double* __restrict__ blob, double* arena) {
  __shared__ double red[kWarps * kMaxRows];
  const Task tk = tasks[blockIdx.x];
  const int J = (tk.m + 31) >> 5;
  if (J <= 1)      run_task<1>(tk, terms, blob, arena, red);
  else if (J == 2) run_task<2>(tk, terms, blob, arena, red);
  else if (J <= 4) run_task<4>(tk, terms, blob, arena, red);
  else             run_task<8>(tk, terms, blob, arena, red);
}

// q_tree[i] = q[perm[i] * ld]  (tree order gather, reference q[index_set])
static __global__ void gather_perm_kernel(const double* __restrict__ q, int64_t ld,
                                   const int32_t* __restrict__ perm, double* __restrict__ out,
                                   int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = q[(int64_t)perm[i] * ld];
}

// phi[perm[i] * ld] = phi_tree[i]  (reference phi[index_set] +=, disjoint slices)
static __global__ void scatter_perm_kernel(const double* __restrict__ in,
                                    const int32_t* __restrict__ perm, double* __restrict__ phi,
                                    int64_t ld, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    phi[(int64_t)perm[i] * ld] = in[i];
}

// Batched-RHS arena: KB / 8 planes of 8 doubles per slot; RHS b of slot s at
// (b >> 3) * ps + 8 s + (b & 7) (h2g_stream.cuh, stream_mma_kernel).
// batched RHS: q_tree (slot i of the planes at `out`) = q[perm[i] * ld + col0 + b]
// (thread = one (slot, RHS) pair, RHS fastest: a row of q is read as one
// contiguous run of KB doubles and lands as contiguous 64-byte plane rows)
template <int KB>
__global__ void gather_batch_kernel(const double* __restrict__ q, int64_t ld, int64_t col0,
                                    int nb, const int32_t* __restrict__ perm,
                                    double* __restrict__ out, int64_t n, int64_t ps) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * KB;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / KB;
    const int b = (int)(t % KB);
    out[(b >> 3) * ps + i * 8 + (b & 7)] = b < nb ? q[(int64_t)perm[i] * ld + col0 + b] : 0.0;
  }
}

// batched RHS: phi[perm[i] * ld + col0 + b] = phi_tree (planes at `in`), b < nb
template <int KB>
__global__ void scatter_batch_kernel(const double* __restrict__ in,
                                     const int32_t* __restrict__ perm, double* __restrict__ phi,
                                     int64_t ld, int64_t col0, int nb, int64_t n, int64_t ps) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * KB;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / KB;
    const int b = (int)(t % KB);
    if (b < nb) phi[(int64_t)perm[i] * ld + col0 + b] = in[(b >> 3) * ps + i * 8 + (b & 7)];
  }
}

// multi-GPU exchange: copy (src, dst, len) slot ranges between buffers
struct CopyRange {
  int64_t src, dst, len;
};

static __global__ void copy_ranges_kernel(const CopyRange* __restrict__ r, int n,
                                   const double* __restrict__ src, double* __restrict__ dst) {
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const CopyRange c = r[k];
    for (int64_t i = threadIdx.x; i < c.len; i += blockDim.x) dst[c.dst + i] = src[c.src + i];
  }
}

// Split-K reduce for the batched-RHS arena (KB values per slot): y = sum of
// the task's P partial blocks in piece order (the batched form of the
// [partials] * ones GEMV task of the single-RHS schedule).
struct RedTask {
  int64_t y_off;       // slot of y[0]
  int64_t part;        // slot of partial 0, row 0 (partial p at part + p * m)
  int32_t m;
  int32_t P;
};

template <int KB>
__global__ void reduce_partials_kernel(const RedTask* __restrict__ t, int n,
                                       double* __restrict__ arena, int64_t ps) {
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const RedTask r = t[k];
    const int64_t len = (int64_t)r.m * 8;  // per plane
    for (int64_t i = threadIdx.x; i < len * (KB / 8); i += blockDim.x) {
      const int64_t pl = i / len, ii = i - pl * len;
      const double* src = arena + pl * ps + r.part * 8 + ii;
      double acc = 0.0;
      for (int p = 0; p < r.P; ++p) acc += src[(int64_t)p * len];
      arena[pl * ps + r.y_off * 8 + ii] = acc;
    }
  }
}

// phi[perm[i] * ld] = phi_tree[i] for tree rows i in [i0, i1) (owned rows)
static __global__ void scatter_rows_kernel(const double* __restrict__ in, const int32_t* __restrict__ perm,
                                    double* __restrict__ phi, int64_t ld, int64_t i0, int64_t i1) {
  for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < i1;
       i += (int64_t)gridDim.x * blockDim.x)
    phi[(int64_t)perm[i] * ld] = in[i];
}

}  // namespace h2g
