// h2g_p2p_batched.cuh — batched-RHS kernel-evaluation engine (sm_100a).
//
// Multi-RHS products of plans with kernel-evaluated blocks (the only form in
// which BASELINE config 5 fits, and config 4's Gaussian blocks): every entry
// K[t_i(X), s_o(Y)] / K[t^X, t^Y] (reference engine.py:176-179, 309-318;
// entry rule kernels.py:36-57) is evaluated ONCE and multiplied with all KB
// right-hand sides -- 11 fp64 instructions per entry for 1/r plus KB
// multiply-adds, against KB x 12 for a loop over the columns.
//
// Work lists are those of the single-RHS P2P engine (h2g_p2p.cuh: P2PTask /
// P2PChunk, stored terms as direct loads, no TMA stages); vectors live in the
// batched arena of the tensor-pipe engine (h2g_kernels.cuh): RHS b of slot s
// at (b >> 3) * ps + 8 s + (b & 7).
//
// Mapping: one CTA (4 warps) per task, fetched dynamically; rows in blocks of
// kPBRows; inside a warp lanes form G = 32 / L groups of L, lane (g, l) owns
// rows l + L j (j < 2) of the block and the chunk's columns g, g + G, ...,
// with 2 x KB accumulators.  A chunk's point records and its X (columns x
// KB) are staged through a per-warp smem double buffer by cp.async.  Groups
// are combined by a fixed xor tree, warps in warp order through smem:
// deterministic, no atomics on data.
#pragma once
#include <cstdint>

#include "h2g_p2p.cuh"

namespace h2g {

constexpr int kPBWarps = 4;
constexpr int kPBThreads = 32 * kPBWarps;
constexpr int kPBRows = 64;          // rows per pass (2 per lane x 32 lanes at most)
#ifndef H2G_PB_CTAS
#define H2G_PB_CTAS 3
#endif
constexpr int kPBCtasPerSm = H2G_PB_CTAS;

template <int KB>
constexpr size_t p2p_batched_smem() {
  return (size_t)kPBWarps * 2 * kP2PChunk * (32 + 8 * KB) +  // records + X double buffers
         (size_t)kPBWarps * kPBRows * KB * 8 + 16;            // cross-warp reduction
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int KT, int DIM, bool FULL, int KB>
__global__ void __launch_bounds__(kPBThreads, kPBCtasPerSm)
p2p_batched_kernel(const P2PTask* __restrict__ tasks, int n_tasks, const Term* __restrict__ terms,
                   const P2PChunk* __restrict__ chunks, const double4* __restrict__ recs,
                   const double* __restrict__ blob, double* arena, int64_t ps, P2PKernel kp,
                   int* ctr) {
  constexpr int NP = KB / 8;  // planes
  extern __shared__ __align__(128) double pb_smem[];
  // per warp: [2][32] records (double4), [2][NP][32][8] X
  double4* srec_all = reinterpret_cast<double4*>(pb_smem);
  double* sx_all = reinterpret_cast<double*>(srec_all + kPBWarps * 2 * kP2PChunk);
  double* red = sx_all + (size_t)kPBWarps * 2 * kP2PChunk * KB;
  int* s_task = reinterpret_cast<int*>(red + (size_t)kPBWarps * kPBRows * KB);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double4* srec = srec_all + warp * 2 * kP2PChunk;
  double* sx = sx_all + (size_t)warp * 2 * kP2PChunk * KB;

  // stage chunk cd into buffer `buf`: lane c copies record c and its X rows
  auto stage_chunk = [&](const P2PChunk& cd, int buf) {
    const int n = cd.n_self & 0xffff;
    if (lane < n) {
      const char* r = reinterpret_cast<const char*>(recs + cd.rec + lane);
      char* d = reinterpret_cast<char*>(srec + buf * kP2PChunk + lane);
      cp_async16(d, r);
      cp_async16(d + 16, r + 16);
#pragma unroll
      for (int pl = 0; pl < NP; ++pl) {
        const char* xs = reinterpret_cast<const char*>(arena + pl * ps + 8 * (cd.x_off + lane));
        char* xd = reinterpret_cast<char*>(sx + ((size_t)(buf * NP + pl) * kP2PChunk + lane) * 8);
#pragma unroll
        for (int h = 0; h < 4; ++h) cp_async16(xd + 16 * h, xs + 16 * h);
      }
    }
    cp_async_commit();
  };

  for (;;) {
    if (threadIdx.x == 0) *s_task = atomicAdd(ctr, 1);
    __syncthreads();
    const int t = *s_task;
    if (t >= n_tasks) break;
    const P2PTask tk = tasks[t];
    const int m = tk.m;
    const int64_t row0 = tk.row_rec;
    for (int rb = 0; rb < m; rb += kPBRows) {
      const int mr = min(kPBRows, m - rb);  // rows of this pass
      int L = 4;
      while (L < 32 && 2 * L < mr) L <<= 1;
      const int G = 32 / L;
      const int g = lane / L, rl = lane % L;
      double px[2], py[2], pz[2];
      double acc[2][KB];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = min(rb + rl + L * j, m - 1);
        double4 p = make_double4(0, 0, 0, 0);
        if (row0 >= 0) p = recs[row0 + r];  // tasks without evaluated chunks have no row records
        px[j] = p.x;
        py[j] = p.y;
        pz[j] = p.z;
#pragma unroll
        for (int b = 0; b < KB; ++b) acc[j][b] = 0.0;
      }
      // ---- evaluated chunks k = k_begin + warp, + kPBWarps, ...
      int k = tk.k_begin + warp;
      int buf = 0;
      P2PChunk cd{}, cn{};
      if (k < tk.k_end) {
        cd = chunks[k];
        stage_chunk(cd, 0);
      }
      while (k < tk.k_end) {
        const int kn = k + kPBWarps;
        if (kn < tk.k_end) {  // next chunk in flight during the evaluation
          cn = chunks[kn];
          stage_chunk(cn, buf ^ 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncwarp();
        const int n = cd.n_self & 0xffff;
        const bool self = FULL && (cd.n_self & kSelfBit) != 0;
        const int64_t col0 = cd.rec;
        const double4* sr = srec + buf * kP2PChunk;
        const double* sxb = sx + (size_t)buf * NP * kP2PChunk * 8;
        for (int c = g; c < n; c += G) {
          const double4 s = sr[c];
          double kv[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const double r2 = dist2<DIM>(px[j], py[j], pz[j], s);
            double v = kfun<KT>(r2, kp);
            if (FULL) {
              v = r2 == 0.0 ? kp.zero_value : v;
              if (self) v = (row0 + rb + rl + L * j == col0 + c) ? kp.self_value : v;
            }
            kv[j] = v;
          }
#pragma unroll
          for (int pl = 0; pl < NP; ++pl) {
            const double2* xr = reinterpret_cast<const double2*>(sxb + ((size_t)pl * kP2PChunk + c) * 8);
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const double2 x2 = xr[h];
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                acc[j][pl * 8 + 2 * h] = fma(kv[j], x2.x, acc[j][pl * 8 + 2 * h]);
                acc[j][pl * 8 + 2 * h + 1] = fma(kv[j], x2.y, acc[j][pl * 8 + 2 * h + 1]);
              }
            }
          }
        }
        __syncwarp();  // the buffer is refilled two chunks later
        cd = cn;
        k = kn;
        buf ^= 1;
      }
      // ---- stored terms (L2L, L2P, BLR U, stored blocks): columns dealt over
      // (warp, lane group) pairs, direct loads
      for (int ti = tk.t_begin; ti < tk.t_end; ++ti) {
        const Term tm = terms[ti];
        const double* A = (tm.a_space ? arena : blob) + tm.a_off;
        // a_space 1 (split-K partials) never reaches the batched P2P lists: those
        // reduce tasks run in the reduce kernel (ensure_batched)
        for (int c = warp * G + g; c < tm.ncols; c += kPBWarps * G) {
          const double* col = A + (int64_t)c * tm.lda;
          double a[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int r = rb + rl + L * j;
            a[j] = r < m ? ld_stream(col + r) : 0.0;
          }
#pragma unroll
          for (int pl = 0; pl < NP; ++pl) {
            const double2* xr = reinterpret_cast<const double2*>(arena + pl * ps + 8 * (tm.x_off + c));
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const double2 x2 = xr[h];
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                acc[j][pl * 8 + 2 * h] = fma(a[j], x2.x, acc[j][pl * 8 + 2 * h]);
                acc[j][pl * 8 + 2 * h + 1] = fma(a[j], x2.y, acc[j][pl * 8 + 2 * h + 1]);
              }
            }
          }
        }
      }
      // ---- combine: lane groups by a fixed xor tree, warps in warp order
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int b = 0; b < KB; ++b)
          for (int off = L; off < 32; off <<= 1)
            acc[j][b] += __shfl_xor_sync(0xffffffffu, acc[j][b], off);
      if (g == 0) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int r = rl + L * j;  // row inside the pass
          if (r < mr) {
            double2* d = reinterpret_cast<double2*>(red + ((size_t)warp * kPBRows + r) * KB);
#pragma unroll
            for (int h = 0; h < KB / 2; ++h) d[h] = make_double2(acc[j][2 * h], acc[j][2 * h + 1]);
          }
        }
      }
      __syncthreads();
      for (int i = threadIdx.x; i < mr * KB; i += kPBThreads) {
        const int r = i / KB, b = i % KB;
        double sum = red[(size_t)r * KB + b];
#pragma unroll
        for (int w = 1; w < kPBWarps; ++w) sum += red[((size_t)w * kPBRows + r) * KB + b];
        arena[(b >> 3) * ps + 8 * (tk.y_off + rb + r) + (b & 7)] = sum;
      }
      __syncthreads();  // red reuse
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

// Launch interface (h2g_p2p_launch.cu).
cudaError_t p2p_batched_launch(int kt, int dim, bool full, int kb, int n_sm, cudaStream_t s,
                               const P2PTask* tasks, int n_tasks, const Term* terms,
                               const P2PChunk* chunks, const double4* recs, const double* blob,
                               double* arena, int64_t ps, const P2PKernel& kp, int* ctr);

}  // namespace h2g
