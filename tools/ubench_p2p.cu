// Microbenchmark of the P2P (kernel-evaluation) engine on synthetic task
// lists shaped like config 3's M2L levels:
//   l5: 32768 targets, ~32 rows, ~119 blocks of ~32 columns   (leaf level)
//   l4:  4096 targets, ~113 rows, ~93 blocks of ~113 columns
// A share 1 - s of every target's block entries is stored (TMA-staged from a
// blob far larger than L2), the rest evaluated (1/r, 3D).  Runs the real
// kernel of csrc/h2g_p2p.cuh; compile-time variants through -D macros:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        --expt-relaxed-constexpr -I include -o ubench_p2p tools/ubench_p2p.cu
//   ./ubench_p2p l5r 0.6
// -DUB_OLD / -DUB_R01 build against earlier revisions of the kernel header for
// comparison (git show <rev>:paper_2309_14085_b200/csrc/h2g_p2p.cuh into
// scratch/old/h2g_p2p_old.cuh resp. scratch/r01/h2g_p2p_r01.cuh, -I that dir).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <random>
#include <vector>

#include <cuda_runtime.h>

#if defined(UB_R01)
#include "h2g_stream.cuh"
#include "h2g_p2p_r01.cuh"   // round-1 kernel (no stages): evaluation-only comparisons
namespace h2g { struct P2PStage { uint64_t src; int64_t x_off; uint32_t bytes; int16_t ncols, shift; }; }
#elif defined(UB_OLD)
#include "h2g_p2p_old.cuh"
#else
#include "../paper_2309_14085_b200/csrc/h2g_p2p.cuh"
#endif

using namespace h2g;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

__global__ void fill(double* p, size_t n, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v * (double)((i * 2654435761ull) % 1024) / 1024.0;
}

int main(int argc, char** argv) {
  const char* level = argc > 1 ? argv[1] : "l5";
  const double share = argc > 2 ? atof(argv[2]) : 1.0;
  const int reps = argc > 3 ? atoi(argv[3]) : 5;
  // lN: uniform synthetic tasks; lNr: the shape of config 3's level N as the
  // native build produces it (two channels per target: ~100 and ~6 source
  // blocks; ranks spread around their mean; one stored L2L block per task)
  int T, m_lo, m_hi, nb, c_lo, c_hi, nb2 = 0, l2l = 0;
  if (!strcmp(level, "l5")) {
    T = 32768; m_lo = 24; m_hi = 40; nb = 119; c_lo = 24; c_hi = 40;
  } else if (!strcmp(level, "l4")) {
    T = 4096; m_lo = 100; m_hi = 126; nb = 93; c_lo = 100; c_hi = 126;
  } else if (!strcmp(level, "l5r")) {
    T = 32768; m_lo = 15; m_hi = 53; nb = 100; c_lo = 15; c_hi = 53; nb2 = 6; l2l = 100;
  } else if (!strcmp(level, "l4r")) {
    T = 4096; m_lo = 71; m_hi = 116; nb = 78; c_lo = 71; c_hi = 116; nb2 = 5; l2l = 100;
  } else if (!strcmp(level, "l5c")) {  // config 5's leaf level: leaves of ~64 points
    T = 32768; m_lo = 48; m_hi = 64; nb = 119; c_lo = 48; c_hi = 64;
  } else {  // l5x: exact 32 x 32 blocks
    T = 32768; m_lo = 32; m_hi = 32; nb = 119; c_lo = 32; c_hi = 32;
  }
  std::mt19937_64 rng(7);
  // triangular around the middle of [lo, hi] (ranks cluster around their mean)
  auto uni = [&](int lo, int hi) {
    const int w = hi - lo + 1;
    return lo + (int)((rng() % (uint64_t)w + rng() % (uint64_t)w) / 2);
  };
  const int64_t n_rec = 1 << 22, n_arena = (1 << 23) + (int64_t)T * 512;
  const int64_t y_base = 1 << 23;
  std::vector<P2PTask> tasks;
  std::vector<P2PChunk> chunks;
  std::vector<P2PStage> stages;
  double* d_blob = nullptr;
  const size_t blob_doubles = (size_t)12 << 27;  // 12 GiB
  CK(cudaMalloc(&d_blob, blob_doubles * 8));
  fill<<<148 * 8, 256>>>(d_blob, blob_doubles, 1e-3);
  size_t boff = 0;
  double n_eval = 0, n_stream = 0;
  struct Blk { int nc; int64_t x_off; bool stored; int32_t rec; };
  std::vector<std::pair<double, std::vector<Blk>>> protos;  // (cost, blocks) per task
  std::vector<int> proto_m;
  for (int t = 0; t < T; ++t) {
    const int m = uni(m_lo, m_hi);
    for (int ch = 0; ch < (nb2 ? 2 : 1); ++ch) {
      const int nblk = ch == 0 ? nb + (nb2 ? (int)(rng() % 21) - 10 : 0) : nb2;
      std::vector<Blk> bl;
      double tot = 0, str = 0;
      for (int b = 0; b < nblk; ++b) {
        Blk k;
        k.nc = uni(c_lo, c_hi);
        k.x_off = (int64_t)(rng() % (uint64_t)((1 << 23) - 256));
        const double e = (double)m * k.nc;
        tot += e;
        k.stored = share < 1.0 && str + e <= (1.0 - share) * tot + 0.5 * e;  // error diffusion
        if (k.stored) str += e;
        k.rec = (int32_t)(n_rec / 2 + rng() % (uint64_t)(n_rec / 2 - 256));  // columns: second half
        bl.push_back(k);
      }
      if (l2l && share < 1.0) {  // the task's L2L block: stored, staged with the M2L share
        Blk k;
        k.nc = l2l + (int)(rng() % 21) - 10;
        k.x_off = (int64_t)(rng() % (uint64_t)((1 << 23) - 256));
        k.stored = true;
        k.rec = 0;
        bl.push_back(k);
        tot += (double)m * k.nc;
      }
      protos.push_back({tot, std::move(bl)});
      proto_m.push_back(m);
    }
  }
  std::vector<int> order(protos.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return protos[a].first > protos[b].first; });  // largest first
  const int n_tasks = (int)order.size();
  for (int oi = 0; oi < n_tasks; ++oi) {
    const int t = order[oi];
    P2PTask q{};
    q.m = proto_m[t];
    q.y_off = y_base + (int64_t)oi * 256;
    q.row_rec = (int32_t)(rng() % (uint64_t)(n_rec / 2 - 256));  // rows: first half of the records
    q.k_begin = (int32_t)chunks.size();
#ifndef UB_R01
    q.s_begin = (int32_t)stages.size();
#endif
    for (const Blk& k : protos[t].second) {
      const int nc = k.nc;
      const int64_t x_off = k.x_off;
      const double e = (double)q.m * nc;
      if (k.stored) {
        n_stream += e;
        if (boff + (size_t)q.m * nc + 2 > blob_doubles) boff = 0;
#if defined(UB_R01)
        fprintf(stderr, "the round-1 kernel has no stages: share must be 1\n");
        return 1;
#elif defined(UB_OLD)
        const int64_t cc = std::max<int64_t>(1, (kP2PStageBytes - 16) / (8 * (int64_t)q.m));
        for (int64_t c0 = 0; c0 < nc; c0 += cc) {
          const int64_t n1 = std::min<int64_t>(cc, nc - c0);
          const uint64_t src = reinterpret_cast<uint64_t>(d_blob + boff + c0 * q.m);
          const uint64_t a = src & ~uint64_t(15);
          const uint64_t en = (src + 8ull * (uint64_t)(q.m * n1) + 15) & ~uint64_t(15);
          P2PStage st{};
          st.src = a; st.x_off = x_off + c0; st.bytes = (uint32_t)(en - a);
          st.ncols = (int16_t)n1; st.shift = (int16_t)((src - a) / 8);
          stages.push_back(st);
        }
#else
        p2p_cut_stages(d_blob + boff, q.m, nc, x_off, stages);
#endif
        boff += (size_t)q.m * nc;
        continue;
      }
      n_eval += e;
      for (int c0 = 0; c0 < nc; c0 += kP2PChunk) {
        P2PChunk c;
        c.x_off = x_off + c0;
        c.rec = k.rec + c0;
        c.n_self = std::min(kP2PChunk, nc - c0);
        chunks.push_back(c);
      }
    }
    q.k_end = (int32_t)chunks.size();
#ifndef UB_R01
    q.s_end = (int32_t)stages.size();
#endif
    tasks.push_back(q);
  }
  T = n_tasks;
  std::vector<double4> recs(n_rec);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  for (auto& r : recs) r = make_double4(U(rng), U(rng), U(rng), 0.0);
  P2PTask* d_tasks; P2PChunk* d_chunks; P2PStage* d_stages; double4* d_recs; double* d_arena; int* d_ctr;
  Term* d_terms;
  CK(cudaMalloc(&d_tasks, tasks.size() * sizeof(P2PTask)));
  CK(cudaMalloc(&d_chunks, (chunks.size() + 1) * sizeof(P2PChunk)));
  CK(cudaMalloc(&d_stages, (stages.size() + 1) * sizeof(P2PStage)));
  CK(cudaMalloc(&d_recs, recs.size() * sizeof(double4)));
  CK(cudaMalloc(&d_arena, (n_arena + 8) * 8));
  CK(cudaMalloc(&d_ctr, 8));
  CK(cudaMalloc(&d_terms, 64));
  CK(cudaMemcpy(d_tasks, tasks.data(), tasks.size() * sizeof(P2PTask), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_chunks, chunks.data(), chunks.size() * sizeof(P2PChunk), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_stages, stages.data(), stages.size() * sizeof(P2PStage), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_recs, recs.data(), recs.size() * sizeof(double4), cudaMemcpyHostToDevice));
  CK(cudaMemset(d_ctr, 0, 8));
  fill<<<148 * 8, 256>>>(d_arena, n_arena, 1.0);
  CK(cudaDeviceSynchronize());
  P2PKernel kp{};
#if defined(UB_R01)
  auto kfn = p2p_tasks_kernel<1, 3>;
  const size_t smem = 0;
  const int threads = kP2PThreads, per_sm = kP2PCtasPerSm;
#elif defined(UB_OLD)
  auto kfn = p2p_tasks_kernel<1, 3, false>;
  const size_t smem = kP2PSmem;
  const int threads = kP2PThreads, per_sm = kP2PCtasPerSm;
#else
  // a streaming warp per CTA when the tasks have TMA stages (as launch_p2p does)
  const bool sw = !stages.empty();
  auto kfn = sw ? p2p_tasks_kernel<1, 3, false, true> : p2p_tasks_kernel<1, 3, false, false>;
  const size_t smem = p2p_smem_bytes(sw);
  const int threads = sw ? kP2PThreadsSW : kP2PThreads, per_sm = sw ? kP2PCtasSW : kP2PCtasPerSm;
#endif
  CK(cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, threads, smem));
  const unsigned grid = 148 * per_sm;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f, sum = 0;
  for (int r = 0; r < reps + 2; ++r) {
    CK(cudaEventRecord(e0));
#if defined(UB_R01)
    kfn<<<grid, threads, smem>>>(d_tasks, T, d_terms, d_chunks, d_recs, d_blob, d_arena, kp, d_ctr);
#else
    kfn<<<grid, threads, smem>>>(d_tasks, T, d_terms, d_chunks, d_stages, d_recs, d_blob,
                                          d_arena, kp, d_ctr);
#endif
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (r >= 2) { best = std::min(best, ms); sum += ms; }
  }
  // checksum of the outputs (identical across layout variants up to summation order)
  std::vector<double> y((size_t)T * 256);  // (T tasks, 256 slots each)
  CK(cudaMemcpy(y.data(), d_arena + y_base, y.size() * 8, cudaMemcpyDeviceToHost));
  double cs = 0;
  for (int t = 0; t < T; ++t)
    for (int r = 0; r < tasks[t].m; ++r) cs += y[(size_t)t * 256 + r];
  const double ms = sum / reps;
  printf("{\"level\": \"%s\", \"share\": %.2f, \"ms\": %.4f, \"best_ms\": %.4f, \"occ\": %d, "
         "\"eval_entries\": %.4g, \"stream_entries\": %.4g, \"eval_Tps\": %.4f, \"stream_GBps\": %.1f, "
         "\"total_Tps\": %.4f, \"stages\": %zu, \"chunks\": %zu, \"checksum\": %.12e}\n",
         level, share, ms, best, occ, n_eval, n_stream, n_eval / ms / 1e9, 8 * n_stream / ms / 1e6,
         (n_eval + n_stream) / ms / 1e9, stages.size(), chunks.size(), cs);
  return 0;
}
