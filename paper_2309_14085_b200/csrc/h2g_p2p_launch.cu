// h2g_p2p_launch.cu — instantiation and launch of the P2P (kernel-evaluation)
// engine's kernels (h2g_p2p.cuh), as their own translation unit so the two
// halves of libh2g.so compile in parallel.
#include <algorithm>

#include <cuda_runtime.h>

#include "h2g_p2p.cuh"
#include "h2g_p2p_batched.cuh"

namespace h2g {

namespace {

template <int KT, int DIM, bool FULL, bool SW>
cudaError_t configure_one() {
  auto k = p2p_tasks_kernel<KT, DIM, FULL, SW>;
  // maximum shared-memory carve-out (L1 is not what these kernels need)
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)p2p_smem_bytes(SW));
}

template <int KT, int DIM>
cudaError_t configure_kd() {
  cudaError_t e;
  if ((e = configure_one<KT, DIM, true, false>()) != cudaSuccess) return e;
  if ((e = configure_one<KT, DIM, false, false>()) != cudaSuccess) return e;
  return configure_one<KT, DIM, false, true>();
}

template <int KT, int DIM, bool FULL, bool SW>
cudaError_t launch_one(bool pdl, unsigned grid, cudaStream_t s, const P2PTask* tasks, int n_tasks,
                       const Term* terms, const P2PChunk* chunks, const P2PStage* stages,
                       const double4* recs, const double* blob, double* arena,
                       const P2PKernel& kp, int* ctr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(SW ? kP2PThreadsSW : kP2PThreads);
  cfg.dynamicSmemBytes = p2p_smem_bytes(SW);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, p2p_tasks_kernel<KT, DIM, FULL, SW>, tasks, n_tasks, terms,
                            chunks, stages, recs, blob, arena, kp, ctr);
}

template <int KT, int DIM>
cudaError_t launch_kd(bool full, bool sw, bool pdl, unsigned grid, cudaStream_t s,
                      const P2PTask* tasks, int n_tasks, const Term* terms, const P2PChunk* chunks,
                      const P2PStage* stages, const double4* recs, const double* blob,
                      double* arena, const P2PKernel& kp, int* ctr) {
  // phases with self blocks never stage (build_p2p_lists): FULL has no streaming warp
  if (full)
    return launch_one<KT, DIM, true, false>(pdl, grid, s, tasks, n_tasks, terms, chunks, stages,
                                            recs, blob, arena, kp, ctr);
  if (sw)
    return launch_one<KT, DIM, false, true>(pdl, grid, s, tasks, n_tasks, terms, chunks, stages,
                                            recs, blob, arena, kp, ctr);
  return launch_one<KT, DIM, false, false>(pdl, grid, s, tasks, n_tasks, terms, chunks, stages,
                                           recs, blob, arena, kp, ctr);
}

template <int KT, int DIM, bool FULL, int KB>
cudaError_t configure_batched_one() {
  auto k = p2p_batched_kernel<KT, DIM, FULL, KB>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)p2p_batched_smem<KB>());
}

template <int KT, int DIM>
cudaError_t configure_batched_kd() {
  cudaError_t e;
  if ((e = configure_batched_one<KT, DIM, true, 8>()) != cudaSuccess) return e;
  if ((e = configure_batched_one<KT, DIM, false, 8>()) != cudaSuccess) return e;
  if ((e = configure_batched_one<KT, DIM, true, 16>()) != cudaSuccess) return e;
  return configure_batched_one<KT, DIM, false, 16>();
}

template <int KT, int DIM>
cudaError_t launch_batched_kd(bool full, int kb, unsigned grid, cudaStream_t s,
                              const P2PTask* tasks, int n_tasks, const Term* terms,
                              const P2PChunk* chunks, const double4* recs, const double* blob,
                              double* arena, int64_t ps, const P2PKernel& kp, int* ctr) {
#define H2G_PB(F, KBv)                                                                      \
  p2p_batched_kernel<KT, DIM, F, KBv><<<grid, kPBThreads, p2p_batched_smem<KBv>(), s>>>(   \
      tasks, n_tasks, terms, chunks, recs, blob, arena, ps, kp, ctr)
  if (kb == 8) {
    if (full) H2G_PB(true, 8); else H2G_PB(false, 8);
  } else {
    if (full) H2G_PB(true, 16); else H2G_PB(false, 16);
  }
#undef H2G_PB
  return cudaGetLastError();
}

}  // namespace

cudaError_t p2p_batched_launch(int kt, int dim, bool full, int kb, int n_sm, cudaStream_t s,
                               const P2PTask* tasks, int n_tasks, const Term* terms,
                               const P2PChunk* chunks, const double4* recs, const double* blob,
                               double* arena, int64_t ps, const P2PKernel& kp, int* ctr) {
  const unsigned grid = (unsigned)std::max(1, std::min(n_tasks, n_sm * kPBCtasPerSm));
#define H2G_KD(KT, DIM)                                                                      \
  return launch_batched_kd<KT, DIM>(full, kb, grid, s, tasks, n_tasks, terms, chunks, recs, \
                                    blob, arena, ps, kp, ctr)
  const bool d3 = dim >= 3;
  if (kt == 0) {
    if (d3) H2G_KD(0, 3); else H2G_KD(0, 2);
  } else if (kt == 1) {
    if (d3) H2G_KD(1, 3); else H2G_KD(1, 2);
  } else {
    if (d3) H2G_KD(2, 3); else H2G_KD(2, 2);
  }
#undef H2G_KD
}

cudaError_t p2p_configure() {
  cudaError_t e;
  if ((e = configure_batched_kd<0, 2>()) != cudaSuccess) return e;
  if ((e = configure_batched_kd<0, 3>()) != cudaSuccess) return e;
  if ((e = configure_batched_kd<1, 2>()) != cudaSuccess) return e;
  if ((e = configure_batched_kd<1, 3>()) != cudaSuccess) return e;
  if ((e = configure_batched_kd<2, 2>()) != cudaSuccess) return e;
  if ((e = configure_batched_kd<2, 3>()) != cudaSuccess) return e;
  if ((e = configure_kd<0, 2>()) != cudaSuccess) return e;
  if ((e = configure_kd<0, 3>()) != cudaSuccess) return e;
  if ((e = configure_kd<1, 2>()) != cudaSuccess) return e;
  if ((e = configure_kd<1, 3>()) != cudaSuccess) return e;
  if ((e = configure_kd<2, 2>()) != cudaSuccess) return e;
  return configure_kd<2, 3>();
}

int p2p_ctas_per_sm(bool sw) { return sw ? kP2PCtasSW : kP2PCtasPerSm; }

cudaError_t p2p_launch(int kt, int dim, bool full, bool sw, bool pdl, unsigned grid,
                       cudaStream_t s, const P2PTask* tasks, int n_tasks, const Term* terms,
                       const P2PChunk* chunks, const P2PStage* stages, const double4* recs,
                       const double* blob, double* arena, const P2PKernel& kp, int* ctr) {
#define H2G_KD(KT, DIM)                                                                         \
  return launch_kd<KT, DIM>(full, sw, pdl, grid, s, tasks, n_tasks, terms, chunks, stages, recs, \
                            blob, arena, kp, ctr)
  const bool d3 = dim >= 3;
  if (kt == 0) {
    if (d3) H2G_KD(0, 3); else H2G_KD(0, 2);
  } else if (kt == 1) {
    if (d3) H2G_KD(1, 3); else H2G_KD(1, 2);
  } else {
    if (d3) H2G_KD(2, 3); else H2G_KD(2, 2);
  }
#undef H2G_KD
}

}  // namespace h2g
