// h2g_eval.cuh — kernel-entry evaluation shared by the P2P engine
// (h2g_p2p.cuh) and the streaming engine's evaluated chunks (h2g_stream.cuh).
//
// Entry rule = Kernel.block (reference kernels.py:36-57): i == j ->
// (diag if set else zero_value) + shift; r == 0, i != j -> zero_value; else
// f(r) with f = log r (Log2D, kernels.py:70-71), 1/r (InverseR, 80-81) or
// the Gaussian of config 4, evaluated as a function of r^2.
#pragma once
#include <cstdint>

namespace h2g {

struct P2PKernel {
  double zero_value;  // r == 0, i != j
  double self_value;  // i == j
  double gauss_c;     // Gaussian: -1 / (2 sigma^2)
  int32_t check;      // 1: points may coincide (r == 0 test in every term)
  int32_t pad;
};

// Bulk prefetch of [p, p + bytes) into L2 (TMA engine, no registers / smem).
__device__ __forceinline__ void prefetch_l2(const void* p, uint64_t bytes) {
  const uint64_t a = reinterpret_cast<uint64_t>(p) & ~uint64_t(15);
  uint64_t n = (reinterpret_cast<uint64_t>(p) + bytes + 15 - a) & ~uint64_t(15);
  while (n > 0) {
    const uint32_t b = (uint32_t)(n < (1u << 20) ? n : (1u << 20));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a + (n - b)), "r"(b) : "memory");
    n -= b;
  }
}

__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// 1/sqrt(r2): MUFU.RSQ64H seed + one third-order Newton step
// (y += y e (1/2 + 3/8 e), e = 1 - r2 y^2): ~1 ulp.
__device__ __forceinline__ double rsqrt_nr(double r2) {
  double y = rsqrt_approx(r2);
  const double e = fma(-r2 * y, y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}

// f as a function of r^2 (kernels.py:70-71, 80-81; Gaussian of config 4)
template <int KT>
__device__ __forceinline__ double kfun(double r2, const P2PKernel& kp) {
  if constexpr (KT == 1) {
    return rsqrt_nr(r2);
  } else if constexpr (KT == 0) {
    return 0.5 * log(r2);
  } else {
    return exp(r2 * kp.gauss_c);
  }
}

template <int DIM>
__device__ __forceinline__ double dist2(double px, double py, double pz, const double4& s) {
  const double dx = px - s.x;
  double r2 = dx * dx;
  if constexpr (DIM >= 2) {
    const double dy = py - s.y;
    r2 = fma(dy, dy, r2);
  }
  if constexpr (DIM >= 3) {
    const double dz = pz - s.z;
    r2 = fma(dz, dz, r2);
  }
  return r2;
}

}  // namespace h2g
