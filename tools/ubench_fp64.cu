// Microbenchmark: fp64 pipe and the pair-kernel evaluation rate on one B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_fp64 tools/ubench_fp64.cu
// Prints DFMA/s, rsqrt.approx.f64 /s and evaluated 1/r pair entries /s
// (the recompute path's inner loop) for the DESIGN.md recompute decision.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c0 = 0.5, c1 = 0.25, c2 = 0.125, c3 = 0.0625;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      c0 = fma(c0, b, a);
      c1 = fma(c1, b, a);
      c2 = fma(c2, b, a);
      c3 = fma(c3, b, a);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + c2 + c3;
}

__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

__global__ void mufu_loop(double* out, int iters) {
  double s0 = 1.0 + threadIdx.x, s1 = 2.0, s2 = 3.0, s3 = 4.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      s0 = rsqrt_approx(s0) + 1.0;
      s1 = rsqrt_approx(s1) + 1.0;
      s2 = rsqrt_approx(s2) + 1.0;
      s3 = rsqrt_approx(s3) + 1.0;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}

// pair loop: rows in registers (J per lane), columns broadcast from smem
template <int J>
__global__ void pair_loop(double* out, int ncol, int reps) {
  __shared__ double4 src[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    src[i] = make_double4(0.001 * i, 0.002 * i, -0.003 * i, 1.0 / (i + 1));
  __syncthreads();
  double px[J], py[J], pz[J], acc[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    px[j] = 0.5 + 0.01 * (threadIdx.x + 32 * j);
    py[j] = -0.3 + 0.001 * j;
    pz[j] = 0.7;
    acc[j] = 0.0;
  }
  for (int r = 0; r < reps; ++r)
    for (int c = 0; c < ncol; ++c) {
      const double4 s = src[c];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const double dx = px[j] - s.x, dy = py[j] - s.y, dz = pz[j] - s.z;
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        double y = rsqrt_approx(r2);
        const double e = fma(-r2 * y, y, 1.0);
        y = fma(y * e, fma(0.375, e, 0.5), y);
        y = r2 == 0.0 ? 0.0 : y;
        acc[j] = fma(y, s.w, acc[j]);
      }
    }
  double t = 0;
#pragma unroll
  for (int j = 0; j < J; ++j) t += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int blocks = nsm * 8, threads = 256, iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  double n = (double)blocks * threads * iters * 64;
  printf("DFMA: %.2f T/s (%.1f TFLOP/s), %.1f per clk per SM at 1.965 GHz\n", n / ms / 1e9,
         2 * n / ms / 1e9, n / (ms * 1e-3) / nsm / 1.965e9);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    mufu_loop<<<blocks, threads>>>(out, iters / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  n = (double)blocks * threads * (iters / 4) * 64;
  printf("rsqrt.approx.f64 (+DADD): %.2f T/s, %.1f per clk per SM\n", n / ms / 1e9,
         n / (ms * 1e-3) / nsm / 1.965e9);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    pair_loop<4><<<blocks, threads>>>(out, 64, 64);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  n = (double)blocks * threads * 4 * 64 * 64;
  printf("1/r pair entries (J=4): %.2f G/s, %.3f per clk per SM, equiv stream %.2f TB/s\n",
         n / ms / 1e6, n / (ms * 1e-3) / nsm / 1.965e9, 8 * n / ms / 1e9);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    pair_loop<2><<<blocks, threads>>>(out, 64, 64);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  n = (double)blocks * threads * 2 * 64 * 64;
  printf("1/r pair entries (J=2): %.2f G/s, %.3f per clk per SM, equiv stream %.2f TB/s\n",
         n / ms / 1e6, n / (ms * 1e-3) / nsm / 1.965e9, 8 * n / ms / 1e9);
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
