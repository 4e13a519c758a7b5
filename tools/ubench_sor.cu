// Microbenchmark (development aid): throughput of the SOR cell update
// (7 dependent-ish FP64 ops, two register operands each) with K independent
// cells per thread, optionally with one 64-bit shuffle per 2 cells.
#include <cstdio>
#include <cuda_runtime.h>

template <int K, bool SH>
__global__ void upd(double* out, double w, int n) {
  double u[K], x[K], y[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    u[k] = threadIdx.x * 1e-3 + k;
    x[k] = k * 0.5;
    y[k] = k * 0.25 + 1.0;
  }
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double nb = y[k];
      if (SH && (k & 1) == 0) nb = __shfl_up_sync(0xffffffffu, y[k], 1);
      const double ns = __dadd_rn(x[k], u[(k + 1) % K]);
      const double we = __dadd_rn(nb, y[(k + 1) % K]);
      const double s = __dadd_rn(ns, we);
      const double a = __dmul_rn(0.25, s);
      const double r = __dsub_rn(a, u[k]);
      const double v = __dadd_rn(u[k], __dmul_rn(w, r));
      x[k] = y[k];
      y[k] = u[k];
      u[k] = v;
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += u[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int K, bool SH>
void run(int nsm, int clk, double* out, int warps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int n = 4000;
  upd<K, SH><<<nsm, 32 * warps>>>(out, 1.5, 10);
  cudaEventRecord(e0);
  upd<K, SH><<<nsm, 32 * warps>>>(out, 1.5, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dp = 7.0 * K * n * 32.0 * warps * nsm;
  printf("K=%d shfl=%d warps/SM=%2d: %.1f FP64 lanes/clk/SM (%.0f%% of 64)\n", K, (int)SH, warps,
         dp / (ms * 1e-3) / nsm / (clk * 1e3), 100 * dp / (ms * 1e-3) / nsm / (clk * 1e3) / 64);
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 24);
  int nsm, clk;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int w : {8, 12, 16, 24}) {
    run<2, false>(nsm, clk, out, w);
    run<4, false>(nsm, clk, out, w);
    run<8, false>(nsm, clk, out, w);
    run<2, true>(nsm, clk, out, w);
    run<4, true>(nsm, clk, out, w);
    run<8, true>(nsm, clk, out, w);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
