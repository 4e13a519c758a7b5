// Microbenchmarks (development aid): FP64 add latency/throughput, shuffle
// latency on sm_100a.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dadd(double* out, long long* cyc, double a, int n) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = __dadd_rn(x, a);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_shfl(double* out, long long* cyc, int n) {
  int x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = __shfl_xor_sync(0xffffffffu, x, 1);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int CH>
__global__ void thr_dadd(double* out, double a, int n) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = a * (threadIdx.x + c);
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __dadd_rn(x[c], a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void thr_shfl(double* out, int n) {
  int x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = __shfl_xor_sync(0xffffffffu, x[c], 1) + 1;
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 26);
  cudaMalloc(&cyc, 64);
  long long h;
  int n = 1000;
  lat_dadd<<<1, 32>>>(out, cyc, 1e-3, n);
  lat_dadd<<<1, 32>>>(out, cyc, 1e-3, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", (double)h / (16.0 * n));
  lat_shfl<<<1, 32>>>(out, cyc, n);
  lat_shfl<<<1, 32>>>(out, cyc, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("SHFL dependent latency: %.2f cycles\n", (double)h / (16.0 * n));
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    int nn = 20000;
    thr_dadd<8><<<nsm, 32 * warps>>>(out, 1e-3, 10);
    cudaEventRecord(e0);
    thr_dadd<8><<<nsm, 32 * warps>>>(out, 1e-3, nn);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)nsm * 32 * warps * 8 * nn;
    printf("DADD throughput, %2d warps/SM x 8 chains: %.2f T/s = %.1f lanes/clk/SM at %d MHz\n", warps,
           ops / ms / 1e9, ops / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1000);
  }
  for (int warps : {4, 8, 16, 32}) {
    int nn = 20000;
    thr_shfl<<<nsm, 32 * warps>>>(out, 10);
    cudaEventRecord(e0);
    thr_shfl<<<nsm, 32 * warps>>>(out, nn);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)nsm * warps * 8 * nn;  // warp-level shuffles
    printf("SHFL throughput, %2d warps/SM: %.3f warp-shfl/clk/SM\n", warps, ops / (ms * 1e-3) / nsm / (clk * 1e3));
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
