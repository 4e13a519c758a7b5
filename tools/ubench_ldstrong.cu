// Latency of 8 independent loads per thread from L2 (development aid):
// weak ld.global.cg vs ld.relaxed.gpu vs ld.volatile, one warp per SM and
// 16 warps per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__device__ __forceinline__ double ld(const double* p) {
  double v;
  if (MODE == 0) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if (MODE == 1) asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  if (MODE == 2) asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if (MODE == 3) v = *p;
  return v;
}

template <int MODE>
__global__ void k(const double* buf, int stride, int reps, double* out, long long* cyc) {
  const double* p = buf + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  double s = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = ld<MODE>(p + i * stride + (r & 7) * 64 * 1024);
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0) / reps;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* buf;
  double* out;
  long long* cyc;
  cudaMalloc(&buf, 256 << 20);
  cudaMemset(buf, 0, 256 << 20);
  cudaMalloc(&out, 64 << 20);
  cudaMalloc(&cyc, 64);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"ld.global.cg", "ld.relaxed.gpu", "ld.volatile", "plain"};
  for (int warps : {1, 16}) {
    for (int mode = 0; mode < 4; ++mode) {
      long long h;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<nsm, 32 * warps>>>(buf, 4096, 200, out, cyc);
        if (mode == 1) k<1><<<nsm, 32 * warps>>>(buf, 4096, 200, out, cyc);
        if (mode == 2) k<2><<<nsm, 32 * warps>>>(buf, 4096, 200, out, cyc);
        if (mode == 3) k<3><<<nsm, 32 * warps>>>(buf, 4096, 200, out, cyc);
      }
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%2d warps/SM, %-15s: %lld cycles per round of 8 independent loads\n", warps, names[mode], h);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
