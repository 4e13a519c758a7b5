// Cost of 8 independent stores per thread + fence (development aid): weak
// st.global vs st.relaxed.gpu vs st.volatile.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__device__ __forceinline__ void st(unsigned long long* p, unsigned long long v) {
  if (MODE == 0) asm volatile("st.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  if (MODE == 1) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  if (MODE == 2) asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  if (MODE == 3) asm volatile("st.global.cg.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int MODE, bool FENCE>
__global__ void k(unsigned long long* buf, int reps, long long* cyc) {
  unsigned long long* p = buf + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
  const size_t stride = (size_t)gridDim.x * blockDim.x * 2;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 8; ++i) st<MODE>(p + i * stride, r);
    if (FENCE) __threadfence();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}

int main() {
  unsigned long long* buf;
  long long* cyc;
  cudaMalloc(&buf, 256 << 20);
  cudaMalloc(&cyc, 64);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"st.global", "st.relaxed.gpu", "st.volatile", "st.global.cg"};
  for (int warps : {1, 16}) {
    for (int mode = 0; mode < 4; ++mode) {
      for (int f = 0; f < 2; ++f) {
        long long h;
        for (int rep = 0; rep < 2; ++rep) {
          if (mode == 0) f ? k<0, true><<<nsm, 32 * warps>>>(buf, 200, cyc) : k<0, false><<<nsm, 32 * warps>>>(buf, 200, cyc);
          if (mode == 1) f ? k<1, true><<<nsm, 32 * warps>>>(buf, 200, cyc) : k<1, false><<<nsm, 32 * warps>>>(buf, 200, cyc);
          if (mode == 2) f ? k<2, true><<<nsm, 32 * warps>>>(buf, 200, cyc) : k<2, false><<<nsm, 32 * warps>>>(buf, 200, cyc);
          if (mode == 3) f ? k<3, true><<<nsm, 32 * warps>>>(buf, 200, cyc) : k<3, false><<<nsm, 32 * warps>>>(buf, 200, cyc);
        }
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%2d warps/SM, %-15s %s: %lld cycles per round of 8 stores\n", warps, names[mode],
               f ? "+fence" : "      ", h);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
