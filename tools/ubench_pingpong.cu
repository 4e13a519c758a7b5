// Ping-pong latency between two CTAs through L2 (development aid): one-way
// latency of a relaxed.gpu store seen by a relaxed.gpu polling load, for CTA
// pairs on SMs chosen by block index.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_rel(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

// blocks a and b ping-pong n times; others idle
__global__ void pingpong(unsigned long long* buf, int a, int b, int n, long long* out, unsigned* sm) {
  if (threadIdx.x != 0) return;
  unsigned long long* ping = buf;
  unsigned long long* pong = buf + 32;
  if ((int)blockIdx.x == a) {
    sm[0] = smid();
    long long t0 = clock64();
    unsigned long long g0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g0));
    for (int i = 1; i <= n; ++i) {
      st_rel(ping, i);
      while (ld_rel(pong) != (unsigned long long)i) {
      }
    }
    unsigned long long g1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g1));
    out[0] = clock64() - t0;
    out[1] = (long long)(g1 - g0);
  } else if ((int)blockIdx.x == b) {
    sm[1] = smid();
    for (int i = 1; i <= n; ++i) {
      while (ld_rel(ping) != (unsigned long long)i) {
      }
      st_rel(pong, i);
    }
  }
}

int main() {
  unsigned long long* buf;
  long long* out;
  unsigned* sm;
  cudaMalloc(&buf, 4096);
  cudaMalloc(&out, 64);
  cudaMalloc(&sm, 64);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int n = 20000;
  for (int b : {1, 2, 8, 37, 74, 100, 147}) {
    cudaMemset(buf, 0, 4096);
    pingpong<<<nsm, 32>>>(buf, 0, b, n, out, sm);
    long long h[2];
    unsigned s[2];
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(s, sm, 8, cudaMemcpyDeviceToHost);
    printf("block 0 (SM %3u) <-> block %3d (SM %3u): one-way %.0f cycles, %.0f ns\n", s[0], b, s[1],
           (double)h[0] / (2.0 * n), (double)h[1] / (2.0 * n));
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
