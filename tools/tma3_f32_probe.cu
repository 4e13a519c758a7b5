// Probe (development aid): does a 3-D tensor TMA of a float box of BX x BY x 1
// work on this device?  usage: tma3_f32_probe BX BY esz promo
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

__global__ void k(const __grid_constant__ CUtensorMap tm, int bytes, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(sm)),
        "l"(&tm), "r"(-2), "r"(-1), "r"(1), "r"(b)
        : "memory");
  }
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(b) : "memory");
  out[threadIdx.x] = ((float*)sm)[threadIdx.x];
}

int main(int argc, char** argv) {
  int BX = atoi(argv[1]), BY = atoi(argv[2]), esz = atoi(argv[3]), promo = atoi(argv[4]);
  int nx = 8, ny = 8, nz = 8, pitch = 32;
  void* buf;
  cudaMalloc(&buf, (size_t)(nz + 2) * (ny + 2) * pitch * esz);
  cudaMemset(buf, 0, (size_t)(nz + 2) * (ny + 2) * pitch * esz);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)nx + 2, (cuuint64_t)ny + 2, (cuuint64_t)nz + 2};
  cuuint64_t str[2] = {(cuuint64_t)pitch * esz, (cuuint64_t)(ny + 2) * pitch * esz};
  cuuint32_t box[3] = {(cuuint32_t)BX, (cuuint32_t)BY, 1u}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, str,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  float* out;
  cudaMalloc(&out, 4096);
  int bytes = BX * BY * esz;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<<<1, 32, 65536>>>(tm, bytes, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("box %dx%d esz %d promo %d: encode %d, run %s\n", BX, BY, esz, promo, (int)r, cudaGetErrorString(e));
  return 0;
}
