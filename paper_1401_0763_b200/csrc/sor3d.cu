// sor3d.cu — NEXT-3: 3-D red-black SOR handle (the paper's future work,
// P:410) behind the sor3d_* entry points of include/sor.h.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "sor_internal.h"
#include "sor3d_tma.cuh"

using namespace sorh;

// NEXT-3: 3-D red-black SOR handle (single GPU, K1-form kernels; see
// k3d_half_sweep).  Loop control as the 2-D natural path: the stop test runs
// in the last CTA of the checking iteration's black launch, later launches
// exit early, the host polls one batch behind.
struct sor3d_grid {
  int64_t nz = 0, ny = 0, nx = 0;
  sor_dtype dt = SOR_F64;
  size_t esz = 8;
  int64_t pitch = 0;
  void* plane = nullptr;        // the current iterate
  void* plane2 = nullptr;       // FUSED kernel: the other plane of the ping-pong
  // default (sor3d_create): FUSED (k3d_tma, one HBM pass per iteration: 208
  // vs 161 GLUP/s in fp64 and 330 vs 225 in fp32 at 512^3)
  int kernel = SOR_KERNEL_NATURAL;
  CUtensorMap tm = {}, tm2 = {};  // 3-D tensor maps of plane / plane2 (k3d_tma source boxes)
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, poll_ev[2] = {nullptr, nullptr};
  DevState* dstate = nullptr;
  DevState* hstate = nullptr;
  double* scratch = nullptr;
  bool failed = false, have_elapsed = false;
  double elapsed_ms = 0.0;
  int device = 0;               // the device current at sor3d_create: every later call runs on it
};

namespace {

int set_error3(sor3d_grid* g, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  if (g && (code == SOR_E_CUDA)) g->failed = true;
  return code;
}

#define CU3(call)                                                                      \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return set_error3(g, SOR_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

void free3d(sor3d_grid* g) {
  if (!g) return;
  if (g->plane) cudaFree(g->plane);
  if (g->plane2) cudaFree(g->plane2);
  if (g->dstate) cudaFree(g->dstate);
  if (g->hstate) cudaFreeHost(g->hstate);
  if (g->scratch) cudaFree(g->scratch);
  if (g->ev0) cudaEventDestroy(g->ev0);
  if (g->ev1) cudaEventDestroy(g->ev1);
  for (int k = 0; k < 2; ++k)
    if (g->poll_ev[k]) cudaEventDestroy(g->poll_ev[k]);
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
}

// (z, y) rows of the full fp64 array <-> the padded device plane
int load3d(sor3d_grid* g, const double* init) {
  const int64_t w = g->nx + 2, nrow = (g->nz + 2) * (g->ny + 2);
  const size_t bytes = (size_t)nrow * g->pitch * g->esz;
  CU3(cudaMemsetAsync(g->plane, 0, bytes, g->stream));
  if (g->dt == SOR_F64) {
    CU3(cudaMemcpy2DAsync(g->plane, g->pitch * 8, init, w * 8, w * 8, nrow, cudaMemcpyDefault, g->stream));
  } else {
    CU3(cudaMemcpyAsync(g->scratch, init, (size_t)nrow * w * 8, cudaMemcpyDefault, g->stream));
    dim3 grid((unsigned)std::min<int64_t>((w + 255) / 256, 1024), (unsigned)std::min<int64_t>(nrow, 65535));
    narrow_rows<<<grid, 256, 0, g->stream>>>(g->scratch, w, (float*)g->plane, g->pitch, nrow, w);
    CU3(cudaGetLastError());
  }
  // both planes carry the shell (the fused kernel never writes planes 0, nz+1)
  CU3(cudaMemcpyAsync(g->plane2, g->plane, bytes, cudaMemcpyDeviceToDevice, g->stream));
  CU3(cudaStreamSynchronize(g->stream));
  return SOR_OK;
}

// 3-D tensor map of a plane for k3d_tma: (x, y, z) = (nx+2, ny+2, nz+2)
// elements, box = the kernel's window of one plane; out-of-range box parts
// read as zeros (never updated cells).
int make_tmap3(sor3d_grid* g, void* plane, CUtensorMap* m) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return set_error3(g, SOR_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[3] = {(cuuint64_t)(g->nx + 2), (cuuint64_t)(g->ny + 2), (cuuint64_t)(g->nz + 2)};
  const cuuint64_t strides[2] = {(cuuint64_t)(g->pitch * g->esz), (cuuint64_t)((g->ny + 2) * g->pitch * g->esz)};
  const cuuint32_t box[3] = {(cuuint32_t)(g->dt == SOR_F64 ? t3_wxb<double>() : t3_wxb<float>()), (cuuint32_t)kT3WY,
                             1u};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = encode(m, g->dt == SOR_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                      plane, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error3(g, SOR_E_CUDA, "cuTensorMapEncodeTiled (3-D) failed (%d)", (int)r);
  return SOR_OK;
}

// One fused iteration with k3d_tma (plane -> plane2, then swap).
template <typename R>
int k3d_tma_iteration(sor3d_grid* g, R w, const IterCtl& ctl) {
  constexpr int smem = t3_smem_bytes<R>();
  static int occ_dev[kMaxDev] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& occ = occ_dev[dev % kMaxDev];
  if (occ == 0) {
    CU3(cudaFuncSetAttribute(k3d_tma<R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CU3(cudaFuncSetAttribute(k3d_tma<R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k3d_tma<R, false>, kT3Threads, smem);
    if (occ <= 0) occ = 1;
  }
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const unsigned bx = (unsigned)((g->nx + kT3X - 1) / kT3X), by = (unsigned)((g->ny + kT3Y - 1) / kT3Y);
  // z chunks: minimise waves x planes per CTA (a chunk also reads ~5 planes
  // of warm-up), so the last wave is not a short tail of CTAs (e.g. 512^3
  // fp64: 666 tiles on 592 resident CTAs -> 8 chunks of 64 planes, 9 full
  // waves), chunks of at least 8 planes
  const int64_t tiles = (int64_t)bx * by, slots = (int64_t)occ * nsm;
  int64_t best_cost = -1, nch = 1;
  for (int64_t c = 1; c <= 64; ++c) {
    const int64_t zc_c = (g->nz + c - 1) / c;
    if (c > 1 && zc_c < 8) break;
    const int64_t waves = (tiles * ((g->nz + zc_c - 1) / zc_c) + slots - 1) / slots;
    const int64_t cost = waves * (zc_c + 5);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      nch = c;
    }
  }
  const int zc = (int)((g->nz + nch - 1) / nch);
  dim3 grid(bx, by, (unsigned)((g->nz + zc - 1) / zc));
  IterCtl c = ctl;
  c.finalize = ctl.ck ? 1 : 0;
  c.nparts = grid.x * grid.y * grid.z;
  if (ctl.ck)
    k3d_tma<R, true><<<grid, kT3Threads, smem, g->stream>>>(g->tm, (R*)g->plane2, g->pitch, (int)g->nz, (int)g->ny,
                                                             (int)g->nx, zc, w, c);
  else
    k3d_tma<R, false><<<grid, kT3Threads, smem, g->stream>>>(g->tm, (R*)g->plane2, g->pitch, (int)g->nz, (int)g->ny,
                                                              (int)g->nx, zc, w, c);
  CU3(cudaGetLastError());
  std::swap(g->plane, g->plane2);
  std::swap(g->tm, g->tm2);
  return SOR_OK;
}

template <typename R>
int k3d_iteration(sor3d_grid* g, R w, const IterCtl& ctl) {
  static int old_fused = -1;  // SOR_K3_OLD=1: the shared-plane z-wavefront of round 2 (A/B only)
  if (old_fused < 0) old_fused = getenv("SOR_K3_OLD") ? 1 : 0;
  if (g->kernel == SOR_KERNEL_FUSED && !old_fused) return k3d_tma_iteration<R>(g, w, ctl);
  if (g->kernel == SOR_KERNEL_FUSED) {
    using G = K3Geo<kX3, kY3>;
    const unsigned bx = (unsigned)((g->nx + 2 + kX3 - 1) / kX3), by = (unsigned)((g->ny + 2 + kY3 - 1) / kY3);
    // z chunks: about two waves of resident CTAs, at least 8 planes each
    static int occ_dev[kMaxDev] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int& occ = occ_dev[dev % kMaxDev];
    if (occ == 0) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k3d_fused<R, false, kX3, kY3>, G::NT, 0);
      if (occ <= 0) occ = 1;
    }
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = std::max<int64_t>(1, (2LL * occ * nsm + bx * by - 1) / ((int64_t)bx * by));
    const int zc = (int)std::max<int64_t>(8, (g->nz + want - 1) / want);
    dim3 grid(bx, by, (unsigned)((g->nz + zc - 1) / zc));
    IterCtl c = ctl;
    c.finalize = ctl.ck ? 1 : 0;
    c.nparts = grid.x * grid.y * grid.z;
    if (ctl.ck)
      k3d_fused<R, true, kX3, kY3><<<grid, G::NT, 0, g->stream>>>((const R*)g->plane, (R*)g->plane2, g->pitch,
                                                                  (int)g->nz, (int)g->ny, (int)g->nx, zc, w, c);
    else
      k3d_fused<R, false, kX3, kY3><<<grid, G::NT, 0, g->stream>>>((const R*)g->plane, (R*)g->plane2, g->pitch,
                                                                   (int)g->nz, (int)g->ny, (int)g->nx, zc, w, c);
    CU3(cudaGetLastError());
    std::swap(g->plane, g->plane2);
    std::swap(g->tm, g->tm2);
    return SOR_OK;
  }
  const int64_t half = (g->nx + 1) / 2;
  dim3 grid((unsigned)((half + 255) / 256), (unsigned)g->ny, (unsigned)g->nz);
  for (int color = 0; color < 2; ++color) {
    IterCtl c = ctl;
    c.finalize = (color == 1 && ctl.ck) ? 1 : 0;
    c.nparts = grid.x * grid.y * grid.z;
    if (ctl.ck && color == 1)
      k3d_half_sweep<R, true><<<grid, 256, 0, g->stream>>>((R*)g->plane, g->pitch, (int)g->nz, (int)g->ny,
                                                           (int)g->nx, color, w, c);
    else if (ctl.ck)
      k3d_half_sweep<R, true><<<grid, 256, 0, g->stream>>>((R*)g->plane, g->pitch, (int)g->nz, (int)g->ny,
                                                           (int)g->nx, color, w, c);
    else
      k3d_half_sweep<R, false><<<grid, 256, 0, g->stream>>>((R*)g->plane, g->pitch, (int)g->nz, (int)g->ny,
                                                            (int)g->nx, color, w, c);
    CU3(cudaGetLastError());
  }
  return SOR_OK;
}

template <typename R>
int run3d(sor3d_grid* g, double omega, int solve, int64_t n, double tol, int64_t K, bool want_last,
          int64_t* iters_out, double* max_out, bool* converged) {
  CU3(cudaMemsetAsync(g->dstate, 0, sizeof(DevState), g->stream));
  CU3(cudaEventRecord(g->ev0, g->stream));
  IterCtl base{};
  base.st = g->dstate;
  base.maxit = n;
  base.K = solve ? K : 1;
  base.tol = tol;
  base.solve = solve;
  base.T = 1;
  const R w = (R)omega;
  const int64_t blk = 64;
  int b = 0;
  int64_t enq = 0;  // iterations enqueued (launches after a stop exit early)
  for (int64_t k0 = 1; k0 <= n; k0 += blk) {
    const int64_t k1 = std::min(n, k0 + blk - 1);
    for (int64_t k = k0; k <= k1; ++k) {
      IterCtl c = base;
      c.k_last = k;
      c.ck = solve ? (k % K == 0) : (want_last && k == n);
      TRY(k3d_iteration<R>(g, w, c));
      ++enq;
    }
    if (solve) {
      CU3(cudaMemcpyAsync(&g->hstate[b & 1], g->dstate, sizeof(DevState), cudaMemcpyDeviceToHost, g->stream));
      CU3(cudaEventRecord(g->poll_ev[b & 1], g->stream));
      if (b >= 1) {
        CU3(cudaEventSynchronize(g->poll_ev[(b - 1) & 1]));
        if (g->hstate[(b - 1) & 1].stop) break;
      }
      ++b;
    }
  }
  CU3(cudaEventRecord(g->ev1, g->stream));
  CU3(cudaMemcpyAsync(&g->hstate[0], g->dstate, sizeof(DevState), cudaMemcpyDeviceToHost, g->stream));
  CU3(cudaStreamSynchronize(g->stream));
  float ms = 0.f;
  CU3(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
  g->elapsed_ms = ms;
  g->have_elapsed = true;
  const DevState& hs = g->hstate[0];
  *converged = hs.converged != 0;
  // the fused kernel swapped planes once per enqueued iteration, but those
  // after the converging one exited without writing
  if (g->kernel == SOR_KERNEL_FUSED && solve && hs.converged && ((enq - hs.conv_iter) & 1)) {
    std::swap(g->plane, g->plane2);
    std::swap(g->tm, g->tm2);
  }
  if (iters_out) *iters_out = solve ? (hs.converged ? hs.conv_iter : n) : n;
  if (max_out) *max_out = (solve || want_last) && n > 0 ? hs.max_change : 0.0;
  return SOR_OK;
}

int usable3(sor3d_grid* g) {
  if (!g) return set_error3(nullptr, SOR_E_INVAL, "handle is NULL");
  if (g->failed) return set_error3(nullptr, SOR_E_STATE, "handle failed earlier (CUDA error); destroy it");
  return SOR_OK;
}

}  // namespace

namespace {
// Every call on a handle runs on the handle's device and restores the
// caller's current device afterwards (as DevGuard in sor_api.cu).
struct DevGuard3 {
  int prev = -1;
  bool changed = false;
  explicit DevGuard3(const sor3d_grid* g) {
    if (g && cudaGetDevice(&prev) == cudaSuccess && prev != g->device)
      changed = cudaSetDevice(g->device) == cudaSuccess;
  }
  ~DevGuard3() {
    if (changed) cudaSetDevice(prev);
  }
};
}  // namespace

extern "C" {

int sor3d_create(sor3d_grid** out, int64_t nz, int64_t ny, int64_t nx, const double* init, sor_dtype dt) {
  if (!out) return set_error3(nullptr, SOR_E_INVAL, "out is NULL");
  *out = nullptr;
  if (!init) return set_error3(nullptr, SOR_E_INVAL, "init is NULL");
  if (dt != SOR_F64 && dt != SOR_F32) return set_error3(nullptr, SOR_E_INVAL, "bad dtype %d", (int)dt);
  if (nz < 1 || ny < 1 || nx < 1 || nz > 65535 || ny > 65535 || nx > (1 << 30))
    return set_error3(nullptr, SOR_E_INVAL, "need 1 <= nz, ny <= 65535 and 1 <= nx");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    return set_error3(nullptr, SOR_E_CUDA, "no CUDA device available; libsor has no CPU fallback");
  }
  int dev = 0;
  cudaDeviceProp prop{};
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess || prop.major != 10)
    return set_error3(nullptr, SOR_E_CUDA, "libsor.so is built for sm_100a (B200)");
  const int64_t n = (nz + 2) * (ny + 2) * (nx + 2);
  const bool on_dev = is_device_ptr(init);
  if (!on_dev && !host_all_finite(init, n))
    return set_error3(nullptr, SOR_E_INVAL, "init contains non-finite values");
  sor3d_grid* g = new sor3d_grid();
  g->device = dev;
  g->nz = nz;
  g->ny = ny;
  g->nx = nx;
  g->dt = dt;
  g->esz = dt == SOR_F64 ? 8 : 4;
  g->kernel = SOR_KERNEL_FUSED;
  g->pitch = round_up(nx + 2, 32);
  int rc = SOR_OK;
  do {
    if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&g->ev0) != cudaSuccess || cudaEventCreate(&g->ev1) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->poll_ev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->poll_ev[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaMalloc(&g->dstate, sizeof(DevState)) != cudaSuccess ||
        cudaMallocHost(&g->hstate, 2 * sizeof(DevState)) != cudaSuccess) {
      rc = set_error3(nullptr, SOR_E_CUDA, "3-D handle setup failed");
      break;
    }
    if (cudaMalloc(&g->plane, (size_t)(nz + 2) * (ny + 2) * g->pitch * g->esz) != cudaSuccess ||
        cudaMalloc(&g->plane2, (size_t)(nz + 2) * (ny + 2) * g->pitch * g->esz) != cudaSuccess ||
        (dt == SOR_F32 && cudaMalloc(&g->scratch, (size_t)n * 8) != cudaSuccess)) {
      cudaGetLastError();
      rc = set_error3(nullptr, SOR_E_NOMEM, "3-D grid allocation failed");
      break;
    }
    if (on_dev) {  // device-resident init: the same non-finite check on the GPU
      // order the reads after the caller's pending work on any stream
      if (cudaDeviceSynchronize() != cudaSuccess) {
        rc = set_error3(nullptr, SOR_E_CUDA, "device synchronize failed");
        break;
      }
      unsigned int* flag = nullptr;
      unsigned int bad = 0;
      if (cudaMalloc(&flag, sizeof(unsigned int)) != cudaSuccess) {
        rc = set_error3(nullptr, SOR_E_NOMEM, "flag allocation failed");
        break;
      }
      cudaMemsetAsync(flag, 0, sizeof(unsigned int), g->stream);
      count_nonfinite<<<4 * prop.multiProcessorCount, 256, 0, g->stream>>>(init, n, flag);
      cudaMemcpyAsync(&bad, flag, sizeof bad, cudaMemcpyDeviceToHost, g->stream);
      const cudaError_t e = cudaStreamSynchronize(g->stream);
      cudaFree(flag);
      if (e != cudaSuccess) {
        rc = set_error3(nullptr, SOR_E_CUDA, "non-finite check failed: %s", cudaGetErrorString(e));
        break;
      }
      if (bad) {
        rc = set_error3(nullptr, SOR_E_INVAL, "init contains non-finite values");
        break;
      }
    }
    rc = load3d(g, init);
    if (rc == SOR_OK) rc = make_tmap3(g, g->plane, &g->tm);
    if (rc == SOR_OK) rc = make_tmap3(g, g->plane2, &g->tm2);
  } while (0);
  if (rc < 0) {
    free3d(g);
    return rc;
  }
  *out = g;
  return SOR_OK;
}

int sor3d_iterate(sor3d_grid* g, double omega, int64_t iters, double* last_max_change) {
  if (int rc = usable3(g); rc < 0) return rc;
  DevGuard3 dg(g);
  if (!(omega > 0.0 && omega < 2.0)) return set_error3(nullptr, SOR_E_INVAL, "omega must satisfy 0 < omega < 2");
  if (iters < 0) return set_error3(nullptr, SOR_E_INVAL, "iters must be >= 0");
  bool conv = false;
  if (g->dt == SOR_F64)
    return run3d<double>(g, omega, 0, iters, 1.0, 1, last_max_change != nullptr, nullptr, last_max_change, &conv);
  return run3d<float>(g, omega, 0, iters, 1.0, 1, last_max_change != nullptr, nullptr, last_max_change, &conv);
}

int sor3d_solve(sor3d_grid* g, double omega, double tol, int64_t maxit, int64_t check_every, int64_t* iters_out,
                double* max_change_out) {
  if (int rc = usable3(g); rc < 0) return rc;
  DevGuard3 dg(g);
  if (!(omega > 0.0 && omega < 2.0)) return set_error3(nullptr, SOR_E_INVAL, "omega must satisfy 0 < omega < 2");
  if (!(tol > 0.0) || !std::isfinite(tol)) return set_error3(nullptr, SOR_E_INVAL, "tol must be finite and > 0");
  if (maxit < 1 || check_every < 1 || check_every > maxit)
    return set_error3(nullptr, SOR_E_INVAL, "need maxit >= 1 and 1 <= check_every <= maxit");
  bool conv = false;
  const int rc = g->dt == SOR_F64
                     ? run3d<double>(g, omega, 1, maxit, tol, check_every, false, iters_out, max_change_out, &conv)
                     : run3d<float>(g, omega, 1, maxit, tol, check_every, false, iters_out, max_change_out, &conv);
  if (rc < 0) return rc;
  return conv ? SOR_OK : SOR_NOT_CONVERGED;
}

int sor3d_download(sor3d_grid* g, double* out) {
  if (int rc = usable3(g); rc < 0) return rc;
  DevGuard3 dg(g);
  if (!out) return set_error3(nullptr, SOR_E_INVAL, "out is NULL");
  const int64_t w = g->nx + 2, nrow = (g->nz + 2) * (g->ny + 2);
  if (g->dt == SOR_F64) {
    CU3(cudaMemcpy2DAsync(out, w * 8, g->plane, g->pitch * 8, w * 8, nrow, cudaMemcpyDefault, g->stream));
  } else {
    dim3 grid((unsigned)std::min<int64_t>((w + 255) / 256, 1024), (unsigned)std::min<int64_t>(nrow, 65535));
    widen_rows<<<grid, 256, 0, g->stream>>>((const float*)g->plane, g->pitch, g->scratch, w, nrow, w);
    CU3(cudaGetLastError());
    CU3(cudaMemcpyAsync(out, g->scratch, (size_t)nrow * w * 8, cudaMemcpyDefault, g->stream));
  }
  CU3(cudaStreamSynchronize(g->stream));
  return SOR_OK;
}

int sor3d_set_kernel(sor3d_grid* g, int kernel) {
  if (int rc = usable3(g); rc < 0) return rc;
  if (kernel != SOR_KERNEL_NATURAL && kernel != SOR_KERNEL_FUSED)
    return set_error3(nullptr, SOR_E_INVAL, "3-D kernels: SOR_KERNEL_NATURAL or SOR_KERNEL_FUSED");
  g->kernel = kernel;
  return SOR_OK;
}

int sor3d_last_elapsed_ms(const sor3d_grid* g, double* ms) {
  if (!g || !ms) return set_error3(nullptr, SOR_E_INVAL, "NULL argument");
  if (!g->have_elapsed) return set_error3(nullptr, SOR_E_STATE, "no iterate/solve call timed yet");
  *ms = g->elapsed_ms;
  return SOR_OK;
}

void sor3d_destroy(sor3d_grid* g) {
  if (!g) return;
  DevGuard3 dg(g);
  if (g->stream) cudaStreamSynchronize(g->stream);
  free3d(g);
}

}  // extern "C"
