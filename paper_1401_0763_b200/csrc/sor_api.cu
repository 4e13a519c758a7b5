// sor_api.cu — C ABI (include/sor.h) and host-side driver of the B200 red-black
// SOR hot path.  Algorithm 1 of arXiv 1401.0763 [P:283-337] re-designed for
// sm_100a: the iteration loop is enqueued on one CUDA stream, the stop test
// runs on the device (fused into the last part of the checking launch), and
// the host polls a pinned copy of the device state once per batch, one batch
// behind, so the GPU never idles on a host round trip.
//
// Multi-GPU (§8(e)): the grid is split into row slabs [S:232-240]; after each
// HBM pass every slab sends its first/last h rows to its neighbours (h = 1
// per half-sweep for K1, h = 2T per T-iteration pass for K3/K4) and, on
// checked iterations, the per-slab max is joined by an allreduce-max.  The
// transport is NCCL over NVLink (dist mode) or device copies (virtual mode).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <map>
#include <tuple>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "sor.h"
#include "sor_kernels.cuh"

using namespace sorb;

namespace {

thread_local std::string g_last_error;

struct Slab {
  int64_t g_lo = 0, g_hi = 0;  // owned global interior rows [g_lo, g_hi)
  int64_t g0 = 0;              // global row of storage row 0 (= g_lo - kRowPad)
  int64_t nstore = 0;          // storage rows
  // planes 0, 1: ping-pong; plane 2 (allocated on the first deferred solve):
  // the speculative pass of the deferred stop test writes the third plane
  void* plane[3] = {nullptr, nullptr, nullptr};
  WaveMaps tmap[3];  // per plane: tensor maps of the wave kernel's source-row boxes
};

enum class Mode { Single, Virtual, Dist };

struct KernelCache {
  int occ_blocks = 0;  // resident CTAs per SM for the wave kernel instance
};

}  // namespace

struct sor_grid {
  int64_t rows = 0, cols = 0;
  sor_dtype dt = SOR_F64;
  size_t esz = 8;
  int64_t pitch = 0;  // elements
  Mode mode = Mode::Single;
  std::vector<Slab> slabs;
  int cur = 0;  // plane holding the current iterate (same for all slabs)
  int kernel = SOR_KERNEL_FUSED;
  int tdepth = 1;
  int device = 0;
  int nsm = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t poll_ev[2] = {nullptr, nullptr};
  DevState* dstate = nullptr;
  DevState* hstate = nullptr;  // pinned, 2 slots for one-batch-behind polling
  double* scratch = nullptr;   // f64 staging for f32 pack/unpack and dist gather
  size_t scratch_bytes = 0;
  unsigned int* dflag = nullptr;
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  int halo_valid = kRowPad;  // rows of the current plane's halos known up to date
  struct PassRec {
    int64_t k_last;
    int src, dst, T;
  };
  std::vector<PassRec> pass_ends;  // wave passes of the current solve segment
  int nplanes = 2;                 // planes in rotation (3 once the deferred solve allocated plane 2)
  int nxt(int p) const { return (p + 1) % nplanes; }
  // deferred stop test: the last checked pass not yet decided, and the slot set
  // the next checked pass contributes to
  bool prev_valid = false;
  int prev_T = 0, prev_ck = 0, prev_set = 0, next_set = 0;
  int64_t prev_k_last = 0;
  // wave-kernel tile tables per (slab, T, occupancy): device int4 array + count
  std::map<std::tuple<int, int, int>, std::pair<int4*, int>> tiles;  // (last iteration, (cur after, T))
  int64_t exact_reruns = 0;  // solve passes re-run with exact maxima (diagnostic)
  int every_ck = 4;          // max-change mode of T-deep solve passes with check_every == 1
  int method = 0;            // 0: red-black SOR; 1: Jacobi (sor_jacobi_*; NEXT-2)
  bool failed = false;
  bool have_elapsed = false;
  double elapsed_ms = 0.0;
  sor_stats st{};
};

namespace {

int set_error(sor_grid* g, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  if (g && (code == SOR_E_CUDA || code == SOR_E_NCCL)) g->failed = true;
  return code;
}

#define CU(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return set_error(g, SOR_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define NC(call)                                                                      \
  do {                                                                                \
    ncclResult_t r_ = (call);                                                         \
    if (r_ != ncclSuccess)                                                            \
      return set_error(g, SOR_E_NCCL, "%s failed: %s", #call, ncclGetErrorString(r_)); \
  } while (0)

#define TRY(expr)             \
  do {                        \
    int rc_ = (expr);         \
    if (rc_ < 0) return rc_;  \
  } while (0)

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int partition(int64_t rows, int P, int p, int64_t* lo, int64_t* hi) {
  if (P < 1 || p < 0 || p >= P || rows < P) return SOR_E_INVAL;
  const int64_t base = rows / P, rem = rows % P;
  const int64_t start = 1 + p * base + std::min<int64_t>(p, rem);
  *lo = start;
  *hi = start + base + (p < rem ? 1 : 0);
  return SOR_OK;
}

template <typename R>
R* col0(void* plane) {
  return reinterpret_cast<R*>(plane) + kColPad;
}

cudaMemcpyKind kDefault = cudaMemcpyDefault;

// ------------------------------------------------------------------ layout
// Copy global rows [ga, gb) of a full (rows+2)x(cols+2) fp64 array into plane p
// of slab s (rounding to fp32 if needed).
// Tensor maps of one storage plane for the wave kernel's TMA row loads: the
// whole (nstore x pitch) plane, boxes of 6 rows (steady state) and 2 rows
// (prologue) x one warp strip (32 * kWaveNC columns).
int make_tmaps(sor_grid* g, Slab& s, int p) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return set_error(g, SOR_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)g->pitch, (cuuint64_t)s.nstore};
  const cuuint64_t strides[1] = {(cuuint64_t)(g->pitch * g->esz)};
  const cuuint32_t estr[2] = {1u, 1u};
  for (int b = 0; b < 2; ++b) {
    const cuuint32_t box[2] = {(cuuint32_t)wave_cols<kWaveNC>(), b == 0 ? 6u : 2u};
    CUresult r = encode(&s.tmap[p].m[b], g->dt == SOR_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        2, s.plane[p], dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(g, SOR_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  }
  return SOR_OK;
}

int load_rows(sor_grid* g, const Slab& s, int p, const double* init, int64_t ga, int64_t gb) {
  if (gb <= ga) return SOR_OK;
  const int64_t w = g->cols + 2;
  if (g->dt == SOR_F64) {
    CU(cudaMemcpy2DAsync(col0<double>(s.plane[p]) + (ga - s.g0) * g->pitch, g->pitch * 8,
                         init + ga * w, w * 8, w * 8, gb - ga, kDefault, g->stream));
    return SOR_OK;
  }
  const int64_t chunk = std::max<int64_t>(1, (int64_t)(g->scratch_bytes / (w * 8)));
  for (int64_t r = ga; r < gb; r += chunk) {
    const int64_t n = std::min(chunk, gb - r);
    CU(cudaMemcpyAsync(g->scratch, init + r * w, n * w * 8, kDefault, g->stream));
    dim3 grid((unsigned)std::min<int64_t>((w + 255) / 256, 1024), (unsigned)std::min<int64_t>(n, 65535));
    narrow_rows<<<grid, 256, 0, g->stream>>>(g->scratch, w, col0<float>(s.plane[p]) + (r - s.g0) * g->pitch,
                                             g->pitch, n, w);
    CU(cudaGetLastError());
  }
  return SOR_OK;
}

// Copy global rows [ga, gb) of plane p of slab s into a full fp64 array.
int store_rows(sor_grid* g, const Slab& s, int p, double* out, int64_t ga, int64_t gb) {
  if (gb <= ga) return SOR_OK;
  const int64_t w = g->cols + 2;
  if (g->dt == SOR_F64) {
    CU(cudaMemcpy2DAsync(out + ga * w, w * 8, col0<double>(s.plane[p]) + (ga - s.g0) * g->pitch,
                         g->pitch * 8, w * 8, gb - ga, kDefault, g->stream));
    return SOR_OK;
  }
  const int64_t chunk = std::max<int64_t>(1, (int64_t)(g->scratch_bytes / (w * 8)));
  for (int64_t r = ga; r < gb; r += chunk) {
    const int64_t n = std::min(chunk, gb - r);
    dim3 grid((unsigned)std::min<int64_t>((w + 255) / 256, 1024), (unsigned)std::min<int64_t>(n, 65535));
    widen_rows<<<grid, 256, 0, g->stream>>>(col0<float>(s.plane[p]) + (r - s.g0) * g->pitch, g->pitch,
                                            g->scratch, w, n, w);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out + r * w, g->scratch, n * w * 8, kDefault, g->stream));
    CU(cudaStreamSynchronize(g->stream));  // scratch is reused by the next chunk
  }
  return SOR_OK;
}

// Host arrays: a branch-free exponent test over the raw bits (vectorisable),
// split across host threads for large grids (the e2e path validates every
// reset; a serial isfinite loop cost ~17 ms per C3 grid).
bool host_all_finite(const double* p, int64_t n) {
  auto scan = [](const double* a, int64_t m) {
    const uint64_t* b = reinterpret_cast<const uint64_t*>(a);
    uint64_t bad = 0;
    for (int64_t i = 0; i < m; ++i) bad |= (uint64_t)(((b[i] >> 52) & 0x7ffu) == 0x7ffu);
    return bad == 0;
  };
  const int64_t kChunk = 1 << 20;
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (n < 4 * kChunk || hw == 1) return scan(p, n);
  std::vector<std::thread> th;
  std::vector<char> ok(hw, 1);
  const int64_t per = (n + hw - 1) / hw;
  for (unsigned t = 0; t < hw; ++t) {
    const int64_t a = (int64_t)t * per, m = std::max<int64_t>(0, std::min(n, a + per) - a);
    th.emplace_back([&, t, a, m] { ok[t] = scan(p + a, m) ? 1 : 0; });
  }
  for (auto& x : th) x.join();
  for (char c : ok)
    if (!c) return false;
  return true;
}

int check_finite(sor_grid* g, const double* init, int64_t n, bool on_device) {
  if (!on_device) {
    if (!host_all_finite(init, n)) {
      for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(init[i])) return set_error(nullptr, SOR_E_INVAL, "init[%lld] is not finite", (long long)i);
    }
    return SOR_OK;
  }
  CU(cudaMemsetAsync(g->dflag, 0, sizeof(unsigned int), g->stream));
  count_nonfinite<<<4 * g->nsm, 256, 0, g->stream>>>(init, n, g->dflag);
  CU(cudaGetLastError());
  unsigned int bad = 0;
  CU(cudaMemcpyAsync(&bad, g->dflag, sizeof bad, cudaMemcpyDeviceToHost, g->stream));
  CU(cudaStreamSynchronize(g->stream));
  if (bad) return set_error(nullptr, SOR_E_INVAL, "init contains non-finite values");
  return SOR_OK;
}

// Fill both planes of every slab from init: global rows within the slab's
// storage window that exist in [0, rows+1] (own rows, ring, initial halos).
int load_all(sor_grid* g, const double* init) {
  for (auto& s : g->slabs) {
    const size_t bytes = (size_t)s.nstore * g->pitch * g->esz;
    CU(cudaMemsetAsync(s.plane[0], 0, bytes, g->stream));
    const int64_t ga = std::max<int64_t>(0, s.g0);
    const int64_t gb = std::min<int64_t>(g->rows + 2, s.g0 + s.nstore);
    TRY(load_rows(g, s, 0, init, ga, gb));
    for (int p = 1; p < 3; ++p)
      if (s.plane[p]) CU(cudaMemcpyAsync(s.plane[p], s.plane[0], bytes, cudaMemcpyDeviceToDevice, g->stream));
  }
  g->cur = 0;
  g->halo_valid = kRowPad;
  CU(cudaStreamSynchronize(g->stream));
  return SOR_OK;
}

int validate_dims(int64_t rows, int64_t cols) {
  if (rows < 1 || cols < 1)
    return set_error(nullptr, SOR_E_INVAL, "rows and cols must be >= 1 (got %lld x %lld)",
                     (long long)rows, (long long)cols);
  if (cols > (int64_t)1 << 30 || rows > (int64_t)1 << 34)
    return set_error(nullptr, SOR_E_INVAL, "grid too large");
  return SOR_OK;
}

void free_grid(sor_grid* g) {
  if (!g) return;
  for (auto& s : g->slabs)
    for (int p = 0; p < 3; ++p)
      if (s.plane[p]) cudaFree(s.plane[p]);
  if (g->dstate) cudaFree(g->dstate);
  if (g->hstate) cudaFreeHost(g->hstate);
  if (g->scratch) cudaFree(g->scratch);
  if (g->dflag) cudaFree(g->dflag);
  if (g->ev0) cudaEventDestroy(g->ev0);
  if (g->ev1) cudaEventDestroy(g->ev1);
  for (int k = 0; k < 2; ++k)
    if (g->poll_ev[k]) cudaEventDestroy(g->poll_ev[k]);
  if (g->own_stream) cudaStreamDestroy(g->own_stream);
  if (g->comm) ncclCommDestroy(g->comm);
  for (auto& kv : g->tiles) cudaFree(kv.second.first);
  delete g;
}

// Common construction.  slabs_lo_hi: owned row ranges of the slabs this
// handle holds.
int build(sor_grid* g, const double* init, const std::vector<std::pair<int64_t, int64_t>>& spans) {
  int dev = 0;
  CU(cudaGetDevice(&dev));
  g->device = dev;
  cudaDeviceProp prop{};
  CU(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10)
    return set_error(g, SOR_E_CUDA, "libsor.so is built for sm_100a (B200); device %d is sm_%d%d",
                     dev, prop.major, prop.minor);
  g->nsm = prop.multiProcessorCount;
  g->esz = g->dt == SOR_F64 ? 8 : 4;
  // row: [kColPad][cols+2][>= one strip of read-ahead], multiple of 32 elements
  g->pitch = round_up(kColPad + g->cols + 2 + wave_cols<kWaveNC>() + 16, 32);
  CU(cudaStreamCreateWithFlags(&g->own_stream, cudaStreamNonBlocking));
  g->stream = g->own_stream;
  CU(cudaEventCreate(&g->ev0));
  CU(cudaEventCreate(&g->ev1));
  for (int k = 0; k < 2; ++k) CU(cudaEventCreateWithFlags(&g->poll_ev[k], cudaEventDisableTiming));
  CU(cudaMalloc(&g->dstate, sizeof(DevState)));
  CU(cudaMemsetAsync(g->dstate, 0, sizeof(DevState), g->stream));
  CU(cudaMallocHost(&g->hstate, 2 * sizeof(DevState)));
  memset(g->hstate, 0, 2 * sizeof(DevState));
  CU(cudaMalloc(&g->dflag, sizeof(unsigned int)));
  g->scratch_bytes = (size_t)std::max<int64_t>(64 << 20, (g->cols + 2) * 8 * 4);
  if (g->dt == SOR_F32 || g->mode == Mode::Dist) {
    cudaError_t e = cudaMalloc(&g->scratch, g->scratch_bytes);
    if (e != cudaSuccess) return set_error(g, SOR_E_NOMEM, "scratch: %s", cudaGetErrorString(e));
  }
  for (auto& sp : spans) {
    Slab s;
    s.g_lo = sp.first;
    s.g_hi = sp.second;
    s.g0 = s.g_lo - kRowPad;
    s.nstore = (s.g_hi - s.g_lo) + 2 * kRowPad;
    for (int p = 0; p < 2; ++p) {
      cudaError_t e = cudaMalloc(&s.plane[p], (size_t)s.nstore * g->pitch * g->esz);
      if (e != cudaSuccess) {
        cudaGetLastError();
        g->slabs.push_back(s);
        return set_error(nullptr, SOR_E_NOMEM, "cudaMalloc of %.3f GB plane failed: %s",
                         (double)s.nstore * g->pitch * g->esz / 1e9, cudaGetErrorString(e));
      }
    }
    g->slabs.push_back(s);
    for (int p = 0; p < 2; ++p) TRY(make_tmaps(g, g->slabs.back(), p));
  }
  const bool on_dev = is_device_ptr(init);
  TRY(check_finite(g, init, (g->rows + 2) * (g->cols + 2), on_dev));
  TRY(load_all(g, init));
  g->st.nslabs = (int32_t)g->slabs.size();
  g->st.rank = g->rank;
  g->st.nranks = g->nranks;
  g->st.row_lo = g->slabs[0].g_lo;
  g->st.row_hi = g->slabs[0].g_hi;
  g->st.pitch_elems = g->pitch;
  g->st.kernel = g->kernel;
  g->st.temporal_depth = g->tdepth;
  return SOR_OK;
}

int create_common(sor_grid** out, int64_t rows, int64_t cols, const double* init, sor_dtype dt,
                  Mode mode, int nslabs, int rank, int nranks, int device, const void* nccl_id) {
  if (!out) return set_error(nullptr, SOR_E_INVAL, "out is NULL");
  *out = nullptr;
  if (!init) return set_error(nullptr, SOR_E_INVAL, "init is NULL");
  if (dt != SOR_F64 && dt != SOR_F32) return set_error(nullptr, SOR_E_INVAL, "bad dtype %d", (int)dt);
  TRY(validate_dims(rows, cols));
  std::vector<std::pair<int64_t, int64_t>> spans;
  if (mode == Mode::Single) {
    spans.push_back({1, rows + 1});
  } else if (mode == Mode::Virtual) {
    if (nslabs < 1 || rows < 8LL * nslabs)
      return set_error(nullptr, SOR_E_INVAL, "virtual: need 1 <= nslabs and rows >= 8*nslabs");
    for (int p = 0; p < nslabs; ++p) {
      int64_t lo, hi;
      partition(rows, nslabs, p, &lo, &hi);
      spans.push_back({lo, hi});
    }
  } else {
    if (nranks < 1 || rank < 0 || rank >= nranks || rows < 8LL * nranks)
      return set_error(nullptr, SOR_E_INVAL, "dist: need 0 <= rank < nranks and rows >= 8*nranks");
    if (!nccl_id) return set_error(nullptr, SOR_E_INVAL, "dist: nccl_id is NULL");
    int64_t lo, hi;
    partition(rows, nranks, rank, &lo, &hi);
    spans.push_back({lo, hi});
  }
  if (mode == Mode::Dist) {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return set_error(nullptr, SOR_E_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    return set_error(nullptr, SOR_E_CUDA, "no CUDA device available (%s); libsor has no CPU fallback",
                     cudaGetErrorString(e));
  }
  sor_grid* g = new sor_grid();
  g->rows = rows;
  g->cols = cols;
  g->dt = dt;
  g->mode = mode;
  g->rank = mode == Mode::Dist ? rank : 0;
  g->nranks = mode == Mode::Dist ? nranks : 1;
  if (mode == Mode::Dist) {
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof id);
    ncclResult_t r = ncclCommInitRank(&g->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      set_error(nullptr, SOR_E_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
      free_grid(g);
      return SOR_E_NCCL;
    }
  }
  int rc = build(g, init, spans);
  if (rc < 0) {
    free_grid(g);
    return rc;
  }
  *out = g;
  return SOR_OK;
}

int usable(sor_grid* g) {
  if (!g) return set_error(nullptr, SOR_E_INVAL, "handle is NULL");
  if (g->failed) return set_error(nullptr, SOR_E_STATE, "handle failed earlier (CUDA/NCCL error); destroy it");
  return SOR_OK;
}

// ------------------------------------------------------------------ halos
// After a pass wrote plane p: each slab sends its first/last h owned rows to
// the neighbouring slabs' halo rows of the same plane.
int exchange(sor_grid* g, int p, int h) {
  const size_t row_bytes = (size_t)g->pitch * g->esz;
  if (g->mode == Mode::Virtual) {
    const int n = (int)g->slabs.size();
    for (int k = 0; k + 1 < n; ++k) {
      Slab& a = g->slabs[k];
      Slab& b = g->slabs[k + 1];
      char* ap = (char*)a.plane[p];
      char* bp = (char*)b.plane[p];
      // a's last h rows -> b's top halo; b's first h rows -> a's bottom halo
      CU(cudaMemcpyAsync(bp + (a.g_hi - h - b.g0) * row_bytes, ap + (a.g_hi - h - a.g0) * row_bytes,
                         h * row_bytes, cudaMemcpyDeviceToDevice, g->stream));
      CU(cudaMemcpyAsync(ap + (b.g_lo - a.g0) * row_bytes, bp + (b.g_lo - b.g0) * row_bytes,
                         h * row_bytes, cudaMemcpyDeviceToDevice, g->stream));
    }
    g->st.halo_exchanges += 1;
    return SOR_OK;
  }
  if (g->mode != Mode::Dist || g->nranks == 1) return SOR_OK;
  Slab& s = g->slabs[0];
  char* pl = (char*)s.plane[p];
  const ncclDataType_t ty = ncclUint8;
  const size_t n = h * row_bytes;
  NC(ncclGroupStart());
  if (g->rank > 0) {
    NC(ncclSend(pl + (s.g_lo - s.g0) * row_bytes, n, ty, g->rank - 1, g->comm, g->stream));
    NC(ncclRecv(pl + (s.g_lo - h - s.g0) * row_bytes, n, ty, g->rank - 1, g->comm, g->stream));
  }
  if (g->rank + 1 < g->nranks) {
    NC(ncclSend(pl + (s.g_hi - h - s.g0) * row_bytes, n, ty, g->rank + 1, g->comm, g->stream));
    NC(ncclRecv(pl + (s.g_hi - s.g0) * row_bytes, n, ty, g->rank + 1, g->comm, g->stream));
  }
  NC(ncclGroupEnd());
  g->st.halo_exchanges += 1;
  return SOR_OK;
}

// Join the per-slab maxima and run the stop test (multi-slab modes).
int join_and_finalize(sor_grid* g, const IterCtl& ctl) {
  if (g->mode == Mode::Dist && g->nranks > 1)
    NC(ncclAllReduce(&g->dstate->maxbits[0][0], &g->dstate->maxbits[0][0], kMaxT * 16, ncclUint64, ncclMax,
                     g->comm, g->stream));
  finalize_kernel<<<1, 32, 0, g->stream>>>(ctl);
  CU(cudaGetLastError());
  g->st.kernel_launches += 1;
  return SOR_OK;
}

bool single_part(const sor_grid* g) { return g->slabs.size() == 1 && g->nranks == 1; }

// ------------------------------------------------------------------ K1
template <typename R>
int k1_iteration(sor_grid* g, R w, IterCtl ctl) {
  const int64_t half = (g->cols + 1) / 2;
  const bool fused_fin = single_part(g) && ctl.ck != 0;
  for (int color = 0; color < 2; ++color) {
    for (auto& s : g->slabs) {
      R* base = col0<R>(s.plane[g->cur]);
      const int64_t nr = s.g_hi - s.g_lo;
      dim3 grid((unsigned)((half + 255) / 256), (unsigned)std::min<int64_t>(nr, 65535));
      IterCtl c = ctl;
      c.finalize = (color == 1 && fused_fin) ? 1 : 0;
      c.nparts = grid.x * grid.y;
      if (ctl.ck)
        k1_half_sweep<R, true><<<grid, 256, 0, g->stream>>>(base, g->pitch, s.g0, g->rows, g->cols,
                                                            s.g_lo, s.g_hi, color, w, c);
      else
        k1_half_sweep<R, false><<<grid, 256, 0, g->stream>>>(base, g->pitch, s.g0, g->rows,
                                                             g->cols, s.g_lo, s.g_hi, color, w, c);
      CU(cudaGetLastError());
      g->st.kernel_launches += 1;
    }
    g->st.half_sweeps += 1;
    TRY(exchange(g, g->cur, 1));
  }
  g->halo_valid = 1;
  g->st.hbm_passes += 2;
  if (ctl.ck && !fused_fin) TRY(join_and_finalize(g, ctl));
  return SOR_OK;
}

// ------------------------------------------------------------------ K3/K4
template <typename R>
constexpr int wave_nst() { return 14; }

// ------------------------------------------------------------------ tiles
// One warp (pair) per tile = (strip, band of owned rows).  A tile runs whole
// 6-step batches and costs about its batch count x (alpha if it must keep
// ring/padding cells fixed, "masked", else 1).  Short bands waste the 4T-2
// warm-up steps and one partial extra wave doubles the tail, so if one wave of
// resident tiles gives bands <= 512 rows the launch is exactly one wave with
// batch counts equalised (one_wave below); otherwise ~8 waves of bands >= 256
// rows in row-major order.
// Geometry: a strip of wc columns overlaps its neighbours by `ghost` columns
// per side; a pass runs S stages (SOR: ghost = S = 2T; Jacobi: S = T).
static bool tile_masked(const sor_grid* g, int ghost, int S, int wc, int s0, int strip, int64_t R0, int64_t R1) {
  const int64_t sw = s0 + (int64_t)strip * (wc - 2 * ghost);
  const int64_t i_first = (R0 - (S - 1)) & ~1LL;
  const int64_t nsteps = (R1 + S - 1 - i_first + 5) / 6 * 6;
  return !((sw >= 1) && (sw + wc - 1 <= g->cols) && (i_first - 1 >= 1) &&
           (i_first + nsteps <= g->rows));
}

int wave_tiles(sor_grid* g, const Slab& s, int slab_idx, int ghost, int S, int wc, int tiles_per_sm, bool split,
               int s0, std::pair<int4*, int>* out) {
  const auto key = std::make_tuple(slab_idx, ((ghost * 16 + S) * 2 + (split ? 1 : 0)) * 1024 + wc, tiles_per_sm);
  auto it = g->tiles.find(key);
  if (it != g->tiles.end()) {
    *out = it->second;
    return SOR_OK;
  }
  static double alpha = -1.0, alpha2 = -1.0, waves = -1.0;
  static int64_t min_h = 0;
  if (alpha < 0) {
    const char* e = getenv("SOR_WAVE_ALPHA");
    alpha = e ? atof(e) : 1.33;  // edge-strip batch (SASS: 555/416 instructions at T=4)
    if (!(alpha >= 1.0)) alpha = 1.33;
    e = getenv("SOR_WAVE_ALPHA2");
    alpha2 = e ? atof(e) : 1.3;  // row-masked batch (measured best on C3; SASS 647/416)
    if (!(alpha2 >= 1.0)) alpha2 = 1.3;
    e = getenv("SOR_WAVE_WAVES");
    waves = e ? atof(e) : 0.0;  // 0 = automatic
    e = getenv("SOR_WAVE_MIN_BAND");
    min_h = e ? atoll(e) : 0;
  }
  const int64_t wout = wc - 2 * ghost;
  const int nstrips = (int)((g->cols + 1 - (s0 + ghost) + wout - 1) / wout);
  const int64_t nrows = s.g_hi - s.g_lo;
  const int64_t slots = (int64_t)g->nsm * tiles_per_sm;
  const int64_t warm = 2 * (S - 1);
  // split strip `w` given the target cost per tile (in row-steps)
  auto split_strip = [&](int w, double cost, std::vector<int4>* tl) {
    int64_t r = s.g_lo;
    while (r < s.g_hi) {
      // try an unmasked-height band first; fall back to the masked height
      int64_t h = std::max<int64_t>(8, (int64_t)(cost - warm));
      bool m = tile_masked(g, ghost, S, wc, s0, w, r, std::min(r + h, s.g_hi));
      if (m) h = std::max<int64_t>(8, (int64_t)(cost / alpha - warm));
      h = std::min<int64_t>(h, s.g_hi - r);
      if (tl) tl->push_back(make_int4(w, (int)r, (int)(r + h), tile_masked(g, ghost, S, wc, s0, w, r, r + h) ? 1 : 0));
      r += h;
    }
  };
  std::vector<int4> tl;
  // One-wave mode (every tile resident at once, so the launch lasts as long as
  // its slowest tile).  A tile runs whole 6-step batches; its cost in
  // unmasked-batch units mirrors the kernel's masking levels (run() in
  // sor_kernels.cuh): batches updating a ring/padding row cost alpha2, the
  // others alpha1 on an edge strip (column selects) and 1 elsewhere.  Each
  // tile gets the most batches whose cost fits the budget Bc; Bc is the
  // smallest budget whose tiles fit in one wave.
  auto tile_cost = [&](int w, int64_t R0, int64_t nb) -> double {
    const int64_t sw = s0 + (int64_t)w * wout;
    const bool col = !(sw >= 1 && sw + wc - 1 <= g->cols);
    const int64_t i_first = (R0 - (S - 1)) & ~1LL;
    const int64_t jA = std::min<int64_t>(nb, std::max<int64_t>(0, -floordiv6((int)(i_first - S))));
    const int64_t jB = std::max<int64_t>(jA, std::min<int64_t>(nb, floordiv6((int)(g->rows - 5 - i_first)) + 1));
    return (double)(jA + (nb - jB)) * alpha2 + (double)(jB - jA) * (col ? alpha : 1.0);
  };
  auto one_wave = [&](double Bc, std::vector<int4>* out_tl) -> int64_t {
    int64_t n = 0;
    for (int w = 0; w < nstrips; ++w) {
      int64_t r = s.g_lo;
      while (r < s.g_hi) {
        const int64_t i_first = (r - (S - 1)) & ~1LL;
        // batches needed to finish every remaining row of the strip; at least
        // enough for kMinBand rows (the solve's probe rows recur every 6 rows
        // from i_first, so a band of >= 6 rows holds one for every stage)
        const int64_t nb_all = (s.g_hi + S - 1 - i_first + 5) / 6;
        const int64_t kMinBand = 8;
        const int64_t nb_min = std::min<int64_t>(nb_all, (kMinBand + (S - 1) + (r - i_first) + 5) / 6);
        int64_t nb = std::min<int64_t>(nb_all, (int64_t)Bc);
        while (nb > nb_min && tile_cost(w, r, nb) > Bc) --nb;
        nb = std::max<int64_t>(nb, nb_min);
        const int64_t h = std::max<int64_t>(1, std::min(s.g_hi - r, i_first + 6 * nb - (S - 1) - r));
        if (out_tl) out_tl->push_back(make_int4(w, (int)r, (int)(r + h), 0));
        ++n;
        r += h;
      }
    }
    return n;
  };
  double Bc = 0.0;
  if (waves <= 0) {
    const double kOneWaveMaxB = (512.0 + warm + 5) / 6;
    for (double b = (double)((warm + 6) / 6 + 1); b <= kOneWaveMaxB; b += 0.125)
      if (one_wave(b, nullptr) <= slots) {
        Bc = b;
        break;
      }
  }
  if (Bc > 0) {
    one_wave(Bc, &tl);
  } else {
    // many waves (C4, C5): ~8 waves of bands >= 256 rows; the block scheduler
    // balances the load dynamically
    double cost;
    if (waves > 0) {
      const int64_t nb = std::max<int64_t>(1, (int64_t)(waves * slots) / nstrips);
      cost = (double)std::max<int64_t>(min_h > 0 ? min_h : 4 * S, (nrows + nb - 1) / nb) + warm;
    } else {
      const int64_t kMinH = min_h > 0 ? min_h : 256;
      const int64_t nb8 = std::max<int64_t>(1, 8 * slots / nstrips);
      cost = (double)std::max<int64_t>(kMinH, (nrows + nb8 - 1) / nb8) + warm;
    }
    for (int w = 0; w < nstrips; ++w) split_strip(w, cost, &tl);
  }
  // row-major order: warps running together stream neighbouring strips of the
  // same rows (shared ghost columns hit in L2, DRAM pages stay open)
  std::stable_sort(tl.begin(), tl.end(),
                   [](const int4& x, const int4& y) { return x.y != y.y ? x.y < y.y : x.x < y.x; });
  int4* d = nullptr;
  CU(cudaMalloc(&d, tl.size() * sizeof(int4)));
  // stream-ordered: a plain cudaMemcpy runs on the legacy stream and, from
  // pageable memory, may return before the DMA lands, while the kernels run on
  // a non-blocking stream, so a kernel could read a half-written table (the
  // suspected cause of one rare fuzz mismatch)
  CU(cudaMemcpyAsync(d, tl.data(), tl.size() * sizeof(int4), cudaMemcpyHostToDevice, g->stream));
  *out = {d, (int)tl.size()};
  g->tiles[key] = *out;
  return SOR_OK;
}

// Programmatic dependent launch between consecutive wave kernels (one slab:
// no NCCL or copy between them); SOR_NO_PDL=1 disables it.
bool wave_pdl(const sor_grid* g) {
  static int off = -1;
  if (off < 0) off = getenv("SOR_NO_PDL") ? 1 : 0;
  return !off && g->slabs.size() == 1 && g->nranks == 1;
}

// Split mode (a warp pair per tile, stages divided between the two warps) for
// T >= 2 unless SOR_WAVE_SPLIT=0 (with -DSOR_WAVE_NOSPLIT_VARIANTS).
[[maybe_unused]] bool wave_split(int T) {
  static int sp = -1;
  if (sp < 0) {
    const char* e = getenv("SOR_WAVE_SPLIT");
    sp = e ? atoi(e) : 1;
  }
  return sp != 0 && T >= 2;
}

template <typename R, int T, int CK, bool SPLIT, int NC>
int launch_wave_TS(sor_grid* g, const Slab& s, R w, const IterCtl& ctl, bool fused_fin) {
  constexpr int NST = wave_nst<R>();
  constexpr int smem = wave_smem_bytes<R, NST, SPLIT, NC>();
  constexpr int per_cta = wave_tiles_per_cta(SPLIT);
  static int occ = 0;  // resident CTAs/SM for this instance
  if (occ == 0) {
    CU(cudaFuncSetAttribute(wave_kernel<R, T, NST, CK, SPLIT, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wave_kernel<R, T, NST, CK, SPLIT, NC>, kWaveWarps * 32, smem);
    if (occ <= 0) occ = 1;
  }
  WaveArgs<R> a;
  a.src = col0<R>(s.plane[g->cur]);
  a.dst = col0<R>(s.plane[g->nxt(g->cur)]);
  a.pitch = g->pitch;
  a.g0 = s.g0;
  a.rows = g->rows;
  a.cols = g->cols;
  a.r_lo = s.g_lo;
  a.r_hi = s.g_hi;
  a.w = w;
  a.s0 = -4 * ((2 * T + 3) / 4);
  const int slab_idx = (int)(&s - &g->slabs[0]);
  std::pair<int4*, int> tt{nullptr, 0};
  TRY(wave_tiles(g, s, slab_idx, 2 * T, 2 * T, wave_cols<NC>(), occ * per_cta, SPLIT, a.s0, &tt));
  a.tiles = tt.first;
  a.ntiles = tt.second;
  const unsigned blocks = (unsigned)((a.ntiles + per_cta - 1) / per_cta) + (ctl.defer ? 1 : 0);
  IterCtl c = ctl;
  c.finalize = fused_fin ? 1 : 0;
  c.nparts = blocks;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kWaveWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = g->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  // PDL only for one-wave launches: in a multi-wave launch the next grid's
  // early CTAs would hold slots its own tail needs (measured: C5 -0.5%, C3 +2%)
  cfg.numAttrs = (wave_pdl(g) && blocks <= (unsigned)(occ * g->nsm)) ? 1 : 0;
  CU(cudaLaunchKernelEx(&cfg, wave_kernel<R, T, NST, CK, SPLIT, NC>, a, c, s.tmap[g->cur]));
  g->st.kernel_launches += 1;
  return SOR_OK;
}

template <typename R, int T, int CK>
int launch_wave_T(sor_grid* g, const Slab& s, R w, const IterCtl& ctl, bool fused_fin) {
  // 4 columns per lane: wider lanes (NC = 6, 8; bitwise equal) measured
  // slower on B200 at every T (fewer resident warps outweigh the extra ILP)
  // T >= 2: warp pairs (split); the single-warp variant is built only with
  // -DSOR_WAVE_NOSPLIT_VARIANTS (SOR_WAVE_SPLIT=0 then selects it)
#ifdef SOR_WAVE_NOSPLIT_VARIANTS
  if (T >= 2 && wave_split(T)) return launch_wave_TS<R, T, CK, (T >= 2), kWaveNC>(g, s, w, ctl, fused_fin);
  return launch_wave_TS<R, T, CK, false, kWaveNC>(g, s, w, ctl, fused_fin);
#else
  return launch_wave_TS<R, T, CK, (T >= 2), kWaveNC>(g, s, w, ctl, fused_fin);
#endif
}

template <typename R, int CK>
int launch_wave(sor_grid* g, const Slab& s, int T, R w, const IterCtl& ctl, bool fused_fin) {
  if (CK >= 3 && T == 1) return launch_wave_T<R, 1, 2>(g, s, w, ctl, fused_fin);  // unused combination
  switch (T) {
    case 1: return launch_wave_T<R, 1, CK>(g, s, w, ctl, fused_fin);
    case 2: return launch_wave_T<R, 2, CK>(g, s, w, ctl, fused_fin);
    case 3: return launch_wave_T<R, 3, CK>(g, s, w, ctl, fused_fin);
    case 4: return launch_wave_T<R, 4, CK>(g, s, w, ctl, fused_fin);
  }
  return set_error(nullptr, SOR_E_INVAL, "temporal depth %d unsupported", T);
}

// Jacobi pass (NEXT-2): jacobi_kernel on the wave tiles with ghost G and T stages.
template <typename R, int T, int CK>
int launch_jacobi_T(sor_grid* g, const Slab& s, const IterCtl& ctl, bool fused_fin) {
  constexpr int NST = wave_nst<R>();
  constexpr int smem = kWaveWarps * wave_smem_per_warp<R, NST, kWaveNC>();
  constexpr int G = jacobi_ghost(T);
  static int occ = 0;
  if (occ == 0) {
    CU(cudaFuncSetAttribute(jacobi_kernel<R, T, NST, CK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, jacobi_kernel<R, T, NST, CK>, kWaveWarps * 32, smem);
    if (occ <= 0) occ = 1;
  }
  WaveArgs<R> a;
  a.src = col0<R>(s.plane[g->cur]);
  a.dst = col0<R>(s.plane[g->nxt(g->cur)]);
  a.pitch = g->pitch;
  a.g0 = s.g0;
  a.rows = g->rows;
  a.cols = g->cols;
  a.r_lo = s.g_lo;
  a.r_hi = s.g_hi;
  a.w = R(1);
  a.s0 = -4 * ((G + 3) / 4);
  const int slab_idx = (int)(&s - &g->slabs[0]);
  std::pair<int4*, int> tt{nullptr, 0};
  TRY(wave_tiles(g, s, slab_idx, G, T, wave_cols<kWaveNC>(), occ * kWaveWarps, false, a.s0, &tt));
  a.tiles = tt.first;
  a.ntiles = tt.second;
  const unsigned blocks = (unsigned)((a.ntiles + kWaveWarps - 1) / kWaveWarps) + (ctl.defer ? 1 : 0);
  IterCtl c = ctl;
  c.finalize = fused_fin ? 1 : 0;
  c.nparts = blocks;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kWaveWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = g->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (wave_pdl(g) && blocks <= (unsigned)(occ * g->nsm)) ? 1 : 0;
  CU(cudaLaunchKernelEx(&cfg, jacobi_kernel<R, T, NST, CK>, a, c, s.tmap[g->cur]));
  g->st.kernel_launches += 1;
  return SOR_OK;
}

template <typename R, int CK>
int launch_jacobi(sor_grid* g, const Slab& s, int T, const IterCtl& ctl, bool fused_fin) {
  switch (T) {
    case 1: return launch_jacobi_T<R, 1, CK>(g, s, ctl, fused_fin);
    case 2: return launch_jacobi_T<R, 2, CK>(g, s, ctl, fused_fin);
    case 3: return launch_jacobi_T<R, 3, CK>(g, s, ctl, fused_fin);
    case 4: return launch_jacobi_T<R, 4, CK>(g, s, ctl, fused_fin);
  }
  return set_error(nullptr, SOR_E_INVAL, "temporal depth %d unsupported", T);
}

// One HBM pass of ctl.T iterations ending at iteration ctl.k_last.
template <typename R>
int wave_pass(sor_grid* g, R w, IterCtl ctl) {
  const int T = ctl.T;
  const bool fused_fin = single_part(g) && ctl.ck != 0 && !ctl.defer;
  if (!single_part(g) && g->halo_valid < 2 * T) TRY(exchange(g, g->cur, 2 * T));
  for (auto& s : g->slabs) {
    if (g->method == 1) {  // Jacobi: exact maxima only (ck 1 or 2)
      if (ctl.ck >= 2)
        TRY((launch_jacobi<R, 2>(g, s, T, ctl, fused_fin)));
      else if (ctl.ck == 1)
        TRY((launch_jacobi<R, 1>(g, s, T, ctl, fused_fin)));
      else
        TRY((launch_jacobi<R, 0>(g, s, T, ctl, fused_fin)));
      continue;
    }
    if (ctl.ck == 4)
      TRY((launch_wave<R, 4>(g, s, T, w, ctl, fused_fin)));
    else if (ctl.ck == 3)
      TRY((launch_wave<R, 3>(g, s, T, w, ctl, fused_fin)));
    else if (ctl.ck == 2)
      TRY((launch_wave<R, 2>(g, s, T, w, ctl, fused_fin)));
    else if (ctl.ck == 1)
      TRY((launch_wave<R, 1>(g, s, T, w, ctl, fused_fin)));
    else
      TRY((launch_wave<R, 0>(g, s, T, w, ctl, fused_fin)));
  }
  const int src = g->cur;
  g->cur = g->nxt(src);
  g->st.half_sweeps += g->method == 1 ? T : 2 * T;  // Jacobi: one sweep per iteration
  g->st.hbm_passes += 1;
  TRY(exchange(g, g->cur, 2 * T));
  g->halo_valid = 2 * T;
  if (ctl.ck && !fused_fin && !ctl.defer) TRY(join_and_finalize(g, ctl));
  g->pass_ends.push_back({ctl.k_last, src, g->cur, T});
  return SOR_OK;
}

// ------------------------------------------------------------------ K5
template <typename R>
int k5_run(sor_grid* g, R w, int solve, int64_t n_iter, double tol, int64_t K, int measure_last) {
  const Slab& s = g->slabs[0];
  const size_t smem = (size_t)(g->rows + 2) * (g->cols + 2) * sizeof(R);
  CU(cudaFuncSetAttribute(k5_small_solve<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k5_small_solve<R><<<1, 1024, smem, g->stream>>>(col0<R>(s.plane[g->cur]), g->pitch, s.g0, (int)g->rows,
                                                  (int)g->cols, w, solve, n_iter, tol, K, measure_last,
                                                  g->dstate);
  CU(cudaGetLastError());
  g->st.kernel_launches += 1;
  return SOR_OK;
}

size_t k5_limit_bytes() { return 200 * 1024; }

// ------------------------------------------------------------------ drivers
int begin_call(sor_grid* g) {
  g->st.kernel_launches = 0;
  g->st.half_sweeps = 0;
  g->st.halo_exchanges = 0;
  g->st.checks = 0;
  g->st.hbm_passes = 0;
  g->have_elapsed = false;
  g->pass_ends.clear();
  g->exact_reruns = 0;
  g->st.exact_reruns = 0;
  CU(cudaMemsetAsync(g->dstate, 0, sizeof(DevState), g->stream));
  CU(cudaEventRecord(g->ev0, g->stream));
  return SOR_OK;
}

int end_call(sor_grid* g, DevState* out) {
  CU(cudaEventRecord(g->ev1, g->stream));
  CU(cudaMemcpyAsync(&g->hstate[0], g->dstate, sizeof(DevState), cudaMemcpyDeviceToHost, g->stream));
  CU(cudaStreamSynchronize(g->stream));
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
  g->elapsed_ms = ms;
  g->have_elapsed = true;
  if (out) *out = g->hstate[0];
  return SOR_OK;
}

int depth_of(const sor_grid* g) { return g->kernel == SOR_KERNEL_TEMPORAL ? g->tdepth : 1; }

// Max-change mode of T-deep solve passes with check_every == 1: 4 (probe
// rows, default: 1.09-1.23x the cost of a plain pass on C3 vs 1.10-1.41x for
// all cells) or 3 (all cells, high words).  SOR_SOLVE_CK=3 overrides.
int solve_ck(int T) {
  static int ck = -1;
  if (ck < 0) {
    const char* e = getenv("SOR_SOLVE_CK");
    ck = e ? atoi(e) : 0;
  }
  (void)T;
  return ck == 3 ? 3 : 4;
}

// Enqueue iterations [k_from, k_to] (1-based within the call).
//  - iterate (base.solve == 0): passes of up to T; the last one reports its
//    last iteration's max-change if check_last.
//  - solve with check_every == 1 and T > 1: passes of T, each reporting the
//    max-change of every iteration it contains (ck = 2).
//  - otherwise: passes end exactly at every checked iteration (ck = 1 there).
template <typename R>
int enqueue_range(sor_grid* g, R w, int64_t k_from, int64_t k_to, const IterCtl& base, bool check_last) {
  const int64_t K = base.K;
  const int T = depth_of(g);
  int64_t k = k_from;
  if (g->kernel == SOR_KERNEL_NATURAL) {
    for (; k <= k_to; ++k) {
      IterCtl c = base;
      c.k_last = k;
      c.T = 1;
      c.ck = base.solve ? (k % K == 0) : (check_last && k == k_to);
      TRY(k1_iteration<R>(g, w, c));
      if (c.ck) g->st.checks += 1;
    }
    return SOR_OK;
  }
  const bool every = base.solve && K == 1 && T > 1;
  while (k <= k_to) {
    int64_t next_check = k_to + 1;
    if (base.solve && !every)
      next_check = ((k + K - 1) / K) * K;
    else if (!base.solve && check_last)
      next_check = k_to;
    const int64_t end = std::min(k_to, next_check);  // inclusive end of this block
    while (k <= end) {
      const int64_t left = end - k + 1;
      int t = (int)(left % T);  // remainder first, so a block ends on a full pass
      if (t == 0) t = T;
      IterCtl c = base;
      c.k_last = k + t - 1;
      c.T = t;
      c.ck = every ? g->every_ck : (c.k_last == next_check ? 1 : 0);
      if (base.defer) {
        // this launch's block 0 decides the last undecided checked pass
        c.prev_valid = g->prev_valid ? 1 : 0;
        c.prev_k_last = g->prev_k_last;
        c.prev_T = g->prev_T;
        c.prev_ck = g->prev_ck;
        c.prev_set = g->prev_set;
        g->prev_valid = false;
        c.set = g->next_set;
        if (c.ck) {
          g->prev_valid = true;
          g->prev_k_last = c.k_last;
          g->prev_T = c.T;
          g->prev_ck = c.ck;
          g->prev_set = c.set;
          g->next_set ^= 1;
        }
      }
      TRY(wave_pass<R>(g, w, c));
      if (c.ck) g->st.checks += every ? t : 1;
      k += t;
    }
  }
  return SOR_OK;
}

template <typename R>
int iterate_impl(sor_grid* g, double omega, int64_t iters, double* last) {
  TRY(begin_call(g));
  const R w = (R)omega;
  if (iters > 0) {
    if (g->kernel == SOR_KERNEL_SMALL) {
      TRY(k5_run<R>(g, w, 0, iters, 1.0, 1, last ? 1 : 0));
      g->st.half_sweeps += 2 * iters;
    } else {
      IterCtl base{};
      base.st = g->dstate;
      base.maxit = iters;
      base.K = 1;
      base.tol = 0.0;
      base.solve = 0;
      TRY(enqueue_range<R>(g, w, 1, iters, base, last != nullptr));
    }
  }
  DevState hs{};
  TRY(end_call(g, &hs));
  if (last) *last = iters > 0 ? hs.max_change : 0.0;
  return SOR_OK;
}

int read_state(sor_grid* g, DevState* out) {
  CU(cudaMemcpyAsync(&g->hstate[0], g->dstate, sizeof(DevState), cudaMemcpyDeviceToHost, g->stream));
  CU(cudaStreamSynchronize(g->stream));
  *out = g->hstate[0];
  return SOR_OK;
}

// The pass of this solve segment that contains iteration k.
bool find_pass(const sor_grid* g, int64_t k, sor_grid::PassRec* out) {
  for (const auto& pe : g->pass_ends) {
    if (k <= pe.k_last && k > pe.k_last - pe.T) {
      *out = pe;
      return true;
    }
  }
  return false;
}

// Re-run the first `depth` iterations of the pass that ended at k_end from its
// source plane (untouched: later passes of the segment exited early), with
// the exact max-change of its last iteration (ck=1) or of every iteration
// (ck=2, solve semantics).  Leaves g->cur on the plane holding the result.
template <typename R>
int rerun_pass(sor_grid* g, R w, const IterCtl& base, const sor_grid::PassRec& pr, int depth, int ck, DevState* out) {
  CU(cudaMemsetAsync(g->dstate, 0, sizeof(DevState), g->stream));
  g->cur = pr.src;  // writes the pass's own destination plane again
  IterCtl c = base;
  c.k_last = pr.k_last - pr.T + depth;
  c.T = depth;
  c.ck = ck;
  c.solve = ck == 2 ? 1 : 0;
  c.defer = 0;
  c.set = 0;
  TRY(wave_pass<R>(g, w, c));
  return read_state(g, out);
}

// Third plane for the deferred stop test (single slab): allocated once, a copy
// of the current plane (ring, padding); false if memory is short.
bool ensure_third_plane(sor_grid* g) {
  if (g->nplanes == 3) return true;
  if (!single_part(g)) return false;
  static int off = -1;
  if (off < 0) off = getenv("SOR_NO_DEFER") ? 1 : 0;
  if (off) return false;
  Slab& s = g->slabs[0];
  const size_t bytes = (size_t)s.nstore * g->pitch * g->esz;
  if (cudaMalloc(&s.plane[2], bytes) != cudaSuccess) {
    cudaGetLastError();
    s.plane[2] = nullptr;
    return false;
  }
  if (cudaMemcpyAsync(s.plane[2], s.plane[g->cur], bytes, cudaMemcpyDeviceToDevice, g->stream) != cudaSuccess ||
      make_tmaps(g, s, 2) != SOR_OK) {
    cudaFree(s.plane[2]);
    s.plane[2] = nullptr;
    return false;
  }
  g->nplanes = 3;
  return true;
}

template <typename R>
int solve_impl(sor_grid* g, double omega, double tol, int64_t maxit, int64_t K, int64_t* iters_out,
               double* max_out) {
  TRY(begin_call(g));
  const R w = (R)omega;
  DevState hs{};
  bool converged = false;
  int64_t done = maxit;
  double maxc = 0.0;
  if (g->kernel == SOR_KERNEL_SMALL) {
    TRY(k5_run<R>(g, w, 1, maxit, tol, K, 0));
    TRY(end_call(g, &hs));
    g->st.checks = hs.checks;
    converged = hs.converged != 0;
    done = converged ? hs.conv_iter : maxit;
    maxc = hs.max_change;
  } else {
    IterCtl base{};
    base.st = g->dstate;
    base.maxit = maxit;
    base.K = K;
    base.tol = tol;
    base.solve = 1;
    {
      uint64_t tb;
      memcpy(&tb, &tol, 8);
      base.tol_hi = (unsigned)(tb >> 32);
    }
    const bool fast = g->kernel != SOR_KERNEL_NATURAL && K == 1 && depth_of(g) > 1;  // ck=3/4 passes
    // Deferred stop test (wave kernels, one slab): no ticket at the end of a
    // checked pass; the next launch's block 0 decides it while the rest of
    // that launch runs speculatively into the third plane, and the launch
    // after exits early once a test stopped.  Pass p's source plane survives
    // pass p+1 (three-plane rotation), so an exact re-run is always possible.
    base.defer = (g->kernel != SOR_KERNEL_NATURAL && ensure_third_plane(g)) ? 1 : 0;
    // batches of whole check blocks (and whole passes); poll one batch behind
    const int64_t unit = std::max<int64_t>(K, depth_of(g));
    static int64_t batch_its = -1;  // iterations enqueued between polls (SOR_SOLVE_BATCH)
    if (batch_its < 0) {
      const char* e = getenv("SOR_SOLVE_BATCH");
      batch_its = e ? std::max<int64_t>(1, atoll(e)) : 64;
    }
    const int64_t blk = std::max<int64_t>(unit, (int64_t)((batch_its + unit - 1) / unit) * unit);
    int64_t k = 1;
    int64_t checks = 0;
    // far from convergence the probe (ck=4) proves "not converged" at 1/6 of
    // the max-change cost; after its first inconclusive pass the solve is
    // near the end and switches to all cells (ck=3) to avoid repeated re-runs
    g->every_ck = g->method == 1 ? 2 : solve_ck(depth_of(g));
    int probe_misses = 0;
    while (true) {
      // one segment: iterations k..maxit until the device stops the loop
      CU(cudaMemsetAsync(g->dstate, 0, sizeof(DevState), g->stream));
      g->pass_ends.clear();
      g->prev_valid = false;
      g->next_set = 0;
      int b = 0;
      for (int64_t kk = k; kk <= maxit;) {
        const int64_t k_to = std::min(maxit, kk + blk - 1);
        TRY(enqueue_range<R>(g, w, kk, k_to, base, false));
        CU(cudaMemcpyAsync(&g->hstate[b & 1], g->dstate, sizeof(DevState), cudaMemcpyDeviceToHost,
                           g->stream));
        CU(cudaEventRecord(g->poll_ev[b & 1], g->stream));
        kk = k_to + 1;
        if (b >= 1) {
          CU(cudaEventSynchronize(g->poll_ev[(b - 1) & 1]));
          if (g->hstate[(b - 1) & 1].stop) break;
        }
        ++b;
      }
      if (base.defer && g->prev_valid) {
        // the last enqueued checked pass has no successor to decide it
        IterCtl c = base;
        c.k_last = g->prev_k_last;
        c.T = g->prev_T;
        c.ck = g->prev_ck;
        c.set = g->prev_set;
        c.defer = 0;
        finalize_kernel<<<1, 32, 0, g->stream>>>(c);
        CU(cudaGetLastError());
        g->st.kernel_launches += 1;
        g->prev_valid = false;
      }
      TRY(read_state(g, &hs));
      checks += hs.checks;
      if (g->kernel == SOR_KERNEL_NATURAL) {  // in place, exact checks: nothing to redo
        converged = hs.converged != 0;
        done = converged ? hs.conv_iter : maxit;
        maxc = hs.max_change;
        break;
      }
      sor_grid::PassRec pr{};
      if (hs.ambiguous) {
        // ck=3: high words tied with tol's; ck=4: the probe could not exclude
        // convergence.  Decide this pass exactly
        g->exact_reruns += 1;
        if (getenv("SOR_DEBUG")) fprintf(stderr, "[sor] exact re-run at iteration %lld\n", (long long)hs.amb_iter);
        if (!find_pass(g, hs.amb_iter, &pr))
          return set_error(g, SOR_E_STATE, "internal: pass of iteration %lld not found", (long long)hs.amb_iter);
        checks -= (hs.amb_iter - (pr.k_last - pr.T + 1)) + 1;  // the exact pass re-counts them
        DevState ex{};
        TRY(rerun_pass<R>(g, w, base, pr, pr.T, 2, &ex));
        if (ex.converged) {
          checks += ex.checks;
          converged = true;
          done = ex.conv_iter;
          const int depth = (int)(done - (pr.k_last - pr.T));
          DevState fin{};
          TRY(rerun_pass<R>(g, w, base, pr, depth, 1, &fin));
          maxc = fin.max_change;
          break;
        }
        checks += ex.checks;
        maxc = ex.max_change;
        // near convergence (exact max within 16x tol) probing would keep
        // failing: switch to all cells.  Far from it (e.g. a probe that saw
        // only still-unchanged rows) keep probing.
        {
          static double sw = -1.0;
          if (sw < 0) {
            const char* e = getenv("SOR_SOLVE_SWITCH");
            sw = e ? atof(e) : 16.0;
          }
          if (getenv("SOR_DEBUG"))
            fprintf(stderr, "[sor] re-run at %lld: probe hi %.6e exact %.6e (tol %.3e)\n", (long long)hs.amb_iter,
                    hs.max_change, ex.max_change, tol);
          // a probe that keeps missing far from convergence (nothing changes
          // on its rows yet) would cost a re-run per pass: after the second
          // inconclusive probe check all cells instead
          if (ex.max_change < sw * tol || ++probe_misses >= 2) g->every_ck = 3;
        }
        k = pr.k_last + 1;  // g->cur now holds X_{k_last}
        if (k > maxit) {
          done = maxit;
          break;
        }
        continue;
      }
      if (hs.converged) {
        converged = true;
        done = hs.conv_iter;
      } else {
        done = maxit;
      }
      if (!find_pass(g, done, &pr))
        return set_error(g, SOR_E_STATE, "internal: pass of iteration %lld not found", (long long)done);
      if (fast) {
        // X_done and its exact max-change: re-run the pass up to `done`
        DevState fin{};
        TRY(rerun_pass<R>(g, w, base, pr, (int)(done - (pr.k_last - pr.T)), 1, &fin));
        maxc = fin.max_change;
      } else {
        g->cur = pr.dst;  // passes end on checked iterations
        maxc = hs.max_change;
      }
      break;
    }
    TRY(end_call(g, &hs));
    g->st.checks = checks;
    g->st.exact_reruns = g->exact_reruns;
  }
  g->st.half_sweeps = g->method == 1 ? done : 2 * done;
  if (iters_out) *iters_out = converged ? done : maxit;
  if (max_out) *max_out = maxc;
  return converged ? SOR_OK : SOR_NOT_CONVERGED;
}

int validate_omega(double omega) {
  if (!(omega > 0.0 && omega < 2.0))
    return set_error(nullptr, SOR_E_INVAL, "omega must satisfy 0 < omega < 2 (P:100), got %g", omega);
  return SOR_OK;
}

}  // namespace

// ======================================================================= ABI
extern "C" {

const char* sor_last_error(void) { return g_last_error.c_str(); }

int sor_partition_rows(int64_t rows, int P, int p, int64_t* lo, int64_t* hi) {
  if (!lo || !hi) return set_error(nullptr, SOR_E_INVAL, "NULL output");
  int rc = partition(rows, P, p, lo, hi);
  if (rc) return set_error(nullptr, rc, "partition: need P >= 1, 0 <= p < P, rows >= P");
  return SOR_OK;
}

int sor_create(sor_grid** out, int64_t N, const double* init, sor_dtype dt) {
  return create_common(out, N, N, init, dt, Mode::Single, 1, 0, 1, 0, nullptr);
}

int sor_create_rect(sor_grid** out, int64_t rows, int64_t cols, const double* init, sor_dtype dt) {
  return create_common(out, rows, cols, init, dt, Mode::Single, 1, 0, 1, 0, nullptr);
}

int sor_create_virtual(sor_grid** out, int64_t rows, int64_t cols, const double* init, sor_dtype dt,
                       int nslabs) {
  return create_common(out, rows, cols, init, dt, Mode::Virtual, nslabs, 0, 1, 0, nullptr);
}

int sor_create_dist(sor_grid** out, int64_t rows, int64_t cols, const double* init, sor_dtype dt,
                    int rank, int nranks, int device, const void* nccl_id) {
  return create_common(out, rows, cols, init, dt, Mode::Dist, 1, rank, nranks, device, nccl_id);
}

int sor_nccl_unique_id(void* out128) {
  if (!out128) return set_error(nullptr, SOR_E_INVAL, "NULL output");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return set_error(nullptr, SOR_E_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  memcpy(out128, &id, sizeof id);
  return SOR_OK;
}

int sor_set_kernel(sor_grid* g, int kernel, int temporal_depth) {
  TRY(usable(g));
  switch (kernel) {
    case SOR_KERNEL_NATURAL:
    case SOR_KERNEL_FUSED:
      g->kernel = kernel;
      g->tdepth = 1;
      break;
    case SOR_KERNEL_TEMPORAL:
      if (temporal_depth < 1 || temporal_depth > 4)
        return set_error(nullptr, SOR_E_INVAL, "temporal_depth must be in [1,4], got %d", temporal_depth);
      if (g->slabs.size() > 1 || g->nranks > 1) {
        for (auto& s : g->slabs)
          if (s.g_hi - s.g_lo < 2 * temporal_depth)
            return set_error(nullptr, SOR_E_INVAL, "slab of %lld rows too thin for T=%d",
                             (long long)(s.g_hi - s.g_lo), temporal_depth);
      }
      g->kernel = kernel;
      g->tdepth = temporal_depth;
      break;
    case SOR_KERNEL_SMALL: {
      if (!single_part(g))
        return set_error(nullptr, SOR_E_UNSUPPORTED, "SOR_KERNEL_SMALL needs a single-slab grid");
      const size_t bytes = (size_t)(g->rows + 2) * (g->cols + 2) * g->esz;
      if (bytes > k5_limit_bytes())
        return set_error(nullptr, SOR_E_UNSUPPORTED, "grid of %zu bytes exceeds shared memory", bytes);
      g->kernel = kernel;
      g->tdepth = 1;
      break;
    }
    default:
      return set_error(nullptr, SOR_E_INVAL, "unknown kernel %d", kernel);
  }
  g->st.kernel = g->kernel;
  g->st.temporal_depth = g->tdepth;
  return SOR_OK;
}

int sor_set_stream(sor_grid* g, void* cuda_stream) {
  TRY(usable(g));
  CU(cudaStreamSynchronize(g->stream));
  g->stream = cuda_stream ? (cudaStream_t)cuda_stream : g->own_stream;
  return SOR_OK;
}

int sor_iterate(sor_grid* g, double omega, int64_t iters, double* last_max_change) {
  TRY(usable(g));
  TRY(validate_omega(omega));
  if (iters < 0) return set_error(nullptr, SOR_E_INVAL, "iters must be >= 0");
  if (g->dt == SOR_F64) return iterate_impl<double>(g, omega, iters, last_max_change);
  return iterate_impl<float>(g, omega, iters, last_max_change);
}

int sor_solve(sor_grid* g, double omega, double tol, int64_t maxit, int64_t check_every,
              int64_t* iters_out, double* max_change_out) {
  TRY(usable(g));
  TRY(validate_omega(omega));
  if (!(tol > 0.0) || !std::isfinite(tol)) return set_error(nullptr, SOR_E_INVAL, "tol must be finite and > 0");
  if (maxit < 1) return set_error(nullptr, SOR_E_INVAL, "maxit must be >= 1");
  if (check_every < 1 || check_every > maxit)
    return set_error(nullptr, SOR_E_INVAL, "need 1 <= check_every <= maxit (S:114)");
  if (g->dt == SOR_F64) return solve_impl<double>(g, omega, tol, maxit, check_every, iters_out, max_change_out);
  return solve_impl<float>(g, omega, tol, maxit, check_every, iters_out, max_change_out);
}

namespace {
struct MethodGuard {  // run one call with the Jacobi method, then restore SOR
  sor_grid* g;
  explicit MethodGuard(sor_grid* gg) : g(gg) { g->method = 1; }
  ~MethodGuard() { g->method = 0; }
};
int jacobi_usable(sor_grid* g) {
  if (g->kernel != SOR_KERNEL_FUSED && g->kernel != SOR_KERNEL_TEMPORAL)
    return set_error(nullptr, SOR_E_UNSUPPORTED, "Jacobi runs on the FUSED / TEMPORAL kernels only");
  return SOR_OK;
}
}  // namespace

int sor_jacobi_iterate(sor_grid* g, int64_t iters, double* last_max_change) {
  TRY(usable(g));
  TRY(jacobi_usable(g));
  if (iters < 0) return set_error(nullptr, SOR_E_INVAL, "iters must be >= 0");
  MethodGuard mg(g);
  if (g->dt == SOR_F64) return iterate_impl<double>(g, 1.0, iters, last_max_change);
  return iterate_impl<float>(g, 1.0, iters, last_max_change);
}

int sor_jacobi_solve(sor_grid* g, double tol, int64_t maxit, int64_t check_every, int64_t* iters_out,
                     double* max_change_out) {
  TRY(usable(g));
  TRY(jacobi_usable(g));
  if (!(tol > 0.0) || !std::isfinite(tol)) return set_error(nullptr, SOR_E_INVAL, "tol must be finite and > 0");
  if (maxit < 1) return set_error(nullptr, SOR_E_INVAL, "maxit must be >= 1");
  if (check_every < 1 || check_every > maxit)
    return set_error(nullptr, SOR_E_INVAL, "need 1 <= check_every <= maxit (S:114)");
  MethodGuard mg(g);
  if (g->dt == SOR_F64) return solve_impl<double>(g, 1.0, tol, maxit, check_every, iters_out, max_change_out);
  return solve_impl<float>(g, 1.0, tol, maxit, check_every, iters_out, max_change_out);
}

int sor_download(sor_grid* g, double* out) {
  TRY(usable(g));
  if (g->mode != Mode::Dist || g->rank == 0) {
    if (!out) return set_error(nullptr, SOR_E_INVAL, "out is NULL");
  }
  CU(cudaStreamSynchronize(g->stream));
  if (g->mode != Mode::Dist) {
    const int n = (int)g->slabs.size();
    for (int k = 0; k < n; ++k) {
      const Slab& s = g->slabs[k];
      const int64_t ga = k == 0 ? 0 : s.g_lo;
      const int64_t gb = k == n - 1 ? g->rows + 2 : s.g_hi;
      TRY(store_rows(g, s, g->cur, out, ga, gb));
    }
    CU(cudaStreamSynchronize(g->stream));
    return SOR_OK;
  }
  // dist: rank 0 gathers every slab (owned rows; first/last include the ring)
  const Slab& s = g->slabs[0];
  const size_t row_bytes = (size_t)g->pitch * g->esz;
  const int64_t my_a = g->rank == 0 ? 0 : s.g_lo;
  const int64_t my_b = g->rank == g->nranks - 1 ? g->rows + 2 : s.g_hi;
  if (g->rank == 0) {
    TRY(store_rows(g, s, g->cur, out, my_a, my_b));
    for (int p = 1; p < g->nranks; ++p) {
      int64_t lo, hi;
      partition(g->rows, g->nranks, p, &lo, &hi);
      const int64_t a = lo, b = p == g->nranks - 1 ? g->rows + 2 : hi;
      // receive into a temporary slab-shaped buffer, then unpack
      void* tmp = nullptr;
      CU(cudaMalloc(&tmp, (size_t)(b - a) * row_bytes));
      NC(ncclRecv(tmp, (b - a) * row_bytes, ncclUint8, p, g->comm, g->stream));
      Slab t;
      t.g0 = a;
      t.plane[0] = (char*)tmp - 0;  // rows start at global row a
      t.nstore = b - a;
      t.plane[1] = t.plane[0];
      int rc = store_rows(g, t, 0, out, a, b);
      CU(cudaStreamSynchronize(g->stream));
      cudaFree(tmp);
      if (rc < 0) return rc;
    }
  } else {
    NC(ncclSend((char*)s.plane[g->cur] + (my_a - s.g0) * row_bytes, (my_b - my_a) * row_bytes,
                ncclUint8, 0, g->comm, g->stream));
  }
  CU(cudaStreamSynchronize(g->stream));
  return SOR_OK;
}

int sor_download_rows(sor_grid* g, int64_t row_a, int64_t row_b, double* out) {
  TRY(usable(g));
  if (g->mode == Mode::Dist) return set_error(nullptr, SOR_E_UNSUPPORTED, "download_rows: not on dist handles");
  if (!out || row_a < 0 || row_b > g->rows + 2 || row_a >= row_b)
    return set_error(nullptr, SOR_E_INVAL, "download_rows: need 0 <= row_a < row_b <= rows+2 and out");
  CU(cudaStreamSynchronize(g->stream));
  const int n = (int)g->slabs.size();
  const int64_t w = g->cols + 2;
  for (int k = 0; k < n; ++k) {
    const Slab& s = g->slabs[k];
    const int64_t sa = std::max(row_a, k == 0 ? (int64_t)0 : s.g_lo);
    const int64_t sb = std::min(row_b, k == n - 1 ? g->rows + 2 : s.g_hi);
    if (sa >= sb) continue;
    // store_rows indexes `out` by global row; shift the base accordingly
    TRY(store_rows(g, s, g->cur, out - row_a * w, sa, sb));
  }
  CU(cudaStreamSynchronize(g->stream));
  return SOR_OK;
}

int sor_reset(sor_grid* g, const double* init) {
  TRY(usable(g));
  if (!init) return set_error(nullptr, SOR_E_INVAL, "init is NULL");
  const bool on_dev = is_device_ptr(init);
  TRY(check_finite(g, init, (g->rows + 2) * (g->cols + 2), on_dev));
  return load_all(g, init);
}

int sor_last_elapsed_ms(const sor_grid* g, double* ms) {
  if (!g || !ms) return set_error(nullptr, SOR_E_INVAL, "NULL argument");
  if (!g->have_elapsed) return set_error(nullptr, SOR_E_STATE, "no iterate/solve call timed yet");
  *ms = g->elapsed_ms;
  return SOR_OK;
}

int sor_get_stats(const sor_grid* g, sor_stats* out) {
  if (!g || !out) return set_error(nullptr, SOR_E_INVAL, "NULL argument");
  *out = g->st;
  return SOR_OK;
}

void sor_destroy(sor_grid* g) {
  if (!g) return;
  if (g->stream) cudaStreamSynchronize(g->stream);
  free_grid(g);
}

}  // extern "C"

// ====================================================================== 3-D
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
  // default NATURAL: the fused z-wavefront is bitwise equal but slower on
  // B200 (f64 57 vs 158 GLUP/s at 512^3: the correctly rounded division on its
  // per-plane critical path, one CTA barrier per plane)
  int kernel = SOR_KERNEL_NATURAL;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, poll_ev[2] = {nullptr, nullptr};
  DevState* dstate = nullptr;
  DevState* hstate = nullptr;
  double* scratch = nullptr;
  bool failed = false, have_elapsed = false;
  double elapsed_ms = 0.0;
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

template <typename R>
int k3d_iteration(sor3d_grid* g, R w, const IterCtl& ctl) {
  if (g->kernel == SOR_KERNEL_FUSED) {
    dim3 grid((unsigned)((g->nx + 2 + kX3 - 1) / kX3), (unsigned)((g->ny + 2 + kY3 - 1) / kY3));
    IterCtl c = ctl;
    c.finalize = ctl.ck ? 1 : 0;
    c.nparts = grid.x * grid.y;
    if (ctl.ck)
      k3d_fused<R, true><<<grid, kW3P * kW3Y, 0, g->stream>>>((const R*)g->plane, (R*)g->plane2, g->pitch,
                                                             (int)g->nz, (int)g->ny, (int)g->nx, w, c);
    else
      k3d_fused<R, false><<<grid, kW3P * kW3Y, 0, g->stream>>>((const R*)g->plane, (R*)g->plane2, g->pitch,
                                                              (int)g->nz, (int)g->ny, (int)g->nx, w, c);
    CU3(cudaGetLastError());
    std::swap(g->plane, g->plane2);
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
  if (g->kernel == SOR_KERNEL_FUSED && solve && hs.converged && ((enq - hs.conv_iter) & 1))
    std::swap(g->plane, g->plane2);
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
  g->nz = nz;
  g->ny = ny;
  g->nx = nx;
  g->dt = dt;
  g->esz = dt == SOR_F64 ? 8 : 4;
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
  if (g->stream) cudaStreamSynchronize(g->stream);
  free3d(g);
}

}  // extern "C"
