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

#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <random>

#include "sor_internal.h"
#include "wave2.cuh"

static_assert(SOR_MAX_T == sorb::kMaxT, "include/sor.h and the kernels disagree on the deepest T");

namespace sorh {
thread_local std::string g_last_error;
}  // namespace sorh

using namespace sorh;

namespace sorh {

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


cudaMemcpyKind kDefault = cudaMemcpyDefault;

// ------------------------------------------------------------------ dist-IPC rendezvous
// The ranks of a dist-IPC handle are processes on one node.  They meet in a
// POSIX shared-memory segment named by the 128-byte id (sor_ipc_unique_id on
// rank 0, broadcast by the caller), publish their CUDA-IPC handles there and
// use it as a host barrier for the collective calls (create, reset,
// download, the start of iterate/solve, exact re-runs, and every pass in
// lockstep mode).  Kernels synchronise through device flags (HaloLink,
// DistComm), never through this segment.
struct RankInfo {
  cudaIpcMemHandle_t plane[3];
  cudaIpcMemHandle_t comm;
  int64_t g_lo, g_hi, g0, nstore;
  char bus_id[32];
  int nplanes;
  int ok;
  unsigned long long seq;
};
struct ShmHdr {
  uint32_t magic;
  uint32_t nranks;
  std::atomic<uint32_t> arrived;
  std::atomic<uint32_t> generation;
  std::atomic<int32_t> status;  // rank 0's verdict on the init (scatter), shared with all
  RankInfo rank[kMaxRanks];
};
static_assert(std::atomic<uint32_t>::is_always_lock_free, "process-shared atomics need lock-free types");
constexpr uint32_t kShmMagic = 0x534f5242u;  // "SORB"

struct ShmSeg {
  ShmHdr* h = nullptr;
  std::string name;
  bool owner = false;
};

int shm_open_seg(sor_grid* g, const char* id, int rank, int nranks) {
  char name[128];
  memcpy(name, id, 127);
  name[127] = 0;
  if (name[0] != '/' || strlen(name) < 8) return set_error(nullptr, SOR_E_INVAL, "dist-ipc: bad id (use sor_ipc_unique_id)");
  ShmSeg* s = new ShmSeg();
  s->name = name;
  int fd = -1;
  if (rank == 0) {
    fd = shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) {
      delete s;
      return set_error(nullptr, SOR_E_STATE, "dist-ipc: shm_open(%s) failed (id reused?)", name);
    }
    if (ftruncate(fd, sizeof(ShmHdr)) != 0) {
      close(fd);
      shm_unlink(name);
      delete s;
      return set_error(nullptr, SOR_E_STATE, "dist-ipc: ftruncate failed");
    }
    s->owner = true;
  } else {
    const auto t0 = std::chrono::steady_clock::now();
    while ((fd = shm_open(name, O_RDWR, 0600)) < 0) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
        delete s;
        return set_error(nullptr, SOR_E_STATE, "dist-ipc: rank %d: segment %s never appeared", rank, name);
      }
      usleep(1000);
    }
    struct stat stt{};
    const auto t1 = std::chrono::steady_clock::now();
    while (fstat(fd, &stt) == 0 && (size_t)stt.st_size < sizeof(ShmHdr)) {
      if (std::chrono::steady_clock::now() - t1 > std::chrono::seconds(120)) {
        close(fd);
        delete s;
        return set_error(nullptr, SOR_E_STATE, "dist-ipc: rank %d: segment %s never sized", rank, name);
      }
      usleep(1000);
    }
  }
  void* p = mmap(nullptr, sizeof(ShmHdr), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) {
    if (rank == 0) shm_unlink(name);
    delete s;
    return set_error(nullptr, SOR_E_STATE, "dist-ipc: mmap failed");
  }
  s->h = reinterpret_cast<ShmHdr*>(p);
  if (rank == 0) {
    s->h->nranks = (uint32_t)nranks;
    s->h->arrived.store(0);
    s->h->generation.store(0);
    s->h->status.store(0);
    std::atomic_thread_fence(std::memory_order_seq_cst);
    __atomic_store_n(&s->h->magic, kShmMagic, __ATOMIC_RELEASE);
  } else {
    const auto t0 = std::chrono::steady_clock::now();
    while (__atomic_load_n(&s->h->magic, __ATOMIC_ACQUIRE) != kShmMagic) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
        munmap(p, sizeof(ShmHdr));
        delete s;
        return set_error(nullptr, SOR_E_STATE, "dist-ipc: segment never initialised");
      }
      usleep(500);
    }
    if (s->h->nranks != (uint32_t)nranks) {
      munmap(p, sizeof(ShmHdr));
      delete s;
      return set_error(nullptr, SOR_E_INVAL, "dist-ipc: nranks mismatch between ranks");
    }
  }
  g->shm = s;
  return SOR_OK;
}

void shm_close_seg(ShmSeg* s) {
  if (!s) return;
  if (s->h) munmap(s->h, sizeof(ShmHdr));
  if (s->owner) shm_unlink(s->name.c_str());
  delete s;
}

// Host barrier of all ranks (sense by generation).  Spins with yields; gives
// up after `timeout_s` (a rank that died or diverged must not hang the rest).
int shm_barrier(sor_grid* g, double timeout_s = 300.0) {
  ShmHdr* h = g->shm->h;
  const uint32_t gen = h->generation.load(std::memory_order_acquire);
  if (h->arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == h->nranks) {
    h->arrived.store(0, std::memory_order_relaxed);
    h->generation.fetch_add(1, std::memory_order_acq_rel);
    return SOR_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  unsigned spins = 0;
  while (h->generation.load(std::memory_order_acquire) == gen) {
    if (++spins > 256) {
      sched_yield();
      if ((spins & 1023) == 0 &&
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
      {
        g->failed = true;  // the ranks disagree on the call sequence; nothing can recover
        return set_error(g, SOR_E_STATE, "dist-ipc: barrier timed out on rank %d", g->rank);
      }
    }
  }
  return SOR_OK;
}

// Barrier of a dist-IPC handle; a no-op for every other handle.
int dist_barrier(sor_grid* g) {
  if (g->transport != Transport::Ipc) return SOR_OK;
  return shm_barrier(g);
}

// Dist-IPC: every rank takes the largest pass sequence number of all ranks
// (passes enqueued after a stop exit early without releasing any flag, so
// any common value at least as large as every released one is consistent).
int sync_seq(sor_grid* g) {
  if (g->transport != Transport::Ipc) return SOR_OK;
  ShmHdr* h = g->shm->h;
  h->rank[g->rank].seq = g->seq;
  TRY(shm_barrier(g));
  unsigned long long m = 0;
  for (int q = 0; q < g->nranks; ++q) m = std::max<unsigned long long>(m, h->rank[q].seq);
  TRY(shm_barrier(g));
  g->seq = m;
  return SOR_OK;
}

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
  for (int b = 0; b < 4; ++b) {
    // wave kernel: 6-row and 2-row boxes; skew-2 wave kernel: 4-row and 3-row
    static const cuuint32_t hgt[4] = {6u, 2u, (cuuint32_t)kW2Batch, 3u};
    const cuuint32_t box[2] = {(cuuint32_t)wave_cols<kWaveNC>(), hgt[b]};
    CUtensorMap* m = b < 2 ? &s.tmap[p].m[b] : &s.tmap2[p].m[b - 2];
    CUresult r = encode(m, g->dt == SOR_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
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
  // a device-resident init may still be being written by the caller's work on
  // another stream (torch's current stream, the legacy stream): order every
  // read of it after all of that work
  CU(cudaDeviceSynchronize());
  CU(cudaMemsetAsync(g->dflag, 0, sizeof(unsigned int), g->stream));
  count_nonfinite<<<4 * g->nsm, 256, 0, g->stream>>>(init, n, g->dflag);
  CU(cudaGetLastError());
  unsigned int bad = 0;
  CU(cudaMemcpyAsync(&bad, g->dflag, sizeof bad, cudaMemcpyDeviceToHost, g->stream));
  CU(cudaStreamSynchronize(g->stream));
  if (bad) return set_error(nullptr, SOR_E_INVAL, "init contains non-finite values");
  return SOR_OK;
}

void reset_plane_info(sor_grid* g) {
  for (auto& pi : g->pinfo) pi = PlaneInfo{};
  g->cur = 0;
  g->halo_valid = kRowPad;
}

// Fill every plane of slab s from init: global rows within the slab's storage
// window that exist in [0, rows+1] (own rows, ring, initial halos).
int load_slab(sor_grid* g, const Slab& s, const double* init) {
  const size_t bytes = (size_t)s.nstore * g->pitch * g->esz;
  CU(cudaMemsetAsync(s.plane[0], 0, bytes, g->stream));
  const int64_t ga = std::max<int64_t>(0, s.g0);
  const int64_t gb = std::min<int64_t>(g->rows + 2, s.g0 + s.nstore);
  TRY(load_rows(g, s, 0, init, ga, gb));
  for (int p = 1; p < 3; ++p)
    if (s.plane[p]) CU(cudaMemcpyAsync(s.plane[p], s.plane[0], bytes, cudaMemcpyDeviceToDevice, g->stream));
  return SOR_OK;
}

int load_all(sor_grid* g, const double* init) {
  for (auto& s : g->slabs) TRY(load_slab(g, s, init));
  reset_plane_info(g);
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
  if (g->device >= 0) cudaSetDevice(g->device);
  for (void* p : g->ipc_opened) cudaIpcCloseMemHandle(p);
  for (auto& s : g->slabs)
    for (int p = 0; p < 3; ++p)
      if (s.plane[p]) cudaFree(s.plane[p]);
  if (g->dstate) cudaFree(g->dstate);
  if (g->hstate) cudaFreeHost(g->hstate);
  if (g->scratch) cudaFree(g->scratch);
  if (g->dflag) cudaFree(g->dflag);
  if (g->gbar) cudaFree(g->gbar);
  if (g->rflags) cudaFree(g->rflags);
  if (g->flagbuf) cudaFree(g->flagbuf);
  if (g->djoin) cudaFree(g->djoin);
  if (g->vctl) cudaFree(g->vctl);
  if (g->vhost) cudaFreeHost(g->vhost);
  if (g->ev0) cudaEventDestroy(g->ev0);
  if (g->ev1) cudaEventDestroy(g->ev1);
  for (int k = 0; k < 2; ++k)
    if (g->poll_ev[k]) cudaEventDestroy(g->poll_ev[k]);
  if (g->own_stream) cudaStreamDestroy(g->own_stream);
  if (g->comm) ncclCommDestroy(g->comm);
  for (auto& kv : g->tiles) cudaFree(kv.second.first);
  shm_close_seg(g->shm);
  delete g;
}

// Device buffers, streams and the slabs' planes (zeroed; not loaded).
int build(sor_grid* g, const std::vector<std::pair<int64_t, int64_t>>& spans, int nplanes) {
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
  CU(cudaMalloc(&g->gbar, sizeof(unsigned int)));
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
    const size_t bytes = (size_t)s.nstore * g->pitch * g->esz;
    for (int p = 0; p < nplanes; ++p) {
      cudaError_t e = cudaMalloc(&s.plane[p], bytes);
      if (e != cudaSuccess) {
        cudaGetLastError();
        g->slabs.push_back(s);
        return set_error(nullptr, SOR_E_NOMEM, "cudaMalloc of %.3f GB plane failed: %s", (double)bytes / 1e9,
                         cudaGetErrorString(e));
      }
      CU(cudaMemsetAsync(s.plane[p], 0, bytes, g->stream));
    }
    g->slabs.push_back(s);
    for (int p = 0; p < nplanes; ++p) TRY(make_tmaps(g, g->slabs.back(), p));
  }
  g->nplanes = nplanes;
  // halo flags: per slab a top and a bottom array of nflags (one per strip of
  // any layout); dist-IPC puts them behind this rank's DistComm header
  g->nflags = (int)(g->cols / 64 + 8);
  if (g->push) {
    const size_t fl = (size_t)2 * g->nflags * sizeof(unsigned long long);
    const size_t hdr = g->mode == Mode::Dist ? sizeof(DistComm) : 0;
    const size_t bytes = hdr + fl * g->slabs.size();
    CU(cudaMalloc(&g->flagbuf, bytes));
    CU(cudaMemsetAsync(g->flagbuf, 0, bytes, g->stream));
    for (size_t k = 0; k < g->slabs.size(); ++k) {
      auto* f = reinterpret_cast<unsigned long long*>((char*)g->flagbuf + hdr + fl * k);
      g->slabs[k].ftop = f;
      g->slabs[k].fbot = f + g->nflags;
    }
    g->H = 2 * kMaxTLink;
  }
  if (g->mode == Mode::Virtual) {  // neighbours are the adjacent slabs
    const int n = (int)g->slabs.size();
    for (int k = 0; k < n; ++k) {
      for (int d = 0; d < 2; ++d) {
        const int q = d == 0 ? k - 1 : k + 1;
        if (q < 0 || q >= n) continue;
        Neighbour& nb = d == 0 ? g->slabs[k].up : g->slabs[k].dn;
        nb.ok = true;
        for (int p = 0; p < 3; ++p) nb.plane[p] = g->slabs[q].plane[p];
        nb.ftop = g->slabs[q].ftop;
        nb.fbot = g->slabs[q].fbot;
        nb.g0 = g->slabs[q].g0;
      }
    }
  }
  CU(cudaStreamSynchronize(g->stream));
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

// ---- dist over NCCL: rank 0 scatters the init (fp64 rows) to every rank
int scatter_nccl(sor_grid* g, const double* init) {
  const int64_t w = g->cols + 2;
  const Slab& me = g->slabs[0];
  int32_t* dstat = reinterpret_cast<int32_t*>(g->dflag);
  // rank 0's verdict on the init first, so a bad init fails every rank
  if (g->rank == 0) {
    const bool on_dev = is_device_ptr(init);
    const int rc = check_finite(g, init, (g->rows + 2) * w, on_dev);
    const int32_t st = rc < 0 ? 1 : 0;
    CU(cudaMemcpyAsync(dstat, &st, sizeof st, cudaMemcpyHostToDevice, g->stream));
  }
  NC(ncclBroadcast(dstat, dstat, 1, ncclInt32, 0, g->comm, g->stream));
  int32_t st = 0;
  CU(cudaMemcpyAsync(&st, dstat, sizeof st, cudaMemcpyDeviceToHost, g->stream));
  CU(cudaStreamSynchronize(g->stream));
  if (st) return set_error(nullptr, SOR_E_INVAL, "init (rank 0) contains non-finite values");
  if (g->rank == 0) TRY(load_slab(g, me, init));
  // a staging buffer of whole rows for the transfers
  const int64_t chunk = std::max<int64_t>(1, (int64_t)((64 << 20) / (w * 8)));
  double* xbuf = nullptr;
  CU(cudaMalloc(&xbuf, (size_t)chunk * w * 8));
  int rc = SOR_OK;
  for (int p = 1; p < g->nranks && rc == SOR_OK; ++p) {
    int64_t lo, hi;
    partition(g->rows, g->nranks, p, &lo, &hi);
    const int64_t ga = std::max<int64_t>(0, lo - kRowPad), gb = std::min<int64_t>(g->rows + 2, hi + kRowPad);
    if (g->rank != 0 && g->rank != p) continue;
    for (int64_t r = ga; r < gb && rc == SOR_OK; r += chunk) {
      const int64_t n = std::min(chunk, gb - r);
      ncclResult_t nr;
      if (g->rank == 0) {
        if (cudaMemcpyAsync(xbuf, init + r * w, n * w * 8, kDefault, g->stream) != cudaSuccess) {
          rc = set_error(g, SOR_E_CUDA, "scatter: copy failed");
          break;
        }
        nr = ncclSend(xbuf, n * w, ncclFloat64, p, g->comm, g->stream);
      } else {
        nr = ncclRecv(xbuf, n * w, ncclFloat64, 0, g->comm, g->stream);
      }
      if (nr != ncclSuccess) {
        rc = set_error(g, SOR_E_NCCL, "scatter: %s", ncclGetErrorString(nr));
        break;
      }
      if (g->rank == p) {
        if (r == ga) {
          if (cudaMemsetAsync(me.plane[0], 0, (size_t)me.nstore * g->pitch * g->esz, g->stream) != cudaSuccess) {
            rc = set_error(g, SOR_E_CUDA, "scatter: memset failed");
            break;
          }
        }
        rc = load_rows(g, me, 0, xbuf - r * w, r, r + n);
      }
      if (cudaStreamSynchronize(g->stream) != cudaSuccess) rc = set_error(g, SOR_E_CUDA, "scatter: sync failed");
    }
  }
  cudaFree(xbuf);
  TRY(rc);
  if (g->rank != 0) {
    const size_t bytes = (size_t)me.nstore * g->pitch * g->esz;
    for (int p = 1; p < 3; ++p)
      if (me.plane[p]) CU(cudaMemcpyAsync(me.plane[p], me.plane[0], bytes, cudaMemcpyDeviceToDevice, g->stream));
  }
  reset_plane_info(g);
  CU(cudaStreamSynchronize(g->stream));
  return SOR_OK;
}

// ---- dist over CUDA IPC: publish, map, scatter
int ipc_open(sor_grid* g, const cudaIpcMemHandle_t& h, void** out) {
  CU(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  g->ipc_opened.push_back(*out);
  return SOR_OK;
}

int ipc_connect(sor_grid* g, const char* id) {
  TRY(shm_open_seg(g, id, g->rank, g->nranks));
  ShmHdr* H = g->shm->h;
  Slab& s = g->slabs[0];
  RankInfo& me = H->rank[g->rank];
  for (int p = 0; p < 3; ++p) CU(cudaIpcGetMemHandle(&me.plane[p], s.plane[p]));
  CU(cudaIpcGetMemHandle(&me.comm, g->flagbuf));
  me.g_lo = s.g_lo;
  me.g_hi = s.g_hi;
  me.g0 = s.g0;
  me.nstore = s.nstore;
  me.nplanes = 3;
  CU(cudaDeviceGetPCIBusId(me.bus_id, sizeof me.bus_id, g->device));
  me.ok = 1;
  TRY(shm_barrier(g));
  // ranks sharing a GPU run in lockstep: kernels of different processes on
  // one device are time-sliced, never co-resident, so none may wait on another
  bool share = getenv("SOR_DIST_LOCKSTEP") != nullptr;
  for (int q = 0; q < g->nranks; ++q)
    for (int r = q + 1; r < g->nranks; ++r)
      if (strncmp(H->rank[q].bus_id, H->rank[r].bus_id, sizeof me.bus_id) == 0) share = true;
  g->lockstep = share;
  DistJoinTab tab{};
  tab.nranks = g->nranks;
  tab.rank = g->rank;
  const size_t fl_off = sizeof(DistComm);
  if (g->rank == 0) g->rslabs.resize(g->nranks);
  for (int q = 0; q < g->nranks; ++q) {
    const RankInfo& ri = H->rank[q];
    void* comm = nullptr;
    void* pl[3] = {nullptr, nullptr, nullptr};
    if (q == g->rank) {
      comm = g->flagbuf;
      for (int p = 0; p < 3; ++p) pl[p] = s.plane[p];
    } else {
      TRY(ipc_open(g, ri.comm, &comm));
      if (q == g->rank - 1 || q == g->rank + 1 || g->rank == 0)
        for (int p = 0; p < 3; ++p) TRY(ipc_open(g, ri.plane[p], &pl[p]));
    }
    tab.comm[q] = reinterpret_cast<DistComm*>(comm);
    auto* f = reinterpret_cast<unsigned long long*>((char*)comm + fl_off);
    if (q == g->rank - 1 || q == g->rank + 1) {
      Neighbour& nb = q < g->rank ? s.up : s.dn;
      nb.ok = true;
      for (int p = 0; p < 3; ++p) nb.plane[p] = pl[p];
      nb.ftop = f;
      nb.fbot = f + g->nflags;
      nb.g0 = ri.g0;
    }
    if (g->rank == 0) {
      Slab& rs = g->rslabs[q];
      rs.g_lo = ri.g_lo;
      rs.g_hi = ri.g_hi;
      rs.g0 = ri.g0;
      rs.nstore = ri.nstore;
      for (int p = 0; p < 3; ++p) rs.plane[p] = pl[p];
    }
  }
  CU(cudaMalloc(&g->djoin, sizeof(DistJoinTab)));
  CU(cudaMemcpyAsync(g->djoin, &tab, sizeof tab, cudaMemcpyHostToDevice, g->stream));
  CU(cudaStreamSynchronize(g->stream));
  TRY(shm_barrier(g));
  // every rank has mapped the segment: drop its name now, so the id can
  // rendezvous the next handle at once (the mapping stays valid)
  if (g->shm->owner) {
    shm_unlink(g->shm->name.c_str());
    g->shm->owner = false;
  }
  return SOR_OK;
}

// Rank 0 writes every rank's planes through the IPC mappings; the barrier
// after it publishes them.  A bad init fails every rank (shared status).
int scatter_ipc(sor_grid* g, const double* init) {
  ShmHdr* H = g->shm->h;
  if (g->rank == 0) {
    const bool on_dev = is_device_ptr(init);
    int rc = check_finite(g, init, (g->rows + 2) * (g->cols + 2), on_dev);
    if (rc == SOR_OK) {
      for (int q = 0; q < g->nranks && rc == SOR_OK; ++q) rc = load_slab(g, g->rslabs[q], init);
      if (rc == SOR_OK && cudaStreamSynchronize(g->stream) != cudaSuccess)
        rc = set_error(g, SOR_E_CUDA, "scatter: sync failed");
    }
    H->status.store(rc, std::memory_order_release);
    TRY(shm_barrier(g));
    TRY(rc);
  } else {
    TRY(shm_barrier(g));
    const int rc = H->status.load(std::memory_order_acquire);
    if (rc < 0) return set_error(nullptr, rc, "init rejected on rank 0: %s", rc == SOR_E_INVAL ? "non-finite values" : "error");
  }
  reset_plane_info(g);
  TRY(shm_barrier(g));  // status read by all before it can change again
  return SOR_OK;
}

// (Re)load a handle from `init` (dist: collective; rank 0's init).
int load_grid(sor_grid* g, const double* init) {
  if (g->mode != Mode::Dist) {
    if (!init) return set_error(nullptr, SOR_E_INVAL, "init is NULL");
    const bool on_dev = is_device_ptr(init);
    TRY(check_finite(g, init, (g->rows + 2) * (g->cols + 2), on_dev));
    return load_all(g, init);
  }
  if (g->rank == 0 && !init) return set_error(nullptr, SOR_E_INVAL, "init is NULL on rank 0");
  if (g->transport == Transport::Ipc) return scatter_ipc(g, init);
  return scatter_nccl(g, init);
}

int create_common(sor_grid** out, int64_t rows, int64_t cols, const double* init, sor_dtype dt, Mode mode,
                  int nslabs, int rank, int nranks, int device, const void* id, Transport tr) {
  if (!out) return set_error(nullptr, SOR_E_INVAL, "out is NULL");
  *out = nullptr;
  if (!init && (mode != Mode::Dist || rank == 0)) return set_error(nullptr, SOR_E_INVAL, "init is NULL");
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
    if (tr == Transport::Ipc && nranks > kMaxRanks)
      return set_error(nullptr, SOR_E_INVAL, "dist-ipc: at most %d ranks (one node)", kMaxRanks);
    if (!id) return set_error(nullptr, SOR_E_INVAL, "dist: id is NULL");
    int64_t lo, hi;
    partition(rows, nranks, rank, &lo, &hi);
    spans.push_back({lo, hi});
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    return set_error(nullptr, SOR_E_CUDA, "no CUDA device available (%s); libsor has no CPU fallback",
                     cudaGetErrorString(e));
  }
  if (mode == Mode::Dist) {
    e = cudaSetDevice(device);
    if (e != cudaSuccess) return set_error(nullptr, SOR_E_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  }
  sor_grid* g = new sor_grid();
  g->rows = rows;
  g->cols = cols;
  g->dt = dt;
  g->mode = mode;
  g->rank = mode == Mode::Dist ? rank : 0;
  g->nranks = mode == Mode::Dist ? nranks : 1;
  g->transport = mode == Mode::Dist ? tr : Transport::None;
  g->push = (mode == Mode::Virtual && !getenv("SOR_VIRTUAL_COPY")) || g->transport == Transport::Ipc;
  int rc = SOR_OK;
  if (g->transport == Transport::Nccl) {
    ncclUniqueId nid;
    memcpy(&nid, id, sizeof nid);
    ncclResult_t r = ncclCommInitRank(&g->comm, nranks, nid, rank);
    if (r != ncclSuccess) rc = set_error(nullptr, SOR_E_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  if (rc == SOR_OK) rc = build(g, spans, g->transport == Transport::Ipc ? 3 : 2);
  if (rc == SOR_OK && g->transport == Transport::Ipc) rc = ipc_connect(g, reinterpret_cast<const char*>(id));
  if (rc == SOR_OK) rc = load_grid(g, init);
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
// Host-side halo exchange (virtual copies, NCCL send/recv, or IPC copies in
// lockstep): after a pass wrote plane p, each slab sends its first/last h
// owned rows to the neighbouring slabs' halo rows of the same plane.  The
// push modes (virtual, dist-IPC) use it only when a pass needs more halo
// rows than the last push delivered (K1 passes, a deeper T after set_kernel).
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
    g->pinfo[p].wseq = 0;
    return SOR_OK;
  }
  if (g->mode != Mode::Dist || g->nranks == 1) return SOR_OK;
  Slab& s = g->slabs[0];
  char* pl = (char*)s.plane[p];
  if (g->transport == Transport::Ipc) {
    // every rank's pass is complete before, and every copy after (barriers)
    CU(cudaStreamSynchronize(g->stream));
    TRY(shm_barrier(g));
    if (s.up.ok)
      CU(cudaMemcpyAsync((char*)s.up.plane[p] + (s.g_lo - s.up.g0) * row_bytes, pl + (s.g_lo - s.g0) * row_bytes,
                         h * row_bytes, cudaMemcpyDeviceToDevice, g->stream));
    if (s.dn.ok)
      CU(cudaMemcpyAsync((char*)s.dn.plane[p] + (s.g_hi - h - s.dn.g0) * row_bytes,
                         pl + (s.g_hi - h - s.g0) * row_bytes, h * row_bytes, cudaMemcpyDeviceToDevice, g->stream));
    CU(cudaStreamSynchronize(g->stream));
    TRY(shm_barrier(g));
    g->st.halo_exchanges += 1;
    g->pinfo[p].wseq = 0;
    return SOR_OK;
  }
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
  g->pinfo[p].wseq = 0;
  return SOR_OK;
}

// Cross-rank join mode of the maxima (IterCtl::join_mode).
int join_mode_of(const sor_grid* g) {
  if (g->transport != Transport::Ipc || g->nranks == 1) return 0;
  return g->lockstep ? 2 : 1;
}

// Join the per-slab maxima and run the stop test (multi-slab modes).
int join_and_finalize(sor_grid* g, const IterCtl& ctl) {
  if (g->transport == Transport::Nccl && g->nranks > 1)
    NC(ncclAllReduce(&g->dstate->maxbits[0][0], &g->dstate->maxbits[0][0], 2 * kMaxT * 16, ncclUint64, ncclMax,
                     g->comm, g->stream));
  IterCtl c = ctl;
  c.join = g->djoin;
  c.join_mode = join_mode_of(g);
  finalize_kernel<<<1, 32, 0, g->stream>>>(c);
  CU(cudaGetLastError());
  g->st.kernel_launches += 1;
  if (c.join_mode == 2) {  // lockstep: everyone published before anyone combines
    CU(cudaStreamSynchronize(g->stream));
    TRY(shm_barrier(g));
    c.join_mode = 3;
    finalize_kernel<<<1, 32, 0, g->stream>>>(c);
    CU(cudaGetLastError());
    g->st.kernel_launches += 1;
    CU(cudaStreamSynchronize(g->stream));
    TRY(shm_barrier(g));  // the published slots are read before the next pass can overwrite them
  }
  return SOR_OK;
}

// Device-initiated halo exchange: the link of slab s for a pass src -> dst.
HaloLink make_link(sor_grid* g, const Slab& s, int src, int dst) {
  HaloLink L{};
  if (!g->push) return L;
  L.on = 1;
  L.H = g->H;
  L.seq = g->seq;
  const PlaneInfo& pi = g->pinfo[src];
  L.need = pi.wseq;
  L.pg = pi.pg;
  L.pw = pi.pw;
  L.pgh = pi.pgh;
  L.pn = pi.pn;
  auto off = [&](const Neighbour& nb) -> long long {
    return (long long)(((intptr_t)nb.plane[dst] - (intptr_t)s.plane[dst]) / (intptr_t)g->esz) +
           (long long)(s.g0 - nb.g0) * g->pitch;
  };
  if (s.up.ok) {
    L.up_off = off(s.up);
    L.rel_up = s.up.fbot;
    L.acq_top = s.ftop;
  }
  if (s.dn.ok) {
    L.dn_off = off(s.dn);
    L.rel_dn = s.dn.ftop;
    L.acq_bot = s.fbot;
  }
  return L;
}

int strips_of(const sor_grid* g, int s0, int wc, int ghost) {
  const int64_t wout = wc - 2 * ghost;
  return (int)((g->cols + 1 - (s0 + ghost) + wout - 1) / wout);
}

void record_layout(sor_grid* g, int dst, int s0, int wc, int ghost, int nstrips) {
  PlaneInfo& pi = g->pinfo[dst];
  pi.pg = s0 + ghost;
  pi.pw = wc - 2 * ghost;
  pi.pgh = ghost;
  pi.pn = nstrips;
}

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
               int s0, std::pair<int4*, int>* out, int reserve) {
  const auto key =
      std::make_tuple(slab_idx, ((ghost * 16 + S) * 2 + (split ? 1 : 0)) * 1024 + wc, tiles_per_sm * 64 + reserve);
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
  const int64_t slots = (int64_t)g->nsm * tiles_per_sm - reserve;
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
  if (g->push) {
    // one pushing tile per strip and side (HaloLink): the first band of each
    // strip holds the slab's first H rows, the last band its last H rows
    const int64_t need = std::min<int64_t>(g->H, s.g_hi - s.g_lo);
    std::map<int, std::vector<int4>> by;
    for (const int4& x : tl) by[x.x].push_back(x);
    tl.clear();
    for (auto& kv : by) {
      auto& v = kv.second;
      std::sort(v.begin(), v.end(), [](const int4& x, const int4& y) { return x.y < y.y; });
      while (v.size() > 1 && v.front().z - v.front().y < need) {
        v[1].y = v[0].y;
        v.erase(v.begin());
      }
      while (v.size() > 1 && v.back().z - v.back().y < need) {
        v[v.size() - 2].z = v.back().z;
        v.pop_back();
      }
      for (auto& x : v) tl.push_back(x);
    }
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

// Programmatic dependent launch between consecutive wave kernels (one slab,
// or slabs that push their halos: no NCCL or copy between two launches), for
// one-wave launches only (in a multi-wave launch the next grid's early CTAs
// would hold slots its own tail needs: measured C5 -0.5%, C3 +2%).
// SOR_NO_PDL=1 disables it.
bool wave_pdl(const sor_grid* g, unsigned blocks, int occ) {
  static int off = -1;
  if (off < 0) off = getenv("SOR_NO_PDL") ? 1 : 0;
  return !off && (single_part(g) || g->push) && !g->lockstep && blocks <= (unsigned)(occ * g->nsm);
}

// Skew-2 schedule of the wave kernel (wave2.cuh) for T >= 2 on single-slab
// handles (bitwise equal; C3 T=4 iterate +3 %, C5 +3 %, T=2 +8 %:
// profiles/r2_wave2_ab.txt).  SOR_WAVE2=0 selects the skew-1 schedule.
// Pushing slabs (virtual, dist-IPC) keep the skew-1 kernel (its LINK
// instances).
bool use_wave2(const sor_grid* g, int T) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SOR_WAVE2");
    on = e ? atoi(e) : 1;
  }
  return on != 0 && T >= 2 && !g->push;
}

template <typename R, int T, int CK>
int launch_wave_L(sor_grid* g, const Slab& s, R w, const IterCtl& ctl, bool fused_fin) {
  if (T >= 2 && use_wave2(g, T)) return launch_wave2_T<R, T, CK, false>(g, s, w, ctl, fused_fin);
  return g->push ? launch_wave_T<R, T, CK, true>(g, s, w, ctl, fused_fin)
                 : launch_wave_T<R, T, CK, false>(g, s, w, ctl, fused_fin);
}

template <typename R, int CK>
int launch_wave(sor_grid* g, const Slab& s, int T, R w, const IterCtl& ctl, bool fused_fin) {
  if (CK >= 3 && T == 1) return launch_wave_L<R, 1, 2>(g, s, w, ctl, fused_fin);  // unused combination
  switch (T) {
    case 1: return launch_wave_L<R, 1, CK>(g, s, w, ctl, fused_fin);
    case 2: return launch_wave_L<R, 2, CK>(g, s, w, ctl, fused_fin);
    case 3: return launch_wave_L<R, 3, CK>(g, s, w, ctl, fused_fin);
    case 4: return launch_wave_L<R, 4, CK>(g, s, w, ctl, fused_fin);
    // T > 4: the skew-2 kernel on one slab only (sor_set_kernel enforces it)
    case 5:
      if (!use_wave2(g, 5)) return set_error(nullptr, SOR_E_UNSUPPORTED, "T = 5 needs the skew-2 kernel (SOR_WAVE2)");
      return launch_wave2_T<R, 5, CK, false>(g, s, w, ctl, fused_fin);
    case 6:
      if (!use_wave2(g, 6)) return set_error(nullptr, SOR_E_UNSUPPORTED, "T = 6 needs the skew-2 kernel (SOR_WAVE2)");
      return launch_wave2_T<R, 6, CK, false>(g, s, w, ctl, fused_fin);
  }
  return set_error(nullptr, SOR_E_INVAL, "temporal depth %d unsupported", T);
}

template <typename R, int T, int CK>
int launch_jacobi_L(sor_grid* g, const Slab& s, const IterCtl& ctl, bool fused_fin) {
  return g->push ? launch_jacobi_T<R, T, CK, true>(g, s, ctl, fused_fin)
                 : launch_jacobi_T<R, T, CK, false>(g, s, ctl, fused_fin);
}

template <typename R, int CK>
int launch_jacobi(sor_grid* g, const Slab& s, int T, const IterCtl& ctl, bool fused_fin) {
  switch (T) {
    case 1: return launch_jacobi_L<R, 1, CK>(g, s, ctl, fused_fin);
    case 2: return launch_jacobi_L<R, 2, CK>(g, s, ctl, fused_fin);
    case 3: return launch_jacobi_L<R, 3, CK>(g, s, ctl, fused_fin);
    case 4: return launch_jacobi_L<R, 4, CK>(g, s, ctl, fused_fin);
  }
  return set_error(nullptr, SOR_E_INVAL, "temporal depth %d unsupported", T);
}

// One HBM pass of ctl.T iterations ending at iteration ctl.k_last.
template <typename R>
int wave_pass(sor_grid* g, R w, IterCtl ctl) {
  const int T = ctl.T;
  const int need_rows = g->method == 1 ? T : 2 * T;  // halo rows the pass reads
  const bool fused_fin = single_part(g) && ctl.ck != 0 && !ctl.defer;
  if (!single_part(g) && g->halo_valid < need_rows) TRY(exchange(g, g->cur, 2 * T));
  g->seq += 1;
  ctl.seq = g->seq;
  ctl.join = g->djoin;
  ctl.join_mode = join_mode_of(g);
  for (size_t k = 0; k < g->slabs.size(); ++k) {
    const Slab& s = g->slabs[k];
    IterCtl c = ctl;
    if (k > 0) {  // the deferred decision runs in the first slab's launch only
      c.defer = 0;
      c.prev_valid = 0;
    }
    if (g->method == 1) {  // Jacobi: exact maxima only (ck 1 or 2)
      if (c.ck >= 2)
        TRY((launch_jacobi<R, 2>(g, s, T, c, fused_fin)));
      else if (c.ck == 1)
        TRY((launch_jacobi<R, 1>(g, s, T, c, fused_fin)));
      else
        TRY((launch_jacobi<R, 0>(g, s, T, c, fused_fin)));
      continue;
    }
    if (c.ck == 4)
      TRY((launch_wave<R, 4>(g, s, T, w, c, fused_fin)));
    else if (c.ck == 3)
      TRY((launch_wave<R, 3>(g, s, T, w, c, fused_fin)));
    else if (c.ck == 2)
      TRY((launch_wave<R, 2>(g, s, T, w, c, fused_fin)));
    else if (c.ck == 1)
      TRY((launch_wave<R, 1>(g, s, T, w, c, fused_fin)));
    else
      TRY((launch_wave<R, 0>(g, s, T, w, c, fused_fin)));
  }
  const int src = g->cur;
  const PlaneInfo spi = g->pinfo[src];
  g->cur = g->nxt(src);
  g->st.half_sweeps += g->method == 1 ? T : 2 * T;  // Jacobi: one sweep per iteration
  g->st.hbm_passes += 1;
  if (g->push) {
    // the pass pushed its first/last H rows into the neighbours' halos
    g->pinfo[g->cur].wseq = g->seq;
    g->halo_valid = g->H;
    g->st.halo_exchanges += single_part(g) ? 0 : 1;
  } else {
    TRY(exchange(g, g->cur, 2 * T));
    g->halo_valid = 2 * T;
  }
  if (g->lockstep) {  // ranks sharing a GPU: the pass is complete everywhere before the next one
    CU(cudaStreamSynchronize(g->stream));
    TRY(shm_barrier(g));
  }
  if (ctl.ck && !fused_fin && !ctl.defer) TRY(join_and_finalize(g, ctl));
  g->pass_ends.push_back({ctl.k_last, src, g->cur, T, spi, g->pinfo[g->cur]});
  return SOR_OK;
}

// ------------------------------------------------------------------ K5
template <typename R>
int k5_run(sor_grid* g, R w, int solve, int64_t n_iter, double tol, int64_t K, int measure_last) {
  // register-resident single CTA (K7 form) when the grid fits its window;
  // SOR_K5_SMEM=1 keeps the shared-memory kernel
  static int smem_only = -1;
  if (smem_only < 0) smem_only = getenv("SOR_K5_SMEM") ? 1 : 0;
  if (!smem_only) {
    const int rc = launch_resident_single<R>(g, w, solve, n_iter, tol, K, measure_last);
    if (rc != SOR_E_UNSUPPORTED) return rc;
  }
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
  // dist-IPC: every rank finished its previous call before anyone pushes
  // into a neighbour's planes again
  TRY(dist_barrier(g));
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
  if (g->hstate[0].halo_timeout)
    return set_error(g, SOR_E_CUDA, "halo/join wait timed out (a peer rank never released its rows)");
  if (out) *out = g->hstate[0];
  return SOR_OK;
}

int depth_of(const sor_grid* g) {
  return (g->kernel == SOR_KERNEL_TEMPORAL || g->kernel == SOR_KERNEL_RESIDENT) ? g->tdepth : 1;
}

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

// K6 eligibility: one slab, SOR, both planes L2-resident (the persistent
// kernel's passes re-read what the previous pass wrote; beyond L2 a pass is
// HBM-bound and the per-launch overhead is already amortised).
// SOR_NO_PERSIST=1 disables it.
bool use_persist(const sor_grid* g) {
  static int off = -1;
  if (off < 0) off = getenv("SOR_NO_PERSIST") ? 1 : 0;
  if (off || g->persist_off || !single_part(g) || g->method != 0 || !g->gbar) return false;
  const Slab& s = g->slabs[0];
  const double planes = 2.0 * (double)s.nstore * (double)g->pitch * (double)g->esz;
  return planes <= 48.0 * (1 << 20);
}

// K7 (SOR_KERNEL_RESIDENT, one slab, SOR): register-resident grid, multi-CTA
// (iterate) or one CTA (iterate and solve) when it fits (resident.cuh).
bool use_resident(const sor_grid* g, bool single) {
  if (g->kernel != SOR_KERNEL_RESIDENT || !single_part(g) || g->method != 0) return false;
  return resident_fits(g, single ? 1 : g->tdepth, single);
}

template <typename R>
int persist_passes(sor_grid* g, R w, int T, int npasses) {
  const Slab& s = g->slabs[0];
  int rc = SOR_E_INVAL;
  switch (T) {
    case 1: rc = launch_wave_persist<R, 1>(g, s, w, npasses, g->gbar); break;
    case 2: rc = launch_wave_persist<R, 2>(g, s, w, npasses, g->gbar); break;
    case 3: rc = launch_wave_persist<R, 3>(g, s, w, npasses, g->gbar); break;
    case 4: rc = launch_wave_persist<R, 4>(g, s, w, npasses, g->gbar); break;
  }
  if (rc != SOR_OK) return rc;
  // the kernel alternates between the current plane and the next one (also
  // when a third plane exists for the deferred stop test)
  if (npasses & 1) g->cur = g->nxt(g->cur);
  g->st.half_sweeps += (int64_t)2 * T * npasses;
  g->st.hbm_passes += npasses;
  g->seq += npasses;
  return SOR_OK;
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
  if (!base.solve && k_from == 1 && use_resident(g, false)) {
    // K7: the whole iterate call in one launch
    const int rc = launch_resident_iterate<R>(g, w, k_to, T, check_last);
    if (rc != SOR_E_UNSUPPORTED) return rc;
  }
  if (!base.solve && k_from == 1 && use_resident(g, true)) {
    const int rc = launch_resident_single<R>(g, w, 0, k_to, 1.0, 1, check_last ? 1 : 0);
    if (rc == SOR_OK) {
      g->st.half_sweeps += 2 * k_to;
      if (check_last) g->st.checks += 1;
    }
    if (rc != SOR_E_UNSUPPORTED) return rc;
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
      if (t == T && !base.solve) {
        // K6: the full passes of an iterate block as one persistent launch
        // (all but a measured last pass)
        const int64_t full = left / T - ((check_last && end == k_to) ? 1 : 0);
        if (full >= 2 && T <= kMaxTLink && use_persist(g)) {
          const int rc = persist_passes<R>(g, w, T, (int)std::min<int64_t>(full, 1 << 20));
          if (rc == SOR_OK) {
            k += std::min<int64_t>(full, 1 << 20) * T;
            continue;
          }
          if (rc != SOR_E_UNSUPPORTED) return rc;
          g->persist_off = true;  // tiles do not fit in one wave: pass by pass from now on
        }
      }
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
        c.prev_seq = g->prev_seq;
        g->prev_valid = false;
        c.set = g->next_set;
        if (c.ck) {
          g->prev_valid = true;
          g->prev_k_last = c.k_last;
          g->prev_T = c.T;
          g->prev_ck = c.ck;
          g->prev_set = c.set;
          g->prev_seq = g->seq + 1;  // the sequence number wave_pass gives this pass
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
  if (g->hstate[0].halo_timeout)
    return set_error(g, SOR_E_CUDA, "halo/join wait timed out (a peer rank never released its rows)");
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
  // dist-IPC: the neighbours' speculative passes that read the planes this
  // re-run pushes into are complete (their streams drained, barrier)
  TRY(dist_barrier(g));
  CU(cudaMemsetAsync(g->dstate, 0, sizeof(DevState), g->stream));
  g->cur = pr.src;  // writes the pass's own destination plane again
  g->pinfo[pr.src] = pr.spi;  // passes after it exited early but were booked
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

// Third plane for the deferred stop test: allocated once, a copy of the
// current plane (ring, padding); false if memory is short or the handle's
// ranks cannot defer (NCCL transport: host-side exchanges between passes;
// lockstep IPC ranks: the decision needs a host barrier).  Dist-IPC handles
// allocate it at creation (the neighbours map it).
bool ensure_third_plane(sor_grid* g) {
  static int off = -1;
  if (off < 0) off = getenv("SOR_NO_DEFER") ? 1 : 0;
  if (off || g->lockstep || g->transport == Transport::Nccl) return false;
  if (g->nplanes == 3) return true;
  if (!single_part(g) && !g->push) return false;
  bool ok = true;
  for (auto& s : g->slabs) {
    const size_t bytes = (size_t)s.nstore * g->pitch * g->esz;
    if (cudaMalloc(&s.plane[2], bytes) != cudaSuccess) {
      cudaGetLastError();
      s.plane[2] = nullptr;
      ok = false;
      break;
    }
    if (cudaMemcpyAsync(s.plane[2], s.plane[g->cur], bytes, cudaMemcpyDeviceToDevice, g->stream) != cudaSuccess ||
        make_tmaps(g, s, 2) != SOR_OK) {
      ok = false;
      break;
    }
  }
  if (!ok) {
    cudaStreamSynchronize(g->stream);
    for (auto& s : g->slabs)
      if (s.plane[2]) {
        cudaFree(s.plane[2]);
        s.plane[2] = nullptr;
      }
    return false;
  }
  const int n = (int)g->slabs.size();
  for (int k = 0; k < n; ++k) {
    if (k > 0) g->slabs[k].up.plane[2] = g->slabs[k - 1].plane[2];
    if (k + 1 < n) g->slabs[k].dn.plane[2] = g->slabs[k + 1].plane[2];
  }
  g->pinfo[2] = g->pinfo[g->cur];
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
  if (g->kernel == SOR_KERNEL_SMALL || use_resident(g, true)) {
    if (g->kernel == SOR_KERNEL_SMALL)
      TRY(k5_run<R>(g, w, 1, maxit, tol, K, 0));
    else
      TRY(launch_resident_single<R>(g, w, 1, maxit, tol, K, 0));
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
        if (g->transport == Transport::Nccl) {
          // NCCL ranks must enqueue the same collectives: decide on this
          // batch's state (identical on every rank after the allreduce)
          CU(cudaEventSynchronize(g->poll_ev[b & 1]));
          if (g->hstate[b & 1].stop) break;
        } else if (b >= 1) {
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
        c.seq = g->prev_seq;
        c.join = g->djoin;
        c.join_mode = join_mode_of(g);
        c.defer = 0;
        finalize_kernel<<<1, 32, 0, g->stream>>>(c);
        CU(cudaGetLastError());
        g->st.kernel_launches += 1;
        g->prev_valid = false;
      }
      TRY(read_state(g, &hs));
      // dist-IPC: ranks may have enqueued different numbers of (early-exit)
      // passes after the stop; agree on the sequence counter again
      TRY(sync_seq(g));
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
        g->pinfo[pr.dst] = pr.dpi;
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

// ---- gather (download) of global rows [ra, rb) into out (row ra at out)
int gather_rows(sor_grid* g, int64_t ra, int64_t rb, double* out) {
  const int64_t w = g->cols + 2;
  double* base = out ? out - ra * w : nullptr;  // store_rows indexes by global row
  auto span_of = [&](int q, int nq, int64_t lo, int64_t hi, int64_t* a, int64_t* b) {
    *a = std::max(ra, q == 0 ? (int64_t)0 : lo);
    *b = std::min(rb, q == nq - 1 ? g->rows + 2 : hi);
  };
  if (g->mode != Mode::Dist) {
    CU(cudaStreamSynchronize(g->stream));
    const int n = (int)g->slabs.size();
    for (int k = 0; k < n; ++k) {
      const Slab& s = g->slabs[k];
      int64_t sa, sb;
      span_of(k, n, s.g_lo, s.g_hi, &sa, &sb);
      if (sa < sb) TRY(store_rows(g, s, g->cur, base, sa, sb));
    }
    CU(cudaStreamSynchronize(g->stream));
    return SOR_OK;
  }
  if (g->transport == Transport::Ipc) {  // rank 0 reads every rank's plane
    CU(cudaStreamSynchronize(g->stream));
    TRY(shm_barrier(g));
    int rc = SOR_OK;
    if (g->rank == 0) {
      for (int q = 0; q < g->nranks && rc == SOR_OK; ++q) {
        const Slab& s = g->rslabs[q];
        int64_t sa, sb;
        span_of(q, g->nranks, s.g_lo, s.g_hi, &sa, &sb);
        if (sa < sb) rc = store_rows(g, s, g->cur, base, sa, sb);
      }
      if (rc == SOR_OK && cudaStreamSynchronize(g->stream) != cudaSuccess)
        rc = set_error(g, SOR_E_CUDA, "gather: sync failed");
    }
    TRY(shm_barrier(g));  // nobody changes its planes before rank 0 has read them
    return rc;
  }
  // NCCL: every rank sends its part to rank 0 (whole storage rows)
  const size_t row_bytes = (size_t)g->pitch * g->esz;
  const Slab& me = g->slabs[0];
  CU(cudaStreamSynchronize(g->stream));
  if (g->rank != 0) {
    int64_t sa, sb;
    span_of(g->rank, g->nranks, me.g_lo, me.g_hi, &sa, &sb);
    if (sa < sb)
      NC(ncclSend((char*)me.plane[g->cur] + (sa - me.g0) * row_bytes, (sb - sa) * row_bytes, ncclUint8, 0, g->comm,
                  g->stream));
    CU(cudaStreamSynchronize(g->stream));
    return SOR_OK;
  }
  int64_t sa, sb;
  span_of(0, g->nranks, me.g_lo, me.g_hi, &sa, &sb);
  if (sa < sb) TRY(store_rows(g, me, g->cur, base, sa, sb));
  int64_t maxr = 0;
  for (int p = 1; p < g->nranks; ++p) {
    int64_t lo, hi, a, b;
    partition(g->rows, g->nranks, p, &lo, &hi);
    span_of(p, g->nranks, lo, hi, &a, &b);
    maxr = std::max(maxr, b - a);
  }
  void* tmp = nullptr;
  if (maxr > 0) CU(cudaMalloc(&tmp, (size_t)maxr * row_bytes));
  int rc = SOR_OK;
  for (int p = 1; p < g->nranks && rc == SOR_OK; ++p) {
    int64_t lo, hi, a, b;
    partition(g->rows, g->nranks, p, &lo, &hi);
    span_of(p, g->nranks, lo, hi, &a, &b);
    if (a >= b) continue;
    const ncclResult_t r = ncclRecv(tmp, (b - a) * row_bytes, ncclUint8, p, g->comm, g->stream);
    if (r != ncclSuccess) {
      rc = set_error(g, SOR_E_NCCL, "gather: %s", ncclGetErrorString(r));
      break;
    }
    Slab t;  // the received rows as a slab whose storage row 0 is global row a
    t.g0 = a;
    t.nstore = b - a;
    t.plane[0] = tmp;
    rc = store_rows(g, t, 0, base, a, b);
    if (rc == SOR_OK && cudaStreamSynchronize(g->stream) != cudaSuccess)
      rc = set_error(g, SOR_E_CUDA, "gather: sync failed");
  }
  cudaStreamSynchronize(g->stream);
  if (tmp) cudaFree(tmp);
  return rc;
}

// Every ABI call on a handle runs on the handle's device and restores the
// caller's current device afterwards.
struct DevGuard {
  int prev = -1;
  bool changed = false;
  explicit DevGuard(const sor_grid* g) {
    if (g && cudaGetDevice(&prev) == cudaSuccess && prev != g->device)
      changed = cudaSetDevice(g->device) == cudaSuccess;
  }
  ~DevGuard() {
    if (changed) cudaSetDevice(prev);
  }
};

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
  return create_common(out, N, N, init, dt, Mode::Single, 1, 0, 1, 0, nullptr, Transport::None);
}

int sor_create_rect(sor_grid** out, int64_t rows, int64_t cols, const double* init, sor_dtype dt) {
  return create_common(out, rows, cols, init, dt, Mode::Single, 1, 0, 1, 0, nullptr, Transport::None);
}

int sor_create_virtual(sor_grid** out, int64_t rows, int64_t cols, const double* init, sor_dtype dt,
                       int nslabs) {
  return create_common(out, rows, cols, init, dt, Mode::Virtual, nslabs, 0, 1, 0, nullptr, Transport::None);
}

int sor_create_dist(sor_grid** out, int64_t rows, int64_t cols, const double* init, sor_dtype dt,
                    int rank, int nranks, int device, const void* nccl_id) {
  return create_common(out, rows, cols, init, dt, Mode::Dist, 1, rank, nranks, device, nccl_id, Transport::Nccl);
}

int sor_create_dist_ipc(sor_grid** out, int64_t rows, int64_t cols, const double* init, sor_dtype dt,
                        int rank, int nranks, int device, const void* ipc_id) {
  return create_common(out, rows, cols, init, dt, Mode::Dist, 1, rank, nranks, device, ipc_id, Transport::Ipc);
}

int sor_nccl_unique_id(void* out128) {
  if (!out128) return set_error(nullptr, SOR_E_INVAL, "NULL output");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return set_error(nullptr, SOR_E_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  memcpy(out128, &id, sizeof id);
  return SOR_OK;
}

int sor_ipc_unique_id(void* out128) {
  if (!out128) return set_error(nullptr, SOR_E_INVAL, "NULL output");
  std::random_device rd;
  const unsigned long long r = ((unsigned long long)rd() << 32) ^ rd() ^
                               (unsigned long long)std::chrono::steady_clock::now().time_since_epoch().count();
  char buf[128];
  memset(buf, 0, sizeof buf);
  snprintf(buf, sizeof buf, "/sorb-%d-%016llx", (int)getpid(), r);
  memcpy(out128, buf, sizeof buf);
  return SOR_OK;
}

int sor_set_kernel(sor_grid* g, int kernel, int temporal_depth) {
  TRY(usable(g));
  switch (kernel) {
    case SOR_KERNEL_NATURAL:
      if (g->transport == Transport::Ipc)
        return set_error(nullptr, SOR_E_UNSUPPORTED, "SOR_KERNEL_NATURAL is not available on dist-IPC handles");
      g->kernel = kernel;
      g->tdepth = 1;
      break;
    case SOR_KERNEL_FUSED:
      g->kernel = kernel;
      g->tdepth = 1;
      break;
    case SOR_KERNEL_TEMPORAL:
    case SOR_KERNEL_RESIDENT: {
      if (temporal_depth < 1 || temporal_depth > kMaxT)
        return set_error(nullptr, SOR_E_INVAL, "temporal_depth must be in [1,%d], got %d", kMaxT, temporal_depth);
      // the thinnest slab of any rank (sizes differ by at most one row)
      int64_t thin = g->rows;
      for (auto& s : g->slabs) thin = std::min(thin, s.g_hi - s.g_lo);
      if (g->nranks > 1) thin = g->rows / g->nranks;
      if ((g->slabs.size() > 1 || g->nranks > 1) && thin < 2 * temporal_depth)
        return set_error(nullptr, SOR_E_INVAL, "slab of %lld rows too thin for T=%d", (long long)thin,
                         temporal_depth);
      if (temporal_depth > kMaxTLink && !single_part(g))
        return set_error(nullptr, SOR_E_UNSUPPORTED, "T > %d runs on single-slab handles only", kMaxTLink);
      g->kernel = kernel;
      g->tdepth = temporal_depth;
      break;
    }
    case SOR_KERNEL_SMALL: {
      if (!single_part(g))
        return set_error(nullptr, SOR_E_UNSUPPORTED, "SOR_KERNEL_SMALL needs a single-slab grid");
      const size_t bytes = (size_t)(g->rows + 2) * (g->cols + 2) * g->esz;
      if (bytes > k5_limit_bytes())
        return set_error(nullptr, SOR_E_UNSUPPORTED, "grid of %zu bytes exceeds shared memory", bytes);
      if (g->rows * ((g->cols + 1) / 2) > (int64_t)kK5Cells * 1024)
        return set_error(nullptr, SOR_E_UNSUPPORTED, "grid has more than %d cells of one colour for K5",
                         kK5Cells * 1024);
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
  DevGuard dg(g);
  CU(cudaStreamSynchronize(g->stream));
  g->stream = cuda_stream ? (cudaStream_t)cuda_stream : g->own_stream;
  return SOR_OK;
}

int sor_iterate(sor_grid* g, double omega, int64_t iters, double* last_max_change) {
  TRY(usable(g));
  TRY(validate_omega(omega));
  if (iters < 0) return set_error(nullptr, SOR_E_INVAL, "iters must be >= 0");
  DevGuard dg(g);
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
  DevGuard dg(g);
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
  if (g->kernel != SOR_KERNEL_FUSED && g->kernel != SOR_KERNEL_TEMPORAL && g->kernel != SOR_KERNEL_RESIDENT)
    return set_error(nullptr, SOR_E_UNSUPPORTED, "Jacobi runs on the FUSED / TEMPORAL / RESIDENT kernels only");
  if (depth_of(g) > kMaxTLink)
    return set_error(nullptr, SOR_E_UNSUPPORTED, "Jacobi runs at temporal depth <= %d", kMaxTLink);
  return SOR_OK;
}
}  // namespace

int sor_jacobi_iterate(sor_grid* g, int64_t iters, double* last_max_change) {
  TRY(usable(g));
  TRY(jacobi_usable(g));
  if (iters < 0) return set_error(nullptr, SOR_E_INVAL, "iters must be >= 0");
  DevGuard dg(g);
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
  DevGuard dg(g);
  MethodGuard mg(g);
  if (g->dt == SOR_F64) return solve_impl<double>(g, 1.0, tol, maxit, check_every, iters_out, max_change_out);
  return solve_impl<float>(g, 1.0, tol, maxit, check_every, iters_out, max_change_out);
}

int sor_variant_iterate(sor_grid* g, const sor_variant* v, double omega, int64_t iters, double* last_max_change) {
  TRY(usable(g));
  TRY(validate_omega(omega));
  if (iters < 0) return set_error(nullptr, SOR_E_INVAL, "iters must be >= 0");
  TRY(variant_check(g, v));
  DevGuard dg(g);
  TRY(begin_call(g));
  double m = 0.0;
  const int rc = g->dt == SOR_F64
                     ? variant_run<double>(g, v, omega, 0, iters, 1.0, 1, last_max_change != nullptr, nullptr, &m, nullptr)
                     : variant_run<float>(g, v, omega, 0, iters, 1.0, 1, last_max_change != nullptr, nullptr, &m, nullptr);
  if (rc < 0) return rc;
  TRY(end_call(g, nullptr));
  if (last_max_change) *last_max_change = iters > 0 ? m : 0.0;
  return SOR_OK;
}

int sor_variant_solve(sor_grid* g, const sor_variant* v, double omega, double tol, int64_t maxit,
                      int64_t check_every, int64_t* iters_out, double* max_change_out) {
  TRY(usable(g));
  TRY(validate_omega(omega));
  if (!(tol > 0.0) || !std::isfinite(tol)) return set_error(nullptr, SOR_E_INVAL, "tol must be finite and > 0");
  if (maxit < 1) return set_error(nullptr, SOR_E_INVAL, "maxit must be >= 1");
  if (check_every < 1 || check_every > maxit)
    return set_error(nullptr, SOR_E_INVAL, "need 1 <= check_every <= maxit (S:114)");
  TRY(variant_check(g, v));
  DevGuard dg(g);
  TRY(begin_call(g));
  int64_t it = 0;
  double m = 0.0;
  int conv = 0;
  const int rc = g->dt == SOR_F64
                     ? variant_run<double>(g, v, omega, 1, maxit, tol, check_every, 0, &it, &m, &conv)
                     : variant_run<float>(g, v, omega, 1, maxit, tol, check_every, 0, &it, &m, &conv);
  if (rc < 0) return rc;
  TRY(end_call(g, nullptr));
  if (iters_out) *iters_out = it;
  if (max_change_out) *max_change_out = m;
  return conv ? SOR_OK : SOR_NOT_CONVERGED;
}

int sor_download(sor_grid* g, double* out) {
  TRY(usable(g));
  if ((g->mode != Mode::Dist || g->rank == 0) && !out) return set_error(nullptr, SOR_E_INVAL, "out is NULL");
  DevGuard dg(g);
  if (out && is_device_ptr(out)) CU(cudaDeviceSynchronize());  // the caller's pending reads of `out`
  return gather_rows(g, 0, g->rows + 2, g->mode == Mode::Dist && g->rank != 0 ? nullptr : out);
}

int sor_download_rows(sor_grid* g, int64_t row_a, int64_t row_b, double* out) {
  TRY(usable(g));
  if (row_a < 0 || row_b > g->rows + 2 || row_a >= row_b)
    return set_error(nullptr, SOR_E_INVAL, "download_rows: need 0 <= row_a < row_b <= rows+2");
  if ((g->mode != Mode::Dist || g->rank == 0) && !out) return set_error(nullptr, SOR_E_INVAL, "out is NULL");
  DevGuard dg(g);
  if (out && is_device_ptr(out)) CU(cudaDeviceSynchronize());
  return gather_rows(g, row_a, row_b, g->mode == Mode::Dist && g->rank != 0 ? nullptr : out);
}

int sor_reset(sor_grid* g, const double* init) {
  TRY(usable(g));
  DevGuard dg(g);
  CU(cudaStreamSynchronize(g->stream));
  TRY(dist_barrier(g));  // no rank is still running on the planes being reloaded
  return load_grid(g, init);
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
  DevGuard dg(g);
  if (g->stream) cudaStreamSynchronize(g->stream);
  if (g->transport == Transport::Ipc && g->shm && !g->failed) {
    // no rank frees memory another rank still pushes into or has mapped
    if (shm_barrier(g, 60.0) == SOR_OK) {
      for (void* p : g->ipc_opened) cudaIpcCloseMemHandle(p);
      g->ipc_opened.clear();
      shm_barrier(g, 60.0);
    }
  }
  free_grid(g);
}

}  // extern "C"
