// sor_internal.h — host-side state of a libsor handle, shared by the
// translation units of the library (sor_api.cu: driver + C ABI; wave_*.cu,
// jacobi_inst.cu: kernel instantiations and their launchers; sor3d.cu:
// NEXT-3).  Not part of the C ABI (include/sor.h is).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "sor.h"
#include "sor_kernels.cuh"

namespace sorh {
using namespace sorb;

constexpr int kMaxDev = 64;  // per-device caches (occupancy, function attributes)

// A neighbouring slab as seen from this one: its planes and halo flags,
// either another slab of this handle (virtual) or another rank's memory
// mapped over CUDA IPC (dist).
struct Neighbour {
  bool ok = false;
  void* plane[3] = {nullptr, nullptr, nullptr};
  unsigned long long* ftop = nullptr;  // its top-halo flags
  unsigned long long* fbot = nullptr;  // its bottom-halo flags
  int64_t g0 = 0;
};

struct Slab {
  int64_t g_lo = 0, g_hi = 0;  // owned global interior rows [g_lo, g_hi)
  int64_t g0 = 0;              // global row of storage row 0 (= g_lo - kRowPad)
  int64_t nstore = 0;          // storage rows
  // planes 0, 1: ping-pong; plane 2 (allocated on the first deferred solve,
  // up front for dist-IPC): the speculative pass of the deferred stop test
  void* plane[3] = {nullptr, nullptr, nullptr};
  WaveMaps tmap[3];   // per plane: tensor maps of the wave kernel's source-row boxes (6, 2 rows)
  WaveMaps tmap2[3];  // per plane: the skew-2 wave kernel's boxes (4, 3 rows)
  // device-initiated halo exchange (HaloLink): this slab's flags (released by
  // the neighbours) and the neighbours it pushes to
  unsigned long long* ftop = nullptr;
  unsigned long long* fbot = nullptr;
  Neighbour up, dn;
};

enum class Mode { Single, Virtual, Dist };
enum class Transport { None, Nccl, Ipc };

// Who wrote a plane's halo rows last: the pass's sequence number (0: loaded
// or filled by a host-side exchange, nothing to wait for) and its strip
// layout (HaloLink::pg/pw/pgh/pn).
struct PlaneInfo {
  unsigned long long wseq = 0;
  int pg = 0, pw = 1, pgh = 0, pn = 0;
};

struct ShmSeg;  // dist-IPC host rendezvous (sor_api.cu)

}  // namespace sorh

struct sor_grid {
  int64_t rows = 0, cols = 0;
  sor_dtype dt = SOR_F64;
  size_t esz = 8;
  int64_t pitch = 0;  // elements
  sorh::Mode mode = sorh::Mode::Single;
  std::vector<sorh::Slab> slabs;
  int cur = 0;  // plane holding the current iterate (same for all slabs)
  int kernel = SOR_KERNEL_FUSED;
  int tdepth = 1;
  int device = 0;
  int nsm = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t poll_ev[2] = {nullptr, nullptr};
  sorb::DevState* dstate = nullptr;
  sorb::DevState* hstate = nullptr;  // pinned, 2 slots for one-batch-behind polling
  double* scratch = nullptr;         // f64 staging for f32 pack/unpack and dist scatter/gather
  size_t scratch_bytes = 0;
  unsigned int* dflag = nullptr;
  unsigned int* gbar = nullptr;  // K6: grid-barrier counter of the persistent kernel
  bool persist_off = false;      // K6 tiles did not fit in one wave on this handle
  unsigned long long* rflags = nullptr;  // K7: per-block pass flags (stride 16 words), allocated on first use
  uint64_t rseq = 0;                     // K7: flag base of the next launch
  int rank = 0, nranks = 1;
  sorh::Transport transport = sorh::Transport::None;
  ncclComm_t comm = nullptr;
  // device-initiated halo exchange (virtual slabs, dist over IPC)
  bool push = false;               // wave passes push their edge rows (no exchange copies)
  int H = 0;                       // rows pushed per side
  unsigned long long seq = 0;      // wave passes launched on this handle
  sorh::PlaneInfo pinfo[3];
  void* flagbuf = nullptr;         // virtual: all slabs' flags; dist-IPC: this rank's DistComm + flags
  int nflags = 0;                  // flags per side per slab
  sorb::DistJoinTab* djoin = nullptr;  // dist-IPC: device table of every rank's comm block
  bool lockstep = false;           // dist-IPC ranks sharing a GPU: host barrier after every pass
  sorh::ShmSeg* shm = nullptr;
  std::vector<void*> ipc_opened;   // mappings to close on destroy
  std::vector<sorh::Slab> rslabs;  // dist-IPC rank 0: every rank's slab, mapped (scatter / gather)
  int halo_valid = sorb::kRowPad;  // rows of the current plane's halos known up to date
  struct PassRec {
    int64_t k_last;
    int src, dst, T;
    sorh::PlaneInfo spi, dpi;  // halo bookkeeping of src before / dst after the pass
  };
  std::vector<PassRec> pass_ends;  // wave passes of the current solve segment
  int nplanes = 2;                 // planes in rotation (3 once the deferred solve allocated plane 2)
  int nxt(int p) const { return (p + 1) % nplanes; }
  // deferred stop test: the last checked pass not yet decided, and the slot set
  // the next checked pass contributes to
  bool prev_valid = false;
  int prev_T = 0, prev_ck = 0, prev_set = 0, next_set = 0;
  int64_t prev_k_last = 0;
  unsigned long long prev_seq = 0;
  // wave-kernel tile tables per (slab, layout, occupancy): device int4 array + count
  std::map<std::tuple<int, int, int>, std::pair<int4*, int>> tiles;
  int64_t exact_reruns = 0;  // solve passes re-run with exact maxima (diagnostic)
  int every_ck = 4;          // max-change mode of T-deep solve passes with check_every == 1
  int method = 0;            // 0: red-black SOR; 1: Jacobi (sor_jacobi_*; NEXT-2)
  void* vctl = nullptr;      // NEXT-4 variants: device control block (variants.cu)
  void* vhost = nullptr;     // ... and its pinned host copy
  bool failed = false;
  bool have_elapsed = false;
  double elapsed_ms = 0.0;
  sor_stats st{};
};

namespace sorh {

extern thread_local std::string g_last_error;
int set_error(sor_grid* g, int code, const char* fmt, ...);

#define CU(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return ::sorh::set_error(g, SOR_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define NC(call)                                                                      \
  do {                                                                                \
    ncclResult_t r_ = (call);                                                         \
    if (r_ != ncclSuccess)                                                            \
      return ::sorh::set_error(g, SOR_E_NCCL, "%s failed: %s", #call, ncclGetErrorString(r_)); \
  } while (0)

#define TRY(expr)             \
  do {                        \
    int rc_ = (expr);         \
    if (rc_ < 0) return rc_;  \
  } while (0)

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

template <typename R>
R* col0(void* plane) {
  return reinterpret_cast<R*>(plane) + kColPad;
}

inline bool single_part(const sor_grid* g) { return g->slabs.size() == 1 && g->nranks == 1; }

bool is_device_ptr(const void* p);
bool host_all_finite(const double* p, int64_t n);

// Wave-kernel tiles of slab `s` for a layout (ghost columns per side, S stages,
// strip width wc, tiles per SM, split pairs, strip origin s0); cached.
// `reserve` tiles of the one-wave budget are left free (the deferred stop
// test's decision CTA).
int wave_tiles(sor_grid* g, const Slab& s, int slab_idx, int ghost, int S, int wc, int tiles_per_sm, bool split,
               int s0, std::pair<int4*, int>* out, int reserve = 0);
bool wave_pdl(const sor_grid* g, unsigned blocks, int occ);
// HaloLink of slab `s` for a pass src -> dst with the given strip layout; also
// records the layout as the writer of plane dst.
HaloLink make_link(sor_grid* g, const Slab& s, int src, int dst);
void record_layout(sor_grid* g, int dst, int s0, int wc, int ghost, int nstrips);
int strips_of(const sor_grid* g, int s0, int wc, int ghost);

// Launchers (explicitly instantiated in wave_*.cu / jacobi_inst.cu).
template <typename R, int T, int CK, bool LINK>
int launch_wave_T(sor_grid* g, const Slab& s, R w, const IterCtl& ctl, bool fused_fin);
template <typename R, int T, int CK, bool LINK>
int launch_jacobi_T(sor_grid* g, const Slab& s, const IterCtl& ctl, bool fused_fin);
template <typename R, int T>
int launch_wave_persist(sor_grid* g, const Slab& s, R w, int npasses, unsigned* gbar);
template <typename R, int T, int CK, bool LINK>
int launch_wave2_T(sor_grid* g, const Slab& s, R w, const IterCtl& ctl, bool fused_fin);
bool use_wave2(const sor_grid* g, int T);

// K7 (resident.cu): the grid register-resident across the SMs.  Iterate
// passes of T with neighbour-only exchange (multi-CTA), or one CTA running
// Algorithm 1's loop (single).  SOR_E_UNSUPPORTED if the grid does not fit.
template <typename R>
int launch_resident_iterate(sor_grid* g, R w, int64_t iters, int T, bool check_last);
template <typename R>
int launch_resident_single(sor_grid* g, R w, int solve, int64_t n_iter, double tol, int64_t K, int check_last);
bool resident_fits(const sor_grid* g, int T, bool single);

// NEXT-4 (variants.cu): multi-colour / block red-black SOR on single-GPU
// handles, one HBM pass per iteration.
int variant_check(const sor_grid* g, const sor_variant* v);
template <typename R>
int variant_run(sor_grid* g, const sor_variant* v, double omega, int solve, int64_t n_iter, double tol, int64_t K,
                int measure_last, int64_t* iters_out, double* max_out, int* converged);

}  // namespace sorh
