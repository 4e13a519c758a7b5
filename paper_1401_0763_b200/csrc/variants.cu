// variants.cu — NEXT-4: the parallel SOR variants the paper names beside
// red-black SOR [§3.1, P:147], "multi-color SOR" and "block-parallel SOR",
// behind sor_variant_iterate / sor_variant_solve (include/sor.h).  The paper
// gives no algorithm for either; DESIGN.md §3 readings N4-1 and N4-2 are the
// definitions both this file and the oracle follow:
//
//   multi-colour (N4-1): colour(i, j) = (ca*i + cb*j) mod nc; one iteration
//     = colour phases 0 .. nc-1, phase p applies Eq. 1 [P:97-100] to every
//     cell of colour p (a valid colouring: 5-point neighbours never share a
//     colour, so a phase is one parallel step);
//   block (N4-2): B x B blocks anchored at cell (1, 1), chessboard-coloured
//     (red iff bi+bj even); red blocks, then black blocks; natural
//     (row-major) order inside a block.
//
// One HBM pass per iteration, src -> dst (16 algorithmic bytes per update in
// fp64), on the handle's planes.  A CTA stages its tile plus a ghost ring in
// shared memory, runs every phase of the iteration there and writes its owned
// cells; tiles never synchronise:
//   multi-colour: ring of nc cells.  After phase p every cell at distance
//     >= p+1 from the staged region's edge holds its exact value (it read
//     neighbours at distance >= p, exact after phase p-1), so after nc
//     phases the owned tile (distance >= nc) is exact;
//   block: ring of B+1 cells.  The CTA also sweeps the red blocks of the ring
//     of blocks around its tile (their own neighbours are black, i.e. old
//     source values, within one more cell), so the black blocks of the tile
//     read exact reds.
// Eq. 1 in the canonical order (readings #2-#4: s = (N+S)+(W+E); a = 0.25 s;
// r = a - u; u' = u + w r, every operation rounded, no FMA), |delta| by
// subtraction (reading #5), ordered-bits atomicMax per CTA; the stop test
// (strict <, reading #7) runs in a one-thread decision kernel after each
// checked iteration and later kernels of the batch exit at once.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "sor_internal.h"

using namespace sorh;

namespace {

struct VarCtl {                   // device; one per handle (sor_grid::vctl)
  unsigned long long maxbits;     // running max of the checked iteration
  unsigned long long last_bits;   // max of the last checked iteration
  long long stop_iter;            // iteration (1-based, in this call) that converged
  int stop;                       // solve converged: later launches exit
  int pad;
};

constexpr int kMcTX = 64, kMcTY = 32, kMcThreads = 256;   // multi-colour tile (owned cells)
constexpr int kBpThreads = 128;

struct VarGeom {
  const void* src;
  void* dst;
  long long pitch;   // elements
  long long r0;      // storage row of global row 0
  int rows, cols;
};

template <typename R>
__device__ __forceinline__ R vupd(R n, R s, R wv, R e, R u, R w) {
  const R sum = radd(radd(n, s), radd(wv, e));
  const R a = rmul(R(0.25), sum);
  return radd(u, rmul(w, rsub(a, u)));
}

template <typename R>
__device__ __forceinline__ void cta_max(unsigned long long dmax, unsigned long long* slot) {
  __shared__ unsigned long long wm[32];
  dmax = warp_max_u64(dmax);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) wm[wid] = dmax;
  __syncthreads();
  if (wid == 0) {
    unsigned long long m = lane < nw ? wm[lane] : 0ull;
    m = warp_max_u64(m);
    if (lane == 0 && m) atomicMax(slot, m);
  }
}

// Multi-colour iteration.  cbyte per staged cell: colour (0..7), | 0x10 if
// owned, 0xff if never updated (outside the interior or on the staged edge).
template <typename R>
__global__ void __launch_bounds__(kMcThreads) mc_kernel(VarGeom G, int ca, int cb, int nc, R w, int check,
                                                        VarCtl* ctl, int solve) {
  if (solve && *reinterpret_cast<volatile int*>(&ctl->stop)) return;
  extern __shared__ __align__(16) unsigned char vsm[];
  const int h = nc, W = kMcTX + 2 * h, H = kMcTY + 2 * h, n = W * H;
  R* s = reinterpret_cast<R*>(vsm);
  unsigned char* cbyte = vsm + ((size_t)n * sizeof(R) + 15) / 16 * 16;
  const R* src = reinterpret_cast<const R*>(G.src);
  R* dst = reinterpret_cast<R*>(G.dst);
  const int x0 = 1 + blockIdx.x * kMcTX, y0 = 1 + blockIdx.y * kMcTY;  // first owned cell
  for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
    const int r = idx / W, c = idx - r * W;
    const int gi = y0 - h + r, gj = x0 - h + c;
    const bool in = gi >= 0 && gi <= G.rows + 1 && gj >= 0 && gj <= G.cols + 1;
    s[idx] = in ? src[(G.r0 + gi) * G.pitch + gj] : R(0);
    unsigned char cb8 = 0xff;
    if (gi >= 1 && gi <= G.rows && gj >= 1 && gj <= G.cols && r > 0 && r < H - 1 && c > 0 && c < W - 1) {
      int col = (int)(((long long)ca * gi + (long long)cb * gj) % nc);
      if (col < 0) col += nc;
      cb8 = (unsigned char)col;
      if (r >= h && r < h + kMcTY && c >= h && c < h + kMcTX) cb8 |= 0x10;
    }
    cbyte[idx] = cb8;
  }
  unsigned long long dmax = 0ull;
  for (int p = 0; p < nc; ++p) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
      const unsigned char cb8 = cbyte[idx];
      if ((cb8 & 0x0f) != p || cb8 == 0xff) continue;
      const R u = s[idx];
      const R v = vupd(s[idx - W], s[idx + W], s[idx - 1], s[idx + 1], u, w);
      s[idx] = v;
      if (check && (cb8 & 0x10)) dmax = umax64(dmax, delta_bits(v, u));
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < kMcTX * kMcTY; idx += blockDim.x) {
    const int r = idx / kMcTX, c = idx - r * kMcTX;
    const int gi = y0 + r, gj = x0 + c;
    if (gi <= G.rows && gj <= G.cols) dst[(G.r0 + gi) * G.pitch + gj] = s[(r + h) * W + c + h];
  }
  if (check) cta_max<R>(dmax, &ctl->maxbits);
}

// Block red-black iteration.  The CTA owns MB x MB blocks (tile side MB*B
// cells); staged region = tile + (B+1) cells per side; one thread sweeps
// one block at a time in row-major order.
template <typename R>
__global__ void __launch_bounds__(kBpThreads) bp_kernel(VarGeom G, int B, int MB, R w, int check, VarCtl* ctl,
                                                        int solve) {
  if (solve && *reinterpret_cast<volatile int*>(&ctl->stop)) return;
  extern __shared__ __align__(16) unsigned char vsm[];
  const int TS = MB * B, h = B + 1, W = TS + 2 * h, n = W * W;
  R* s = reinterpret_cast<R*>(vsm);
  const R* src = reinterpret_cast<const R*>(G.src);
  R* dst = reinterpret_cast<R*>(G.dst);
  const int bx0 = blockIdx.x * MB, by0 = blockIdx.y * MB;  // first owned block (global block index)
  const int x0 = 1 + bx0 * B, y0 = 1 + by0 * B;            // its first cell
  for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
    const int r = idx / W, c = idx - r * W;
    const int gi = y0 - h + r, gj = x0 - h + c;
    const bool in = gi >= 0 && gi <= G.rows + 1 && gj >= 0 && gj <= G.cols + 1;
    s[idx] = in ? src[(G.r0 + gi) * G.pitch + gj] : R(0);
  }
  unsigned long long dmax = 0ull;
  const int nbr = MB + 2;  // blocks per side of the staged ring of blocks
  for (int colour = 0; colour < 2; ++colour) {
    __syncthreads();
    // red: the tile's blocks and the ring of blocks; black: the tile's blocks
    const int lo = colour == 0 ? 0 : 1, hi = colour == 0 ? nbr : nbr - 1;
    const int span = hi - lo;
    for (int t = threadIdx.x; t < span * span; t += blockDim.x) {
      const int lbi = lo + t / span, lbj = lo + t % span;     // local block index, ring = 0 / MB+1
      const int gbi = by0 - 1 + lbi, gbj = bx0 - 1 + lbj;     // global block index
      if (gbi < 0 || gbj < 0 || ((gbi + gbj) & 1) != colour) continue;
      const int gi0 = 1 + gbi * B, gj0 = 1 + gbj * B;
      if (gi0 > G.rows || gj0 > G.cols) continue;
      const int ni = min(B, G.rows + 1 - gi0), nj = min(B, G.cols + 1 - gj0);
      const bool own = lbi >= 1 && lbi <= MB && lbj >= 1 && lbj <= MB;
      // staged index of the block's first cell
      const int base = (gi0 - (y0 - h)) * W + (gj0 - (x0 - h));
      for (int i = 0; i < ni; ++i) {
        int o = base + i * W;
        R wv = s[o - 1];  // the row's west neighbour (old, another block, or the ring)
        for (int j = 0; j < nj; ++j, ++o) {
          const R u = s[o];
          const R v = vupd(s[o - W], s[o + W], wv, s[o + 1], u, w);
          s[o] = v;
          wv = v;
          if (check && own) dmax = umax64(dmax, delta_bits(v, u));
        }
      }
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < TS * TS; idx += blockDim.x) {
    const int r = idx / TS, c = idx - r * TS;
    const int gi = y0 + r, gj = x0 + c;
    if (gi <= G.rows && gj <= G.cols) dst[(G.r0 + gi) * G.pitch + gj] = s[(r + h) * W + c + h];
  }
  if (check) cta_max<R>(dmax, &ctl->maxbits);
}

// Stop test of a checked iteration k (Algorithm 1; strict <).
__global__ void var_decide(VarCtl* ctl, long long k, double tol, int solve) {
  if (ctl->stop) return;
  const unsigned long long m = ctl->maxbits;
  ctl->maxbits = 0ull;
  ctl->last_bits = m;
  if (solve && __longlong_as_double((long long)m) < tol) {
    ctl->stop = 1;
    ctl->stop_iter = k;
  }
}

int bp_tile_blocks(int B) {
  int MB = std::max(1, 64 / B);
  while (MB > 1 && MB * B + 2 * (B + 1) > 100) --MB;
  return MB;
}

template <typename R>
size_t var_smem(const sor_variant* v) {
  if (v->kind == SOR_VARIANT_MULTICOLOR) {
    const int n = (kMcTX + 2 * v->nc) * (kMcTY + 2 * v->nc);
    return ((size_t)n * sizeof(R) + 15) / 16 * 16 + (size_t)n;
  }
  const int MB = bp_tile_blocks(v->block), Wd = MB * v->block + 2 * (v->block + 1);
  return (size_t)Wd * Wd * sizeof(R);
}

}  // namespace

namespace sorh {

int variant_check(const sor_grid* g, const sor_variant* v) {
  if (!v) return set_error(nullptr, SOR_E_INVAL, "variant is NULL");
  if (v->kind == SOR_VARIANT_MULTICOLOR) {
    if (v->nc < 2 || v->nc > 8) return set_error(nullptr, SOR_E_UNSUPPORTED, "multi-colour: need 2 <= nc <= 8");
    if (v->ca % v->nc == 0 || v->cb % v->nc == 0)
      return set_error(nullptr, SOR_E_INVAL, "multi-colour: ca and cb must not be multiples of nc (invalid colouring)");
  } else if (v->kind == SOR_VARIANT_BLOCK) {
    if (v->block < 1 || v->block > 32) return set_error(nullptr, SOR_E_UNSUPPORTED, "block SOR: need 1 <= block <= 32");
  } else {
    return set_error(nullptr, SOR_E_INVAL, "unknown variant kind %d", v->kind);
  }
  if (!single_part(g) || g->mode != Mode::Single)
    return set_error(nullptr, SOR_E_UNSUPPORTED, "NEXT-4 variants run on single-GPU handles only");
  return SOR_OK;
}

template <typename R>
int variant_run(sor_grid* g, const sor_variant* v, double omega, int solve, int64_t n_iter, double tol, int64_t K,
                int measure_last, int64_t* iters_out, double* max_out, int* converged) {
  const Slab& sl = g->slabs[0];
  if (!g->vctl) {
    void* p = nullptr;
    CU(cudaMalloc(&p, sizeof(VarCtl)));
    g->vctl = p;
  }
  if (!g->vhost) {
    void* p = nullptr;
    CU(cudaMallocHost(&p, sizeof(VarCtl)));
    g->vhost = p;
  }
  VarCtl* ctl = reinterpret_cast<VarCtl*>(g->vctl);
  VarCtl* hc = reinterpret_cast<VarCtl*>(g->vhost);
  CU(cudaMemsetAsync(ctl, 0, sizeof(VarCtl), g->stream));
  const size_t smem = var_smem<R>(v);
  static bool attr_set[kMaxDev][2][2] = {};
  const int ki = v->kind == SOR_VARIANT_MULTICOLOR ? 0 : 1, di = sizeof(R) == 8 ? 0 : 1;
  if (!attr_set[g->device][ki][di]) {
    if (ki == 0)
      CU(cudaFuncSetAttribute(mc_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    else
      CU(cudaFuncSetAttribute(bp_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    attr_set[g->device][ki][di] = true;
  }
  VarGeom G{};
  G.pitch = g->pitch;
  G.r0 = -sl.g0;
  G.rows = (int)g->rows;
  G.cols = (int)g->cols;
  const R w = (R)omega;
  int a = g->cur, b = a == 0 ? 1 : 0;
  const int a0 = a, b0 = b;
  const int64_t batch = solve ? 256 : std::max<int64_t>(n_iter, 1);
  int64_t done = 0, launches = 0, checks = 0;
  bool stopped = false;
  int64_t k_stop = 0;
  const int MB = ki == 1 ? bp_tile_blocks(v->block) : 0;
  const dim3 grid_mc((unsigned)((g->cols + kMcTX - 1) / kMcTX), (unsigned)((g->rows + kMcTY - 1) / kMcTY));
  const int TS = MB * v->block;
  const dim3 grid_bp(ki == 1 ? (unsigned)((g->cols + TS - 1) / TS) : 1u, ki == 1 ? (unsigned)((g->rows + TS - 1) / TS) : 1u);
  for (int64_t k0 = 1; k0 <= n_iter && !stopped; k0 += batch) {
    const int64_t k1 = std::min(n_iter, k0 + batch - 1);
    for (int64_t k = k0; k <= k1; ++k) {
      const int check = solve ? (k % K == 0) : (measure_last && k == n_iter);
      G.src = col0<R>(sl.plane[a]);
      G.dst = col0<R>(sl.plane[b]);
      if (ki == 0)
        mc_kernel<R><<<grid_mc, kMcThreads, smem, g->stream>>>(G, v->ca, v->cb, v->nc, w, check, ctl, solve);
      else
        bp_kernel<R><<<grid_bp, kBpThreads, smem, g->stream>>>(G, v->block, MB, w, check, ctl, solve);
      ++launches;
      if (check) {
        var_decide<<<1, 1, 0, g->stream>>>(ctl, (long long)k, tol, solve);
        ++launches;
        ++checks;
      }
      std::swap(a, b);
    }
    CU(cudaGetLastError());
    done = k1;
    if (solve) {
      CU(cudaMemcpyAsync(hc, ctl, sizeof(VarCtl), cudaMemcpyDeviceToHost, g->stream));
      CU(cudaStreamSynchronize(g->stream));
      if (hc->stop) {
        stopped = true;
        k_stop = hc->stop_iter;
      }
    }
  }
  if (!solve || !stopped) {
    CU(cudaMemcpyAsync(hc, ctl, sizeof(VarCtl), cudaMemcpyDeviceToHost, g->stream));
    CU(cudaStreamSynchronize(g->stream));
  }
  const int64_t iters = stopped ? k_stop : done;
  g->cur = (iters & 1) ? b0 : a0;  // iteration k writes plane b0 if k is odd
  g->st.kernel_launches += launches;
  g->st.half_sweeps += iters * (ki == 0 ? v->nc : 2);
  g->st.hbm_passes += iters;
  g->st.checks += stopped ? k_stop / K : (solve ? done / K : checks);
  if (iters_out) *iters_out = iters;
  if (max_out) std::memcpy(max_out, &hc->last_bits, sizeof(double));
  if (converged) *converged = stopped ? 1 : 0;
  return SOR_OK;
}

template int variant_run<double>(sor_grid*, const sor_variant*, double, int, int64_t, double, int64_t, int, int64_t*,
                                 double*, int*);
template int variant_run<float>(sor_grid*, const sor_variant*, double, int, int64_t, double, int64_t, int, int64_t*,
                                double*, int*);

}  // namespace sorh
