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

constexpr int kMcTY = 64, kMcThreads = 256;   // multi-colour tile rows (owned cells); width: mc_tile_x
constexpr int kBpThreads = 256;

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

// Staged region [y0s, y0s+H) x [x0s, x0s+W) of src into s (row-major, W
// <= 160 per row): a warp per row, lanes along the row (coalesced).  Each
// thread issues up to 15 loads (3 rows x 5 column chunks) before its first
// shared store, so enough bytes are in flight to cover the HBM latency (one
// load per iteration capped the kernels at ~1.5 TB/s), and no index is
// divided.  Cells outside the grid (never read by an interior update) are 0.
template <typename R>
__device__ __forceinline__ void var_stage(const VarGeom& G, const R* __restrict__ src, R* s, int y0s, int x0s, int H,
                                          int W) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r0 = warp; r0 < H; r0 += 3 * nw) {
    R v[3][5];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int r = r0 + u * nw, gi = y0s + r;
      const bool rok = r < H && gi >= 0 && gi <= G.rows + 1;
      const R* row = src + (G.r0 + gi) * G.pitch;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int c = lane + 32 * k, gj = x0s + c;
        v[u][k] = rok && c < W && gj >= 0 && gj <= G.cols + 1 ? __ldg(row + gj) : R(0);
      }
    }
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int r = r0 + u * nw;
#pragma unroll
      for (int k = 0; k < 5; ++k)
        if (r < H && lane + 32 * k < W) s[r * W + lane + 32 * k] = v[u][k];
    }
  }
}

// The owned TY x TX cells of the staged region (offset h) back to dst.
template <typename R>
__device__ __forceinline__ void var_store(const VarGeom& G, R* dst, const R* s, int y0, int x0, int TY, int TX, int h,
                                          int W) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = warp; r < TY; r += nw) {
    const int gi = y0 + r;
    if (gi > G.rows) break;
    R* row = dst + (G.r0 + gi) * G.pitch;
    for (int c = lane; c < TX; c += 32)
      if (x0 + c <= G.cols) row[x0 + c] = s[(r + h) * W + c + h];
  }
}

// Multi-colour iteration.  The cells of colour p in a staged row are the
// columns f, f+q, f+2q, ... with q = nc / gcd(cb, nc) and f = first[p][ca*i
// mod nc] (a table built per CTA), so a warp updates one row of one colour
// with its lanes packed on those columns (lane m: column f + q*m); the tile
// width TX (host: mc_tile_x) makes a row hold ~32 of them.  Rows go to
// warps round-robin.
template <typename R>
__global__ void __launch_bounds__(kMcThreads) mc_kernel(VarGeom G, int ca, int cb, int nc, int TX, R w, int check,
                                                        VarCtl* ctl, int solve) {
  if (solve && *reinterpret_cast<volatile int*>(&ctl->stop)) return;
  extern __shared__ __align__(16) unsigned char vsm[];
  const int h = nc, W = TX + 2 * h, H = kMcTY + 2 * h;
  R* s = reinterpret_cast<R*>(vsm);
  __shared__ int rowres[kMcTY + 16];  // ca*i mod nc of each staged row (-1: not updated)
  __shared__ int first[8][8];         // [p][row residue]: first staged column >= 1 of colour p, or -1
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int x0 = 1 + blockIdx.x * TX, y0 = 1 + blockIdx.y * kMcTY;  // first owned cell
  const int x0s = x0 - h, y0s = y0 - h;                              // first staged cell
  // residues of ca, cb in [0, nc): ca*i mod nc = (car*i) mod nc, 32-bit (i < 2^27)
  const unsigned car = (unsigned)(ca % nc + nc) % nc, cbr = (unsigned)(cb % nc + nc) % nc;
  int q = nc;
  for (int d = 1; d <= nc; ++d)
    if ((cbr * (unsigned)d) % (unsigned)nc == 0u) {
      q = d;
      break;
    }
  for (int r = threadIdx.x; r < H; r += blockDim.x) {
    const int gi = y0s + r;
    rowres[r] = r > 0 && r < H - 1 && gi >= 1 && gi <= G.rows ? (int)((car * (unsigned)gi) % (unsigned)nc) : -1;
  }
  if (threadIdx.x < nc * nc) {
    const int p = threadIdx.x / nc, rr = threadIdx.x - p * nc;
    int f = -1;
    for (int c = 1; c <= q && f < 0; ++c) {  // staged column c is global column x0s + c (>= -6)
      const unsigned gj = (unsigned)(x0s + c + 8 * nc);  // + a multiple of nc keeps it positive
      if ((int)(((unsigned)rr + (cbr * gj) % (unsigned)nc) % (unsigned)nc) == p) f = c;
    }
    first[p][rr] = f;
  }
  var_stage(G, reinterpret_cast<const R*>(G.src), s, y0s, x0s, H, W);
  unsigned long long dmax = 0ull;
  // Four rows (nw apart: same colour, never neighbours) per warp step, their
  // loads issued before their updates (ILP; one row per step left the
  // kernel latency-bound at 43 % issue).
  const int nchunk = (W - 2 + 32 * q - 1) / (32 * q);
  for (int p = 0; p < nc; ++p) {
    __syncthreads();
    for (int kk = 0; kk < nchunk; ++kk) {
      for (int rb = 1 + warp; rb < H - 1; rb += 4 * nw) {
        R vn[4], vs[4], vw[4], ve[4], vu[4];
        int vo[4];
        bool act[4], own[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = rb + u * nw;
          const int rc = r < H - 1 ? rowres[r] : -1;
          const int f = rc >= 0 ? first[p][rc] : -1;
          const int c = f + q * (lane + 32 * kk), gj = x0s + c;
          act[u] = f >= 0 && c < W - 1 && gj >= 1 && gj <= G.cols;
          own[u] = r >= h && r < h + kMcTY && c >= h && c < h + TX;
          vo[u] = r * W + c;
          if (act[u]) {
            vn[u] = s[vo[u] - W];
            vs[u] = s[vo[u] + W];
            vw[u] = s[vo[u] - 1];
            ve[u] = s[vo[u] + 1];
            vu[u] = s[vo[u]];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (act[u]) {
            const R v = vupd(vn[u], vs[u], vw[u], ve[u], vu[u], w);
            s[vo[u]] = v;
            if (check && own[u]) dmax = umax64(dmax, delta_bits(v, vu[u]));
          }
        }
      }
    }
  }
  __syncthreads();
  var_store(G, reinterpret_cast<R*>(G.dst), s, y0, x0, kMcTY, TX, h, W);
  if (check) cta_max<R>(dmax, &ctl->maxbits);
}

// Block red-black iteration.  The CTA owns MB x MB blocks (tile side MB*B
// cells); staged region = tile + (B+1) cells per side.  A team of B lanes
// sweeps a block as an anti-diagonal wavefront: lane r owns row r of the
// block and at step t updates column t-r, after lane r-1 updated (r-1, t-r)
// and itself (r, t-r-1) at step t-1 and before anyone updates (r+1, t-r) or
// (r, t-r+1): exactly the values the row-major sweep reads (bitwise equal).
template <typename R>
__global__ void __launch_bounds__(kBpThreads) bp_kernel(VarGeom G, int B, int MB, R w, int check, VarCtl* ctl,
                                                        int solve) {
  if (solve && *reinterpret_cast<volatile int*>(&ctl->stop)) return;
  extern __shared__ __align__(16) unsigned char vsm[];
  const int TS = MB * B, h = B + 1, W = TS + 2 * h;
  R* s = reinterpret_cast<R*>(vsm);
  const int bx0 = blockIdx.x * MB, by0 = blockIdx.y * MB;  // first owned block (global block index)
  const int x0 = 1 + bx0 * B, y0 = 1 + by0 * B;            // its first cell
  var_stage(G, reinterpret_cast<const R*>(G.src), s, y0 - h, x0 - h, W, W);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int tpw = 32 / B;  // teams per warp
  const int tiw = lane / B, r = lane - tiw * B;
  const bool lane_ok = tiw < tpw;
  const int nteams = nw * tpw, team = warp * tpw + tiw;
  unsigned long long dmax = 0ull;
  for (int colour = 0; colour < 2; ++colour) {
    __syncthreads();
    // red: the tile's blocks and the ring of blocks (local 0 .. MB+1); black: the tile's
    const int lo = colour == 0 ? 0 : 1, span = colour == 0 ? MB + 2 : MB;
    const int half = (span + 1) / 2, nslots = span * half;
    const int rounds = (nslots + nteams - 1) / nteams;
    for (int m = 0; m < rounds; ++m) {
      const int q = team + m * nteams;
      const int row = q / half, jj = q - row * half;
      const int lbi = lo + row;
      const int gbi = by0 - 1 + lbi;
      // blocks of this colour in the row have local column parity `off`
      const int off = (colour - gbi - (bx0 - 1 + lo)) & 1;
      const int lbj = lo + off + 2 * jj, gbj = bx0 - 1 + lbj;
      const int gi0 = 1 + gbi * B, gj0 = 1 + gbj * B;
      const bool act = lane_ok && q < nslots && lbj < lo + span && gbi >= 0 && gbj >= 0 && gi0 <= G.rows &&
                       gj0 <= G.cols;
      const int ni = act ? min(B, G.rows + 1 - gi0) : 0, nj = act ? min(B, G.cols + 1 - gj0) : 0;
      const bool own = lbi >= 1 && lbi <= MB && lbj >= 1 && lbj <= MB;
      const int o0 = (gi0 - (y0 - h) + r) * W + (gj0 - (x0 - h));  // row r, column 0 of the block
      for (int t = 0; t < 2 * B - 1; ++t) {
        const int j = t - r;
        if (r < ni && j >= 0 && j < nj) {
          const int o = o0 + j;
          const R u = s[o];
          const R v = vupd(s[o - W], s[o + W], s[o - 1], s[o + 1], u, w);
          s[o] = v;
          if (check && own) dmax = umax64(dmax, delta_bits(v, u));
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  var_store(G, reinterpret_cast<R*>(G.dst), s, y0, x0, TS, TS, h, W);
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

// Multi-colour tile width: the staged interior columns of a row (TX + 2nc - 2)
// hold 32k cells of one colour (period q = nc / gcd(cb, nc)) for the largest
// k with TX <= 128; at least 64 columns.
int mc_tile_x(const sor_variant* v) {
  const int nc = v->nc, cbr = ((v->cb % nc) + nc) % nc;
  int q = nc;
  for (int d = 1; d <= nc; ++d)
    if ((cbr * d) % nc == 0) {
      q = d;
      break;
    }
  int best = 0;
  for (int k = 1; 32 * q * k - 2 * nc + 2 <= 128; ++k) best = 32 * q * k - 2 * nc + 2;
  return std::max(best, 64);
}

int bp_tile_blocks(int B) {
  int MB = std::max(1, 64 / B);
  while (MB > 1 && MB * B + 2 * (B + 1) > 100) --MB;
  return MB;
}

template <typename R>
size_t var_smem(const sor_variant* v) {
  if (v->kind == SOR_VARIANT_MULTICOLOR) {
    return (size_t)(mc_tile_x(v) + 2 * v->nc) * (kMcTY + 2 * v->nc) * sizeof(R);
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
  const int TX = ki == 0 ? mc_tile_x(v) : 64;
  const dim3 grid_mc((unsigned)((g->cols + TX - 1) / TX), (unsigned)((g->rows + kMcTY - 1) / kMcTY));
  const int TS = MB * v->block;
  const dim3 grid_bp(ki == 1 ? (unsigned)((g->cols + TS - 1) / TS) : 1u, ki == 1 ? (unsigned)((g->rows + TS - 1) / TS) : 1u);
  for (int64_t k0 = 1; k0 <= n_iter && !stopped; k0 += batch) {
    const int64_t k1 = std::min(n_iter, k0 + batch - 1);
    for (int64_t k = k0; k <= k1; ++k) {
      const int check = solve ? (k % K == 0) : (measure_last && k == n_iter);
      G.src = col0<R>(sl.plane[a]);
      G.dst = col0<R>(sl.plane[b]);
      if (ki == 0)
        mc_kernel<R><<<grid_mc, kMcThreads, smem, g->stream>>>(G, v->ca, v->cb, v->nc, TX, w, check, ctl, solve);
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
