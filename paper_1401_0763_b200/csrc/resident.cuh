// resident.cuh — K7: the grid held in REGISTERS across the SMs (small grids:
// BJ configs[0] and configs[1]).
//
// Method: Eq. 1 [§2.1, P:97-100] in the canonical form of sor_kernels.cuh,
// red phase then black phase [§3.1, P:149, P:198], max-change [P:103,
// P:319-325].  The cost the paper blames for its scaling is the barrier per
// colour phase [P:203, P:314, P:317, P:394]; for grids that fit in the
// register files of the 148 SMs (~1 M cells) that barrier becomes a CTA
// barrier, and the HBM/L2 pass and the kernel launch per pass disappear:
//
//  * Each CTA (CPS per SM) owns a 2-D block of interior cells.  Its WINDOW is
//    the block plus a ring of G = 2T cells (the dependency cone of T red+black
//    iterations: every half-sweep widens it by one cell), held in registers:
//    lane l of warp w owns rows [w*RPW, (w+1)*RPW) and columns
//    [l*NC, (l+1)*NC) of the window.  Window origin rows/columns are even and
//    RPW, NC are even, so the colour of register v[r][c] is (r + c) & 1 at
//    compile time (red = 0; global parity (i + j) even [P:149]).
//  * Half-sweep h (colour h & 1) of a T'-iteration pass has to be exact only
//    within e_h = 2T' - 1 - h of the block: a warp whose rows all lie beyond
//    e_h skips it, other cells beyond e_h (and every non-interior cell) keep
//    their value by predication.  N/S neighbours are the lane's own rows (the
//    rows of the neighbouring warps come through a small shared buffer
//    written at the end of the previous half-sweep), W/E the lane's own
//    columns and one shfl per row.  One __syncthreads per half-sweep (the
//    paper's phase barrier, CTA-local).
//  * After T' iterations the block is exact.  Between passes a block stores
//    the G-deep frame of its block into the plane of the next pass (L2) and
//    releases its flag (barrier, st.release.gpu); the next pass waits only for
//    the 8 neighbouring blocks' flags (ld.acquire.gpu, one thread each) and
//    reloads its ring from their frames.  No grid barrier, no launch per
//    pass.  (A flag-free low-latency format, every 8-byte word tagged with the
//    pass, measured slower: the consumers' polling loads compete with the
//    producers' stores for L2 bandwidth.)
//  * The last pass writes the whole block to the destination plane.  The
//    result is bitwise that of the in-place red-then-black sequence: every
//    cell within the cone reads exactly the values that sequence gives it
//    (by induction over the half-sweeps; cells beyond the cone are never read
//    by cells within it).
//
// Single-CTA form (nb = 1: block = the whole interior, window = the whole
// grid with its Dirichlet ring): no exchange; Algorithm 1's loop with the
// max-change of every K-th iteration reduced in the CTA and the stop test
// [P:319-331] decided by every thread (the K5 role, register-resident).
#pragma once

#include "sor_kernels.cuh"

namespace sorb {

template <typename R>
struct ResArgs {
  R* pa;  // column-0 pointers of the two planes: pass 0 loads the window from
  R* pb;  // pa; the last pass p writes the block to plane ((p + 1) & 1)
  long long pitch, g0;
  int rows, cols;
  int nbx, nby;  // block grid (blockIdx.x = by * nbx + bx)
  int G;         // ghost ring (2T)
  int T;         // iterations per full pass
  int npasses;
  int t_last;    // iterations in the last pass (1..T)
  unsigned long long* flags;  // one per block (stride 16 words): pass p releases seq0 + p + 1
  unsigned long long seq0;
  R w;
  IterCtl ctl;   // st (and, iterate with check_last: ck = 1 ticket finalize over the CTAs)
  int check_last;
  // single CTA: solve (stop test every K) or iterate
  int solve;
  long long n_iter, K;
  double tol;
  unsigned long long* trace;  // development aid (SOR_RES_TRACE): globaltimer per CTA, pass and phase
};

constexpr int kResBig = 1 << 28;

__device__ __forceinline__ unsigned long long cta_umax64_warp(unsigned long long x) {
  const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(x >> 32));
  const unsigned lo = __reduce_max_sync(0xffffffffu, ((unsigned)(x >> 32) == hi) ? (unsigned)x : 0u);
  return ((unsigned long long)hi << 32) | lo;
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename R>
__device__ __forceinline__ R res_shfl_up(R v) {
  return __shfl_up_sync(0xffffffffu, v, 1);
}
template <typename R>
__device__ __forceinline__ R res_shfl_dn(R v) {
  return __shfl_down_sync(0xffffffffu, v, 1);
}

// Exchange buffer of the rows at warp boundaries: xb[colour][warp][top/bot][k][lane],
// k = 0..NC/2-1 the lane's cells of that colour in that row.
template <typename R, int NC>
__device__ __forceinline__ R* res_xb(R* xb, int NW, int colour, int warp, int bot, int k, int lane) {
  return xb + ((((colour * NW + warp) * 2 + bot) * (NC / 2) + k) * 32 + lane);
}

template <typename R, int NC, int RPW>
struct ResCore {
  R v[RPW][NC];
  int rowe[RPW];  // distance of the row from the block (kResBig: not an interior row)
  int cole[NC];   // same for the lane's columns
  int wmin;       // min over the warp's rows of rowe (warp-uniform)
  // NC == 2 (one-CTA form on <= 64 interior columns): the window holds the
  // interior columns only, so lane 0's west and lane 31's east neighbours are
  // the Dirichlet ring columns, kept per row
  R wring[NC == 2 ? RPW : 1], ering[NC == 2 ? RPW : 1];
  bool edge_w, edge_e;

  // Colour-C half-sweep over the cells within e of the block.  Reads the
  // other colour's boundary rows of the neighbouring warps from xb[C ^ 1],
  // writes this colour's boundary rows to xb[C], then __syncthreads.
  // CHK: max |delta| over owned cells (distance 0) into dmax.
  template <int C, bool CHK>
  __device__ __forceinline__ void half(R* xb, int NW, int warp, int lane, int e, R w, unsigned long long& dmax) {
    if (wmin <= e) {  // warp-uniform: a warp entirely outside the cone has nothing to do
      R topN[NC / 2], botS[NC / 2];
#pragma unroll
      for (int k = 0; k < NC / 2; ++k) {
        topN[k] = warp > 0 ? *res_xb<R, NC>(xb, NW, C ^ 1, warp - 1, 1, k, lane) : R(0);
        botS[k] = warp + 1 < NW ? *res_xb<R, NC>(xb, NW, C ^ 1, warp + 1, 0, k, lane) : R(0);
      }
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const int c0 = (r + C) & 1;  // first column of colour C in this row (compile time after unrolling)
        // the lane-neighbour value this row needs (one shfl per row).  No
        // branch per row: cells outside the cone are computed and discarded
        // by the predicate, so the half-sweep is one basic block.
        R nb;
        if (c0 == 0) {
          nb = res_shfl_up(v[r][NC - 1]);
          if (NC == 2 && edge_w) nb = wring[NC == 2 ? r : 0];
        } else {
          nb = res_shfl_dn(v[r][0]);
          if (NC == 2 && edge_e) nb = ering[NC == 2 ? r : 0];
        }
#pragma unroll
        for (int k = 0; k < NC / 2; ++k) {
          const int c = c0 + 2 * k;
          const R uN = r > 0 ? v[r > 0 ? r - 1 : 0][c] : topN[k];
          const R uS = r + 1 < RPW ? v[r + 1 < RPW ? r + 1 : RPW - 1][c] : botS[k];
          const R uW = c > 0 ? v[r][c > 0 ? c - 1 : 0] : nb;
          const R uE = c + 1 < NC ? v[r][c + 1 < NC ? c + 1 : NC - 1] : nb;
          const R u = v[r][c];
          R p;
          const R un = sor_update_p(radd(uN, uS), radd(uW, uE), u, w, p);
          const bool upd = max(rowe[r], cole[c]) <= e;
          if (CHK) {
            if (upd && rowe[r] == 0 && cole[c] == 0) dmax = umax64(dmax, delta_bits(un, u));
          }
          if (upd) v[r][c] = un;
        }
      }
    }
    // this colour's boundary rows for the neighbouring warps' next half-sweep
#pragma unroll
    for (int k = 0; k < NC / 2; ++k) {
      *res_xb<R, NC>(xb, NW, C, warp, 0, k, lane) = v[0][(C & 1) + 2 * k];
      *res_xb<R, NC>(xb, NW, C, warp, 1, k, lane) = v[RPW - 1][((RPW - 1 + C) & 1) + 2 * k];
    }
    __syncthreads();
  }

  // Before a pass: publish the black (colour 1) boundary rows the first red
  // half-sweep reads.
  __device__ __forceinline__ void prime(R* xb, int NW, int warp, int lane) {
#pragma unroll
    for (int k = 0; k < NC / 2; ++k) {
      *res_xb<R, NC>(xb, NW, 1, warp, 0, k, lane) = v[0][1 + 2 * k];
      *res_xb<R, NC>(xb, NW, 1, warp, 1, k, lane) = v[RPW - 1][((RPW - 1 + 1) & 1) + 2 * k];
    }
    __syncthreads();
  }
};

__host__ __device__ constexpr int res_max_threads(int rpw, int cps) {
  return cps >= 2 ? 640 : (rpw <= 4 ? 640 : (rpw <= 6 ? 448 : 384));
}

template <typename R, int NC, int RPW, int CPS>
__global__ void __launch_bounds__(res_max_threads(RPW, CPS), CPS) resident_kernel(ResArgs<R> a) {
  extern __shared__ __align__(16) unsigned char res_smem[];
  R* xb = reinterpret_cast<R*>(res_smem);
  __shared__ unsigned long long wmax[2][32];
  const int NW = (int)(blockDim.x >> 5);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int bx = (int)blockIdx.x % a.nbx, by = (int)blockIdx.x / a.nbx;
  const bool single = a.nbx * a.nby == 1;
  // block [by0, by1) x [bx0, bx1) of interior cells (global indices, 1-based)
  const int bx0 = 1 + (int)((long long)bx * a.cols / a.nbx), bx1 = 1 + (int)((long long)(bx + 1) * a.cols / a.nbx);
  const int by0 = 1 + (int)((long long)by * a.rows / a.nby), by1 = 1 + (int)((long long)(by + 1) * a.rows / a.nby);
  const int G = single ? 1 : a.G;
  // window origin even (colour pattern; a lane's cell pairs are aligned vectors)
  // (NC == 2: origin (-1, 1), interior columns only; the colour pattern is the same)
  const int wx0 = NC == 2 ? 1 : (bx0 - G) & ~1, wy0 = NC == 2 ? -1 : (by0 - G) & ~1;
  const int gi0 = wy0 + warp * RPW, gj0 = wx0 + lane * NC;
  ResCore<R, NC, RPW> core;
  core.wmin = kResBig;
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int gi = gi0 + r;
    const int d = gi < by0 ? by0 - gi : (gi >= by1 ? gi - by1 + 1 : 0);
    core.rowe[r] = (gi >= 1 && gi <= a.rows) ? d : kResBig;
    core.wmin = min(core.wmin, core.rowe[r]);
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int gj = gj0 + c;
    const int d = gj < bx0 ? bx0 - gj : (gj >= bx1 ? gj - bx1 + 1 : 0);
    core.cole[c] = (gj >= 1 && gj <= a.cols) ? d : kResBig;
  }
  // cell masks (bit r*NC + c), computed once so no per-cell predicate or
  // address stays live across the passes: valid (inside the stored grid with
  // its ring), ring (interior cells outside the block within G of it: what
  // the neighbours send every pass), own (in the block), frame (in the block,
  // within G of its edge: what this block sends)
  static_assert(RPW * NC <= 32, "cell masks are 32 bits");
  unsigned m_valid = 0u, m_ring = 0u, m_own = 0u, m_frame = 0u;
#pragma unroll
  for (int r = 0; r < RPW; ++r)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int gi = gi0 + r, gj = gj0 + c, bit = 1 << (r * NC + c);
      const bool valid = gi >= 0 && gi <= a.rows + 1 && gj >= 0 && gj <= a.cols + 1;
      const bool interior = gi >= 1 && gi <= a.rows && gj >= 1 && gj <= a.cols;
      const int di = gi < by0 ? by0 - gi : (gi >= by1 ? gi - by1 + 1 : 0);
      const int dj = gj < bx0 ? bx0 - gj : (gj >= bx1 ? gj - bx1 + 1 : 0);
      const int d = max(di, dj);
      const int inner = min(min(gi - by0, by1 - 1 - gi), min(gj - bx0, bx1 - 1 - gj));
      if (valid) m_valid |= bit;
      if (interior && d > 0 && d <= G) m_ring |= bit;
      if (d == 0) m_own |= bit;
      if (d == 0 && inner < G) m_frame |= bit;
    }
  // element offset of the thread's cell (0, 0) from a plane's column-0 pointer
  // (32-bit: grids of this kernel are small)
  const int off0 = (int)((long long)(gi0 - a.g0) * a.pitch) + gj0;
  const int ipitch = (int)a.pitch;
  // initial window from plane A (the current iterate)
#pragma unroll
  for (int r = 0; r < RPW; ++r)
#pragma unroll
    for (int c = 0; c < NC; ++c)
      core.v[r][c] = (m_valid >> (r * NC + c)) & 1u ? a.pa[off0 + r * ipitch + c] : R(0);
  core.edge_w = NC == 2 && lane == 0;
  core.edge_e = NC == 2 && lane == 31 && gj0 + NC - 1 == a.cols;
  if (NC == 2) {
#pragma unroll
    for (int r = 0; r < (NC == 2 ? RPW : 1); ++r) {
      const int gi = gi0 + r;
      const bool row_ok = gi >= 0 && gi <= a.rows + 1;
      core.wring[r] = row_ok && core.edge_w ? a.pa[off0 + r * ipitch - 1] : R(0);
      core.ering[r] = row_ok && core.edge_e ? a.pa[off0 + r * ipitch + NC] : R(0);
    }
  }

  if (CPS == 1 && single) {
    // ---- one CTA: Algorithm 1's loop [P:301-331] on the register-resident grid
    core.prime(xb, NW, warp, lane);
    long long k = 1, checks = 0;
    double last = 0.0;
    int converged = 0;
    for (; k <= a.n_iter; ++k) {
      const bool check = a.solve ? (k % a.K == 0) : (a.check_last && k == a.n_iter);
      unsigned long long dmax = 0ull;
      if (check) {
        core.template half<0, true>(xb, NW, warp, lane, 0, a.w, dmax);
        core.template half<1, true>(xb, NW, warp, lane, 0, a.w, dmax);
        dmax = cta_umax64_warp(dmax);
        if (lane == 0) wmax[k & 1][warp] = dmax;
        __syncthreads();
        unsigned long long m = lane < NW ? wmax[k & 1][lane] : 0ull;
        m = cta_umax64_warp(m);
        last = __longlong_as_double((long long)m);
        ++checks;
        if (a.solve && last < a.tol) {  // every thread decides the same (strict <)
          converged = 1;
          break;
        }
      } else {
        core.template half<0, false>(xb, NW, warp, lane, 0, a.w, dmax);
        core.template half<1, false>(xb, NW, warp, lane, 0, a.w, dmax);
      }
    }
    DevState* st = a.ctl.st;
    if (threadIdx.x == 0) {
      st->checks += checks;
      if (checks) st->max_change = last;
      if (converged) {
        st->converged = 1;
        st->conv_iter = k;
      }
      st->iters_done = k > a.n_iter ? a.n_iter : k;
      st->stop = 1;
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if ((m_own >> (r * NC + c)) & 1u) a.pa[off0 + r * ipitch + c] = core.v[r][c];
    return;
  }

  // ---- multi-CTA iterate: T-deep passes with neighbour-only exchange
  unsigned long long dmax = 0ull;
  for (int p = 0; p < a.npasses; ++p) {
    const int Tp = p + 1 == a.npasses ? a.t_last : a.T;
    auto mark = [&](int ev) {
      if (a.trace && threadIdx.x == 0 && p < 64) a.trace[((size_t)blockIdx.x * 64 + p) * 8 + ev] = globaltimer_ns();
    };
    mark(0);
    if (p > 0) {
      // the 8 neighbouring blocks' frames of pass p-1: one thread per
      // neighbour acquires its flag, then every thread reloads its ring cells
      // from the plane the frames were stored to (L2)
      if (threadIdx.x < 9 && threadIdx.x != 4) {
        const int ny = by + (int)threadIdx.x / 3 - 1, nx = bx + (int)threadIdx.x % 3 - 1;
        if (ny >= 0 && ny < a.nby && nx >= 0 && nx < a.nbx) {
          const unsigned long long* f = a.flags + 16 * (ny * a.nbx + nx);
          const unsigned long long want = a.seq0 + (unsigned long long)p;
          if (ld_acquire_gpu_u64(f) < want) {
            const unsigned long long t0 = globaltimer_ns();
            unsigned spins = 0;
            while (ld_acquire_gpu_u64(f) < want) {
              if ((++spins & 255u) == 0u && globaltimer_ns() - t0 > 8000000000ull) {
                atomicExch(&a.ctl.st->halo_timeout, 1);
                break;
              }
            }
          }
        }
      }
      __syncthreads();
      const R* src = (p & 1) ? a.pb : a.pa;
#pragma unroll
      for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int c = 0; c < NC; ++c)
          if ((m_ring >> (r * NC + c)) & 1u) core.v[r][c] = __ldcg(src + off0 + r * ipitch + c);
    }
    core.prime(xb, NW, warp, lane);
    mark(1);
    for (int t = 0; t < Tp; ++t) {
      const int e = 2 * (Tp - t) - 1;  // red reach; black: e - 1
      if (a.check_last && p + 1 == a.npasses && t + 1 == Tp) {
        core.template half<0, true>(xb, NW, warp, lane, e, a.w, dmax);
        core.template half<1, true>(xb, NW, warp, lane, e - 1, a.w, dmax);
      } else {
        core.template half<0, false>(xb, NW, warp, lane, e, a.w, dmax);
        core.template half<1, false>(xb, NW, warp, lane, e - 1, a.w, dmax);
      }
    }
    mark(2);
    {
      // the frame (or, after the last pass, the whole block) to the next plane;
      // then release this block's flag (the barrier orders every thread's
      // stores before thread 0's fence and release)
      R* dst = (p & 1) ? a.pa : a.pb;
      const unsigned m_st = p + 1 < a.npasses ? m_frame : m_own;
#pragma unroll
      for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int c = 0; c < NC; ++c)
          if ((m_st >> (r * NC + c)) & 1u) dst[off0 + r * ipitch + c] = core.v[r][c];
      if (p + 1 < a.npasses) {
        __syncthreads();
        // the barrier orders every thread's frame stores before thread 0's
        // release (causality: CTA scope, then GPU scope; a separate
        // __threadfence measured 2 % slower and adds nothing to the ordering)
        if (threadIdx.x == 0)
          st_release_gpu_u64(a.flags + 16 * blockIdx.x, a.seq0 + (unsigned long long)p + 1ull);
      }
    }
    mark(3);
  }
  if (a.check_last) {
    dmax = cta_umax64_warp(dmax);
    if (lane == 0) wmax[0][warp] = dmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m = 0ull;
      for (int k = 0; k < NW; ++k) m = umax64(m, wmax[0][k]);
      contribute(a.ctl, 0, m);
      maybe_finalize(a.ctl);
    }
  }
}

}  // namespace sorb
