// sor_kernels.cuh — sm_100a kernels of the red-black SOR hot path.
//
// Method: arXiv 1401.0763 (P:n = PAPER.md line n).  Per interior cell, Eq. 1
// [§2.1, P:97-100] in the canonical form of include/sor.h:
//     s = (uN+uS)+(uW+uE); a = 0.25*s; r = a - u; u' = u + w*r
// written with __dadd_rn/__dmul_rn (__fadd_rn/__fmul_rn) so no FMA
// contraction or reassociation can change a bit (readings #3-#4).  Colour of
// (g, j) with g the GLOBAL row: red iff (g + j) even [P:149]; red phase first,
// black phase reads the new reds [P:198].  Max-change [P:103, P:319-325] =
// max |u' - u| over owned interior cells, reduced as ordered u64 bits.
//
// Kernels:
//   k1_half_sweep  K1: one colour phase in place (natural layout), one thread
//                  per cell of that colour; 2 launches per iteration.
//   wave_kernel    K3 (T=1) / K4 (T>1): T red+black iterations per HBM pass.
//                  One warp streams a 128-column strip down a band of rows in
//                  registers: src row i+1 enters, stage s (half-sweep s, colour
//                  s&1) updates row i-s, the last stage emits finished row
//                  i-2T+1 to dst.  N/S neighbours are in the lane's own
//                  registers, one of W/E in the lane, the other one lane away
//                  (one shuffle per cell pair).  Strips overlap by 2T columns
//                  and bands by 2T rows of redundant ("ghost") work so warps
//                  never synchronise.  Out-of-place src -> dst, so the result
//                  is bitwise that of the in-place red/black sequence
//                  (DESIGN.md §5.2).
//   k5_small_solve K5: whole grid in one CTA's shared memory; all iterations,
//                  max-change and stop test in one launch.
//   finalize_kernel  stop test after a cross-slab (virtual / NCCL) max.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace sorb {

constexpr int kColPad = 32;   // storage columns left of global column 0
constexpr int kRowPad = 24;   // storage rows above/below a slab's owned rows + halo
constexpr int kWaveWarps = 4; // warps per CTA in wave_kernel (independent warps)
constexpr int kWaveNC = 4;     // columns per lane in wave_kernel (strip = 32*kWaveNC columns)

constexpr int kMaxT = 6;      // max temporal depth (iterations per HBM pass; > kMaxTLink: one slab, SOR only)
constexpr int kMaxTLink = 4;  // max depth of multi-slab handles, Jacobi and the skew-1 / persistent kernels

// Wave-kernel build options (A/B experiments; the defaults are the product):
// SOR_WAVE_HOIST issues every stage's lane-neighbour shuffle at the start of
// a step instead of just before the stage.
#ifndef SOR_WAVE_HOIST
#define SOR_WAVE_HOIST 0
#endif

struct DevState {
  // ordered bits of max |delta| per iteration of a pass, in two slot sets
  // (consecutive passes of a deferred solve alternate); one 128-B line each
  // so the per-CTA atomics of different slots hit different L2 slices
  unsigned long long maxbits[2][kMaxT][16];
  unsigned int ticket;         // finishing-part counter for the fused finalize
  int stop;                    // solve: converged or maxit reached -> later launches exit
  int converged;
  int conv_t;                  // index within its pass of the converging iteration
  int ambiguous;               // ck=3: a hi-word max tied with tol's; host resolves exactly
  long long amb_iter;
  long long iters_done;        // iterations finished in this call
  long long conv_iter;
  long long checks;
  double max_change;           // last checked max-change
  int halo_timeout;            // a halo wait gave up (dist: a peer never released its rows)
};

// ---------------------------------------------------------------- multi-GPU
// Per-rank communication block (device memory, mapped by the other ranks of a
// dist handle over CUDA IPC; SURVEY 8(e) path B).  `done`/`pub` join the
// per-rank max-changes of a checked pass (E2): a rank publishes its local
// maxima of pass `seq` in pub[seq & 1] and then releases done = seq; every
// rank reads all ranks' pub once their done >= seq.  The halo flags follow the
// header in the same allocation: top[nflags] (released by rank-1 after it
// pushed its last rows into this rank's top halo) and bot[nflags] (rank+1).
constexpr int kMaxRanks = 8;  // one NVSwitch node
struct DistComm {
  unsigned long long done;
  unsigned long long pad0[15];
  unsigned long long pub[2][kMaxT];
  unsigned long long pad1[16 - (2 * kMaxT) % 16];
};
struct DistJoinTab {           // device-resident: every rank's comm block, mapped
  DistComm* comm[kMaxRanks];
  int nranks, rank;
};

// Loop control of one launch (a pass of `T` iterations ending at k_last).
struct IterCtl {
  DevState* st;         // nullptr: no max-change, no loop control
  long long k_last;     // 1-based index (in this call) of the pass's last iteration
  long long maxit;
  long long K;          // check_every (solve)
  double tol;
  int T;                // iterations in this pass
  int ck;               // 0: no max-change; 1: exact, of iteration k_last; 2: exact, of every
                        // iteration; 3: high 32 bits only, of every iteration (stop decision
                        // exact unless the high words tie with tol's -> ambiguous); 4: as 3 on
                        // a probe subset (1/6 of the rows): a lower bound, so "probe >= tol"
                        // proves "not converged" and anything else is resolved exactly
  unsigned int tol_hi;  // high 32 bits of tol (ck=3)
  int solve;            // apply the stop test / early exit
  int finalize;         // this launch's last part runs the stop test (ticket)
  unsigned int nparts;  // number of ticket takers (warps or CTAs) in this launch
  int set;              // maxbits slot set this launch contributes to
  // Deferred stop test (wave kernel, single slab, solve): no ticket; block 0
  // of this launch runs the stop test of the PREVIOUS pass (prev_*, slot set
  // set^1) while the other blocks compute this pass speculatively into the
  // third plane.  The launch after it exits early if that test stopped.
  int defer;
  int prev_valid;
  int prev_T, prev_ck, prev_set;
  long long prev_k_last;
  // Cross-rank join of the maxima (dist over IPC): 0 none (one DevState sees
  // every slab), 1 publish + wait + combine (concurrent ranks), 2 publish
  // only, 3 combine only (lockstep ranks sharing a GPU: a host barrier runs
  // between 2 and 3, so no kernel ever waits on another process).
  const DistJoinTab* join;
  int join_mode;
  unsigned long long seq;       // this pass's sequence number (halo flags, join)
  unsigned long long prev_seq;  // sequence number of the pass the decision block decides
};

__host__ __device__ __forceinline__ int floordiv6(int x) { return x >= 0 ? x / 6 : -((5 - x) / 6); }

// ---------------------------------------------------------------- arithmetic
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double rdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float rdiv(float a, float b) { return __fdiv_rn(a, b); }

// s/6 correctly rounded (reading N3-1) without the division routine: the
// quotient q0 = RN(s*RN(1/6)) is corrected once with its exact remainder
// r = s - 6*q0 (an FMA), q = RN(q0 + r*RN(1/6)) (Markstein).  Verified equal
// to the IEEE division for every float32 with a normal quotient (exhaustive)
// and 5e8 random float64 (tools/div6_check.c).  Below that range (|s| <
// 1.5*2^-1020, zeros included) s is an integer k of units 2^-1074 (2^-149
// for fp32) and the quotient is subnormal: RN(s/6) = k/6 rounded to nearest
// even in the same units, which is its bit pattern (tools/div6_tiny_check.c:
// exhaustive for fp32, every k < 2^24 and 5e8 random values for fp64).  Inf
// and NaN return s.  The FMAs here are the algorithm, not a contraction of
// the canonical update.  (The integer path replaces a call of the division
// routine, which the diffusion front of a zero-initialised grid, full of
// subnormal values, used to take on every warp it crossed.)
static __device__ __noinline__ double div6_tiny(double s) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(s);
  const unsigned long long sign = b & 0x8000000000000000ull, a = b ^ sign;
  if (a >= 0x7ff0000000000000ull) return s;  // inf, NaN
  const unsigned long long E = a >> 52, m = a & 0xfffffffffffffull;
  const unsigned long long k = E == 0 ? m : ((0x10000000000000ull | m) << (E - 1));
  unsigned long long q = k / 6ull;
  const unsigned long long r = k - 6ull * q;
  if (r > 3ull || (r == 3ull && (q & 1ull))) ++q;
  return __longlong_as_double((long long)(sign | q));
}
static __device__ __noinline__ float div6_tiny(float s) {
  const unsigned b = __float_as_uint(s);
  const unsigned sign = b & 0x80000000u, a = b ^ sign;
  if (a >= 0x7f800000u) return s;  // inf, NaN
  const unsigned E = a >> 23, m = a & 0x7fffffu;
  const unsigned k = E == 0 ? m : ((0x800000u | m) << (E - 1));
  unsigned q = k / 6u;
  const unsigned r = k - 6u * q;
  if (r > 3u || (r == 3u && (q & 1u))) ++q;
  return __uint_as_float(sign | q);
}
__device__ __forceinline__ double div6(double s) {
  const double yi = 1.0 / 6.0;
  const double q0 = __dmul_rn(s, yi);
  const double r = __fma_rn(-q0, 6.0, s);
  const double q1 = __fma_rn(r, yi, q0);
  const unsigned long long a = (unsigned long long)__double_as_longlong(s) & 0x7fffffffffffffffull;
  // normal range: |s| in [0x1.8p-1020, DBL_MAX]; zeros (a zero-initialised
  // interior is full of them) keep their sign without the integer path
  if (a - 0x0038000000000000ull <= 0x7fefffffffffffffull - 0x0038000000000000ull) return q1;
  if (a == 0ull) return s;
  return div6_tiny(s);
}
__device__ __forceinline__ float div6(float s) {
  const float yi = 1.0f / 6.0f;
  const float q0 = __fmul_rn(s, yi);
  const float r = __fmaf_rn(-q0, 6.0f, s);
  const float q1 = __fmaf_rn(r, yi, q0);
  const unsigned a = __float_as_uint(s) & 0x7fffffffu;
  // normal range: |s| in [0x1.8p-124, FLT_MAX]; zeros keep their sign
  if (a - 0x01c00000u <= 0x7f7fffffu - 0x01c00000u) return q1;
  if (a == 0u) return s;
  return div6_tiny(s);
}

// Eq. 1, BJ form, canonical order.  ns = uN+uS and we = uW+uE are formed by the
// caller (addition is commutative, so which operand is W and which E is moot).
template <typename R>
__device__ __forceinline__ R sor_update(R ns, R we, R u, R w) {
  const R s = radd(ns, we);
  const R a = rmul(R(0.25), s);
  const R r = rsub(a, u);
  return radd(u, rmul(w, r));
}

// Same, also returning the correction p = w*r (u' = u + p).
template <typename R>
__device__ __forceinline__ R sor_update_p(R ns, R we, R u, R w, R& p) {
  const R s = radd(ns, we);
  const R a = rmul(R(0.25), s);
  const R r = rsub(a, u);
  p = rmul(w, r);
  return radd(u, p);
}

// |u' - u| as ordered u64 bits; fp32 widened exactly first.
__device__ __forceinline__ unsigned long long delta_bits(double un, double u) {
  return (unsigned long long)__double_as_longlong(fabs(rsub(un, u)));
}
__device__ __forceinline__ unsigned long long delta_bits(float un, float u) {
  return (unsigned long long)__double_as_longlong((double)fabsf(rsub(un, u)));
}
__device__ __forceinline__ int hi_bits(double x) { return __double2hiint(x); }
__device__ __forceinline__ int hi_bits(float x) { return __double2hiint((double)x); }
__device__ __forceinline__ unsigned int max3u(unsigned int a, unsigned int b, unsigned int c) {
  return max(a, max(b, c));
}
__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = umax64(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

__device__ __forceinline__ int ld_stop(const DevState* st) {
  return *reinterpret_cast<const volatile int*>(&st->stop);
}

// Stop test of Algorithm 1 [P:319-331] for the iterations of one pass (T
// iterations ending at k_last, max-change mode ck); their maxima are complete
// in st->maxbits[set].  Strict '<' (reading #7).
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Spin (one thread) until *p >= v; gives up after ~8 s and reports it (a peer
// that never releases must not hang the GPU).
__device__ __forceinline__ bool wait_geq_sys(const unsigned long long* p, unsigned long long v, DevState* st) {
  if (ld_acquire_sys(p) >= v) return true;
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_sys(p) < v) {
    __nanosleep(100);
    if (globaltimer_ns() - t0 > 8000000000ull) {
      if (st) atomicExch(&st->halo_timeout, 1);
      return false;
    }
  }
  return true;
}

// E2 over IPC: publish this rank's maxima of pass `seq` (slot set `set`) and/or
// fold every rank's published maxima into them (join_mode, see IterCtl).
__device__ __forceinline__ void join_maxima(DevState* st, const IterCtl& ctl, int set, unsigned long long seq) {
  if (!ctl.join || ctl.join_mode == 0) return;
  const DistJoinTab& J = *ctl.join;
  DistComm* mine = J.comm[J.rank];
  if (ctl.join_mode == 1 || ctl.join_mode == 2) {
    for (int t = 0; t < kMaxT; ++t) mine->pub[seq & 1][t] = st->maxbits[set][t][0];
    __threadfence_system();
    st_release_sys(&mine->done, seq);
  }
  if (ctl.join_mode == 1 || ctl.join_mode == 3) {
    for (int q = 0; q < J.nranks; ++q) {
      if (q == J.rank) continue;
      DistComm* c = J.comm[q];
      wait_geq_sys(&c->done, seq, st);
      for (int t = 0; t < kMaxT; ++t) {
        const unsigned long long v = *reinterpret_cast<volatile unsigned long long*>(&c->pub[seq & 1][t]);
        if (v > st->maxbits[set][t][0]) st->maxbits[set][t][0] = v;
      }
    }
  }
}

__device__ __forceinline__ void finalize_pass(DevState* st, const IterCtl& ctl, long long k_last, int T, int ck,
                                              int set, unsigned long long seq) {
  join_maxima(st, ctl, set, seq);
  if (ctl.join_mode == 2) return;  // lockstep: the decision runs after the host barrier
  const long long k0 = k_last - (T - 1);
  st->ticket = 0u;
  for (int t = 0; t < T; ++t) {
    const long long k = k0 + t;
    const bool every = ck >= 2;
    const int slot = every ? t : 0;
    const bool checked = every ? (!ctl.solve || k % ctl.K == 0) : (t == T - 1);
    if (!checked) continue;
    if (ck >= 3) {
      // non-negative doubles order like their bit patterns: a smaller high
      // word decides '<', a larger one '>='; equal high words are ambiguous
      const unsigned int h = (unsigned int)(st->maxbits[set][slot][0] >> 32);
      st->checks += 1;
      st->iters_done = k;
      st->max_change = __longlong_as_double((long long)((unsigned long long)h << 32));
      if (ck == 4) {
        // probe max <= full max: only "probe > tol" is conclusive
        if (h <= ctl.tol_hi) {
          st->ambiguous = 1;
          st->amb_iter = k;
          st->stop = 1;
          break;
        }
        continue;
      }
      if (h < ctl.tol_hi) {
        st->converged = 1;
        st->conv_iter = k;
        st->conv_t = t;
        st->stop = 1;
        break;
      }
      if (h == ctl.tol_hi) {
        st->ambiguous = 1;
        st->amb_iter = k;
        st->stop = 1;
        break;
      }
      continue;
    }
    const double m = __longlong_as_double((long long)st->maxbits[set][slot][0]);
    st->checks += 1;
    st->max_change = m;
    st->iters_done = k;
    if (ctl.solve && m < ctl.tol) {
      st->converged = 1;
      st->conv_iter = k;
      st->conv_t = t;
      st->stop = 1;
      break;
    }
  }
  for (int t = 0; t < kMaxT; ++t) st->maxbits[set][t][0] = 0ull;
  if (ctl.solve && k_last >= ctl.maxit) st->stop = 1;
  __threadfence();
}
__device__ __forceinline__ void finalize_pass(DevState* st, const IterCtl& ctl) {
  finalize_pass(st, ctl, ctl.k_last, ctl.T, ctl.ck, ctl.set, ctl.seq);
}

// One part (warp or CTA) contributes its maxima; the last part finalizes.
__device__ __forceinline__ void contribute(const IterCtl& ctl, int slot, unsigned long long bits) {
  if (bits) atomicMax(&ctl.st->maxbits[ctl.set][slot][0], bits);
}
__device__ __forceinline__ void maybe_finalize(const IterCtl& ctl) {
  if (ctl.finalize) {
    __threadfence();
    const unsigned int t = atomicAdd(&ctl.st->ticket, 1u);
    if (t == ctl.nparts - 1u) {
      __threadfence();
      finalize_pass(ctl.st, ctl);
    }
  }
}

static __global__ void finalize_kernel(IterCtl ctl) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (ctl.solve && ld_stop(ctl.st)) return;
    finalize_pass(ctl.st, ctl);
  }
}

// ---------------------------------------------------------------- K1
// One colour phase (updateGridRed / updateGridBlack) over owned
// global rows [r_lo, r_hi), in place.  Code 2's stride-2 form:
// thread t of row g updates column j0(g) + 2t, no parity branch per cell.
template <typename R, bool CHECK>
__global__ void __launch_bounds__(256) k1_half_sweep(R* base, long long pitch, long long g0,
                                                     long long rows, long long cols,
                                                     long long r_lo, long long r_hi, int color,
                                                     R w, IterCtl ctl) {
  if (ctl.st && ctl.solve && ld_stop(ctl.st)) return;
  unsigned long long dmax = 0ull;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long g = r_lo + blockIdx.y; g < r_hi; g += gridDim.y) {
    const long long j = ((((g + 1) & 1) == color) ? 1 : 2) + 2 * t;
    if (j <= cols && g >= 1 && g <= rows) {
      const R* up = base + (g - 1 - g0) * pitch;
      R* uc = base + (g - g0) * pitch;
      const R* dn = base + (g + 1 - g0) * pitch;
      const R u = uc[j];
      const R un = sor_update(radd(up[j], dn[j]), radd(uc[j - 1], uc[j + 1]), u, w);
      if (CHECK) dmax = umax64(dmax, delta_bits(un, u));
      uc[j] = un;
    }
  }
  if (CHECK) {
    dmax = warp_max_u64(dmax);
    __shared__ unsigned long long wmax[8];
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = dmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m = 0ull;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) m = umax64(m, wmax[k]);
      contribute(ctl, 0, m);
      maybe_finalize(ctl);
    }
  }
}

// ---------------------------------------------------------------- K3 / K4
// The two tensor maps of a source plane (6-row and 2-row boxes), passed by
// value as one __grid_constant__ kernel parameter.
struct WaveMaps {
  CUtensorMap m[2];
};

// Device-initiated halo exchange (SURVEY 8(e) path B): the tiles that finish
// a slab's first / last H owned rows also store them into the neighbouring
// slab's destination plane (a CUDA-IPC mapping of another GPU's memory, or
// another slab of a virtual grid) and then release that neighbour's flag of
// their strip with this pass's sequence number.  The tiles whose results
// depend on halo rows wait for the flags of every producer strip whose tile
// reads or writes their columns (RAW for the halo, WAR for the plane they
// are about to push into), so interior tiles never wait and no global
// barrier or copy kernel separates two passes.
struct HaloLink {
  long long up_off, dn_off;       // elements from this slab's dst cell to the same cell in the
                                  // upper / lower neighbour's dst plane
  unsigned long long* rel_up;     // upper neighbour's bottom-halo flags (indexed by our strip)
  unsigned long long* rel_dn;     // lower neighbour's top-halo flags
  const unsigned long long* acq_top;  // our top-halo flags (released by the upper neighbour)
  const unsigned long long* acq_bot;  // our bottom-halo flags
  unsigned long long seq;         // released value (this pass)
  unsigned long long need;        // wait until flags >= need
  int H;                          // rows pushed per side (>= the halo any pass reads)
  int pg, pw, pgh, pn;            // producer strip layout of the awaited pass: strip s owns
                                  // [pg + s*pw, pg + (s+1)*pw), reads pgh columns more per side;
                                  // pn strips
  int on;                         // 0: no link (single slab / host-side exchange)
};

__host__ __device__ __forceinline__ int floordiv_i(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// Lane 0 of the tile's streaming warp: wait for the producer strips whose
// tiles touch columns [c_a, c_b) (their owned range widened by pgh).
__device__ __forceinline__ void halo_wait(const unsigned long long* flags, const HaloLink& L, int c_a, int c_b,
                                          DevState* st) {
  const int s_a = max(0, floordiv_i(c_a - L.pgh - L.pg, L.pw));
  const int s_b = min(L.pn - 1, floordiv_i(c_b + L.pgh - 1 - L.pg, L.pw));
  for (int s = s_a; s <= s_b; ++s)
    if (!wait_geq_sys(flags + s, L.need, st)) return;
}

// The storing warp of a tile, after the tile: copy its owned cells of rows
// [max(R0, lo), min(R1, hi)) from the local dst plane (written by this same
// lane, so program order makes them visible) to the neighbour, then release.
template <typename R, int NC>
__device__ __forceinline__ void halo_push_rows(R* dst, long long g0, long long pitch, long long off, int c0,
                                               int own_lo, int own_hi, int ra, int rb, int lane,
                                               unsigned long long* flag, unsigned long long seq) {
  for (int r = ra; r < rb; ++r) {
    const R* src = dst + (long long)(r - g0) * pitch + c0;
#pragma unroll
    for (int h = 0; h < NC / 2; ++h) {
      const int cp = c0 + 2 * h;
      if (cp >= own_lo && cp + 1 < own_hi) {
        const R x = src[2 * h], y = src[2 * h + 1];
        R* q = dst + (long long)(r - g0) * pitch + c0 + off + 2 * h;
        q[0] = x;
        q[1] = y;
      }
    }
  }
  __threadfence_system();
  __syncwarp();
  if (lane == 0) st_release_sys(flag, seq);
}

template <typename R>
struct WaveArgs {
  const R* src;      // column 0 of storage row 0 (plane + kColPad)
  R* dst;
  long long pitch;   // elements
  long long g0;      // global row of storage row 0
  long long rows, cols;
  long long r_lo, r_hi;  // owned global rows written by this launch
  const int4* tiles;  // per tile: (strip, R0, R1, unused) — see wave_tiles
  int ntiles;
  int s0;            // first column of strip 0 (multiple of 4)
  R w;
  HaloLink link;     // device-initiated halo exchange (multi-slab)
};

// A tile whose owned rows lie within `need_rows` of the slab edge depends on
// the halo: its streaming warp waits before the first TMA of source rows.
template <typename R>
__device__ __forceinline__ void tile_halo_wait(const WaveArgs<R>& a, int sw, int wc, int R0, int R1, int need_rows,
                                               int lane, DevState* st) {
  const HaloLink& L = a.link;
  if (!L.on) return;
  const bool top = L.acq_top != nullptr && R0 < a.r_lo + need_rows;
  const bool bot = L.acq_bot != nullptr && R1 > a.r_hi - need_rows;
  if (!(top || bot)) return;
  if (lane == 0) {
    if (top) halo_wait(L.acq_top, L, sw, sw + wc, st);
    if (bot) halo_wait(L.acq_bot, L, sw, sw + wc, st);
    // the rows were written through the generic proxy (peer stores); the
    // tile reads them with TMA (async proxy)
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncwarp();
}
// The storing warp of a tile that finished rows within H of the slab edge
// pushes them (its owned columns: the strip minus `ghost` per side).  The
// tiler gives every strip exactly one such tile per side (sor_api.cu).
template <typename R, int NC>
__device__ __forceinline__ void tile_halo_push(const WaveArgs<R>& a, int sw, int wc, int ghost, int strip, int R0,
                                               int R1, int lane) {
  const HaloLink& L = a.link;
  if (!L.on) return;
  const int c0 = sw + NC * lane;
  const int own_lo = sw + ghost, own_hi = sw + wc - ghost;
  const int lo = (int)a.r_lo, hi = (int)a.r_hi;
  if (L.rel_up != nullptr && R0 < lo + L.H)
    halo_push_rows<R, NC>(a.dst, a.g0, a.pitch, L.up_off, c0, own_lo, own_hi, R0, min(R1, lo + L.H), lane,
                          L.rel_up + strip, L.seq);
  if (L.rel_dn != nullptr && R1 > hi - L.H)
    halo_push_rows<R, NC>(a.dst, a.g0, a.pitch, L.dn_off, c0, own_lo, own_hi, max(R0, hi - L.H), R1, lane,
                          L.rel_dn + strip, L.seq);
}

__device__ __forceinline__ void ldg4(const double* p, double (&x)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3])
               : "l"(p));
}
__device__ __forceinline__ void ldg4(const float* p, float (&x)[4]) {
  asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3])
               : "l"(p));
}
__device__ __forceinline__ void stg4(double* p, const double (&x)[4]) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(x[0]), "d"(x[1]),
               "d"(x[2]), "d"(x[3])
               : "memory");
}
__device__ __forceinline__ void stg4(float* p, const float (&x)[4]) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(x[0]), "f"(x[1]),
               "f"(x[2]), "f"(x[3])
               : "memory");
}

// Lane shuffles by one without the convergence check __shfl_*_sync inserts
// (the warp is converged by construction at every call site).
__device__ __forceinline__ double shfl_up1(double v) {
  int lo = __double2loint(v), hi = __double2hiint(v);
  asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, -1;" : "+r"(lo));
  asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, -1;" : "+r"(hi));
  return __hiloint2double(hi, lo);
}
__device__ __forceinline__ double shfl_dn1(double v) {
  int lo = __double2loint(v), hi = __double2hiint(v);
  asm volatile("shfl.sync.down.b32 %0, %0, 1, 31, -1;" : "+r"(lo));
  asm volatile("shfl.sync.down.b32 %0, %0, 1, 31, -1;" : "+r"(hi));
  return __hiloint2double(hi, lo);
}
__device__ __forceinline__ float shfl_up1(float v) {
  asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, -1;" : "+f"(v));
  return v;
}
__device__ __forceinline__ float shfl_dn1(float v) {
  asm volatile("shfl.sync.down.b32 %0, %0, 1, 31, -1;" : "+f"(v));
  return v;
}

// ---- TMA bulk-copy ring (cp.async.bulk + mbarrier), one ring per warp
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// 2-D tensor TMA of a box of rows x one warp strip (tensor maps built by the
// host over the whole storage plane, see make_tmaps in sor_api.cu); x, y =
// storage column and row of the box corner.  (A 4-D view that interleaves
// lanes' 16-B chunks in shared memory avoids the 2-way bank conflicts of the
// row-major box but measured 25% slower end to end: 16-B inner boxes are slow
// to fetch.)
__device__ __forceinline__ void tma_rows(uint32_t dst, const CUtensorMap* tm, int x, int y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(tm), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Generic shared-memory vector moves of N values (N even), 16-B aligned.
template <int N>
__device__ __forceinline__ void ldsN(const double* p, double (&x)[N]) {
#pragma unroll
  for (int k = 0; k < N / 2; ++k) {
    const double2 v = reinterpret_cast<const double2*>(p)[k];
    x[2 * k] = v.x;
    x[2 * k + 1] = v.y;
  }
}
template <int N>
__device__ __forceinline__ void ldsN(const float* p, float (&x)[N]) {
  if (N % 4 == 0) {
#pragma unroll
    for (int k = 0; k < N / 4; ++k) {
      const float4 v = reinterpret_cast<const float4*>(p)[k];
      x[4 * k] = v.x; x[4 * k + 1] = v.y; x[4 * k + 2] = v.z; x[4 * k + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
      const float2 v = reinterpret_cast<const float2*>(p)[k];
      x[2 * k] = v.x;
      x[2 * k + 1] = v.y;
    }
  }
}
template <int N>
__device__ __forceinline__ void stsN(double* p, const double (&x)[N]) {
#pragma unroll
  for (int k = 0; k < N / 2; ++k) reinterpret_cast<double2*>(p)[k] = make_double2(x[2 * k], x[2 * k + 1]);
}
template <int N>
__device__ __forceinline__ void stsN(float* p, const float (&x)[N]) {
  if (N % 4 == 0) {
#pragma unroll
    for (int k = 0; k < N / 4; ++k)
      reinterpret_cast<float4*>(p)[k] = make_float4(x[4 * k], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < N / 2; ++k) reinterpret_cast<float2*>(p)[k] = make_float2(x[2 * k], x[2 * k + 1]);
  }
}

// Wave-kernel geometry.  NC columns per lane (4, 6 or 8), so a warp strip is
// 32*NC columns; a lane holds NH = NC/2 cells of each colour per row.
template <int NC>
__host__ __device__ constexpr int wave_cols() { return 32 * NC; }

// Shared memory of one tile's source ring: 2 batches of 6 source rows and the
// 2 prologue rows (NST = 14 slots of 32*NC values, row-major), then 3
// mbarriers (one per batch, one for the prologue).
template <typename R, int NST, int NC>
__host__ __device__ constexpr int wave_smem_per_warp() {
  return (NST * wave_cols<NC>() * (int)sizeof(R) + 3 * 8 + 127) / 128 * 128;  // 128-B aligned bases
}
// Split mode: a warp PAIR shares one tile.  The front warp streams the source
// and runs stages [0, T), the back warp runs stages [T, 2T); per step the
// front hands over stage T-1's new row and stage T-2's row of two steps ago
// (NC values per lane) through a 2-batch shared ring synchronised with named
// barriers.  Half the registers per warp -> twice the resident warps.
template <typename R, int NC>
__host__ __device__ constexpr int wave_handoff_bytes() {
  return 2 * 6 * 32 * NC * (int)sizeof(R);  // 2 batches x 6 steps x 32 lanes x NC values
}
template <typename R, int NST, int NC>
__host__ __device__ constexpr int wave_smem_per_pair() {
  return wave_smem_per_warp<R, NST, NC>() + wave_handoff_bytes<R, NC>();
}

// Predicated stores (branch-free, so unrolled steps form one basic block).
__device__ __forceinline__ void stg4_if(bool p, double* a, double x0, double x1, double x2, double x3) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n @q st.global.v4.f64 [%0], {%1,%2,%3,%4};\n}" ::"l"(a),
               "d"(x0), "d"(x1), "d"(x2), "d"(x3), "r"((int)p)
               : "memory");
}
__device__ __forceinline__ void stg4_if(bool p, float* a, float x0, float x1, float x2, float x3) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n @q st.global.v4.f32 [%0], {%1,%2,%3,%4};\n}" ::"l"(a),
               "f"(x0), "f"(x1), "f"(x2), "f"(x3), "r"((int)p)
               : "memory");
}
__device__ __forceinline__ void stg2_if(bool p, double* a, double x, double y) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q st.global.v2.f64 [%0], {%1,%2};\n}" ::"l"(a), "d"(x),
               "d"(y), "r"((int)p)
               : "memory");
}
__device__ __forceinline__ void stg2_if(bool p, float* a, float x, float y) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q st.global.v2.f32 [%0], {%1,%2};\n}" ::"l"(a), "f"(x),
               "f"(y), "r"((int)p)
               : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Register pipeline of one warp.
//
// Lane columns c0..c0+NC-1 (q = 0..NC-1), c0 = s_w + NC*lane.  Step m has
// front row i = i_first + m; it consumes source row i+1 and stage s
// (half-sweep s of the pass, colour s&1) updates row i-s.  With O = i & 1
// (= m & 1), the cells of stage s in row i-s sit at q = O + 2h, h < NH; a
// stage keeps only its own colour ("compact" v[h] <-> q = O+2h of the step
// that made it).  Rows are held in 3-slot rings indexed by (step mod 3), so
// with the loop unrolled 6 ways (parity x ring phase) every register index is
// static and no value is ever moved.  Source rows arrive through an NST-deep
// shared ring filled by TMA, 6 rows per box.
//
// This warp runs stages [SB, SE) of the S = 2T stages: SB == 0 streams the
// source; SB > 0 receives stage SB-1's new row and stage SB-2's row of two
// steps ago from the front warp; SE < S hands the same on; SE == S writes
// finished rows.
//
// CK: 0 = no max-change, 1 = of the pass's last iteration, 2 = of each,
// 3 = high 32 bits of |delta| of each (VIMNMX3), 4 = as 3 on probe rows.
// Masking (cells that must keep their value: the Dirichlet ring and the
// padding around it) is chosen per 6-step batch, warp-uniformly: MK = 0 when
// every cell the batch updates is interior, 1 when only columns of an edge
// strip need it (a lane-constant select), 2 when the batch also updates a ring
// or padding row (first/last batches of the top/bottom bands).  Ownership
// (which computed cells are valid and written: the strip minus its 2T ghost
// columns on each side, the band's rows) applies to every warp.
template <typename R, int T, int NST, int CK, int SB, int SE, int NC>
struct WavePipe {
  static constexpr int S = 2 * T;  // stages (half-sweeps) per pass
  static constexpr int NH = NC / 2;
  static constexpr int WC = wave_cols<NC>();
  static constexpr int NSLOT = CK >= 2 ? T : 1;
  // ghost bands (2T columns) cover whole lanes: one ownership flag per lane
  static constexpr bool LANE_OWN = (2 * T) % NC == 0;
  // CK 4 probes the red stage (s even) of each iteration on the rows with
  // (row - i_first) % 6 == 0: in the 6-step unrolled loop that is the
  // compile-time condition (M6 - s) % 6 == 0.  A lower bound of the
  // iteration's max-change, as the probe must be.
  __host__ __device__ static constexpr bool probe_row(int M6, int s) { return ((M6 - s) % 6 + 6) % 6 == 0; }
  R F[3][NC];                 // source rows, slot = (row - (i_first-1)) % 3 (front warp)
  R C[S - 1][3][NH];          // stage outputs, slot = step % 3 (unused stages vanish)
  unsigned long long dmax[CK == 1 || CK == 2 ? NSLOT : 1];  // CK 1, 2: ordered bits
  unsigned int hmax[CK >= 3 ? NSLOT : 1];                     // CK 3, 4: high words
  unsigned int ownM[NH];           // CK 3/4: 0x7fffffff if column pair h is owned
  unsigned int pf[2];              // CK 4: all-ones iff this batch's probe row 0 / 1 is owned
  bool upd[NC];
  bool ownP[NH];                   // column pair (q=2h, 2h+1) owned by position (see wave_tile)
  int rows, R0, R1;
  int col_mask;                    // 1: edge strip (ring/padding columns), else 0
  R* orow;                         // back: dst address of the row stage S-1 finishes at this step
  // ring: row n >= 2 in batch j = (n-2)/6, slot (j&1)*6 + (n-2)%6, barrier
  // j&1 (phase (j>>1)&1); rows n = 0,1 (prologue) first use slots 10, 11
  const R* ring;
  uint32_t ring_s, bar_s;
  const CUtensorMap* tm;      // tensor maps of the source plane (6-row and 2-row boxes);
  const CUtensorMap* tm2;     // (tm_x, tm_y) = storage (column, row) of (i_first-1, s_w)
  int tm_x, tm_y;
  long long pitch;
  int nbatch;
  int lane;
  R* hand;                    // split: handoff ring [2][6][32][NC]
  int bar_full, bar_empty;    // split: named barrier ids (+ batch parity)
  static constexpr uint32_t ROWB = WC * sizeof(R);
  static constexpr int CH = 16 / (int)sizeof(R);  // values per 16-B chunk

  // lane 0: the 6 rows of batch j as one tensor-TMA box (rows 2+6j .. 7+6j
  // counted from i_first-1)
  __device__ __forceinline__ void issue_batch_tma(int j) {
    const uint32_t bar = bar_s + 8u * (j & 1);
    mbar_expect_tx(bar, 6 * ROWB);
    tma_rows(ring_s + (j & 1) * 6 * ROWB, tm, tm_x, tm_y + 6 * j + 2, bar);
  }
  // lane 0: rows i_first-1, i_first into slots 12, 13 (2-row box)
  __device__ __forceinline__ void issue_prologue() {
    const uint32_t bar = bar_s + 16u;
    mbar_expect_tx(bar, 2 * ROWB);
    tma_rows(ring_s + 12 * ROWB, tm2, tm_x, tm_y, bar);
  }
  // this lane's NC values of one row in a ring slot
  __device__ __forceinline__ void ld_row(const R* row, R (&x)[NC]) { ldsN<NC>(row + NC * lane, x); }

  // Handoff ring layout [batch][step][16-B chunk][lane]: a warp's access to
  // one chunk is 512 contiguous bytes (no bank conflicts).
  __device__ __forceinline__ void hand_st(R* hp, int M6, const R (&x)[NC]) {
#pragma unroll
    for (int k = 0; k < NC / CH; ++k) {
      R* q = hp + ((M6 * (NC / CH) + k) * 32 + lane) * CH;
      if (sizeof(R) == 8)
        *reinterpret_cast<double2*>(q) = make_double2((double)x[2 * k], (double)x[2 * k + 1]);
      else
        *reinterpret_cast<float4*>(q) = make_float4((float)x[4 * k], (float)x[4 * k + 1], (float)x[4 * k + 2], (float)x[4 * k + 3]);
    }
  }
  __device__ __forceinline__ void hand_ld(const R* hp, int M6, R (&x)[NC]) {
#pragma unroll
    for (int k = 0; k < NC / CH; ++k) {
      const R* q = hp + ((M6 * (NC / CH) + k) * 32 + lane) * CH;
      if (sizeof(R) == 8) {
        const double2 v = *reinterpret_cast<const double2*>(q);
        x[2 * k] = (R)v.x;
        x[2 * k + 1] = (R)v.y;
      } else {
        const float4 v = *reinterpret_cast<const float4*>(q);
        x[4 * k] = (R)v.x; x[4 * k + 1] = (R)v.y; x[4 * k + 2] = (R)v.z; x[4 * k + 3] = (R)v.w;
      }
    }
  }

  template <int MK, int M6>
  __device__ __forceinline__ void step(const WaveArgs<R>& a, int i, const R* rowp, R* hp) {
    constexpr int O = M6 & 1;
    constexpr int PH = M6 % 3;          // slot of age 0 (this step)
    constexpr int P1 = (PH + 2) % 3;    // age 1
    constexpr int P2 = (PH + 1) % 3;    // age 2
    if (SB == 0) {
      ld_row(rowp + M6 * WC, F[P1]);  // source row i+1
    } else {
      // stage SB-1's row i-SB+1 of this step, stage SB-2's row i-SB of two
      // steps ago (used only as the old value of stage SB's cells)
      R x[NC];
      hand_ld(hp, M6, x);
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        C[SB - 1][PH][h] = x[h];
        if (SB >= 2) C[SB >= 2 ? SB - 2 : 0][P2][h] = x[NH + h];
      }
    }
    // CK 3: bit s set iff stage s's row i-s is owned (R0 <= i-s < R1)
    unsigned int rowm = 0u;
    if (CK == 3) {
      const int lo_s = max(0, i - R1 + 1), hi_s = min(S - 1, i - R0);
      rowm = hi_s >= lo_s ? (((2u << hi_s) - 1u) & ~((1u << lo_s) - 1u)) : 0u;
    }
#if SOR_WAVE_HOIST
    // the lane-neighbour values every stage of this step needs were produced
    // at the previous step: issue all shuffles first, off the stages'
    // critical path (a shuffle's latency is ~24 cycles on sm_100a)
    R nbs[SE - SB];
#pragma unroll
    for (int s = SB; s < SE; ++s) {
      const R wl = s == 0 ? F[P2][1 - O + 2 * (NH - 1)] : C[s > 0 ? s - 1 : 0][P1][NH - 1];
      const R wf = s == 0 ? F[P2][1 - O] : C[s > 0 ? s - 1 : 0][P1][0];
      nbs[s - SB] = (O == 0) ? shfl_up1(wl) : shfl_dn1(wf);
    }
#endif
#pragma unroll
    for (int s = SB; s < SE; ++s) {
      const int r = i - s;
      R n[NH], sv[NH], w[NH], u[NH];
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        if (s == 0) {
          n[h] = F[PH][O + 2 * h];          // row i-1
          sv[h] = F[P1][O + 2 * h];         // row i+1
          w[h] = F[P2][1 - O + 2 * h];      // row i, other colour
          u[h] = F[P2][O + 2 * h];          // row i, self
        } else {
          const int p = s > 0 ? s - 1 : 0;
          n[h] = C[p][P2][h];               // row r-1
          sv[h] = C[p][PH][h];              // row r+1
          w[h] = C[p][P1][h];               // row r
          if (s == 1) {
            u[h] = F[PH][O + 2 * h];        // source row i-1
          } else {
            const int pp = s >= 2 ? s - 2 : 0;
            u[h] = C[pp][P2][h];
          }
        }
      }
      // W/E neighbours of cell q = O+2h are the other colour's h-1, h (O = 0)
      // or h, h+1 (O = 1); the one outside the lane is the left lane's last
      // (O = 0) or the right lane's first (O = 1)
#if SOR_WAVE_HOIST
      const R nb = nbs[s - SB];
#else
      const R nb = (O == 0) ? shfl_up1(w[NH - 1]) : shfl_dn1(w[0]);
#endif
      R v[NH], pcor[NH];
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const R we = (O == 0) ? radd(h == 0 ? nb : w[h > 0 ? h - 1 : 0], w[h])
                              : radd(w[h], h == NH - 1 ? nb : w[h < NH - 1 ? h + 1 : 0]);
        v[h] = sor_update_p(radd(n[h], sv[h]), we, u[h], a.w, pcor[h]);
        if (MK == 1) {
          v[h] = upd[O + 2 * h] ? v[h] : u[h];
        } else if (MK == 2) {
          const bool rowok = (unsigned)(r - 1) < (unsigned)rows;
          v[h] = (rowok && upd[O + 2 * h]) ? v[h] : u[h];
        }
      }
      if (CK == 4 && (s & 1) == 0 && probe_row(M6, s)) {
        // probe rows of this batch: row i_first+6j (M6 == s) or 6 rows above
        // (M6 == s-6); their ownership masks are set once per batch
        const int pi = M6 < s ? 1 : 0;
#pragma unroll
        for (int h = 0; h < NH; h += 2) {
          const unsigned int hA = (unsigned int)hi_bits(rsub(v[h], u[h])) & ownM[h] & pf[pi];
          const unsigned int hB =
              h + 1 < NH ? (unsigned int)hi_bits(rsub(v[h + 1 < NH ? h + 1 : 0], u[h + 1 < NH ? h + 1 : 0])) &
                               ownM[h + 1 < NH ? h + 1 : 0] & pf[pi]
                         : 0u;
          hmax[s >> 1] = max3u(hmax[s >> 1], hA, hB);
        }
      } else if (CK == 3) {
        // all-ones iff this stage's row is an owned row (bit s of rowm)
        const unsigned int fill = (unsigned int)((int)(rowm << (31 - s)) >> 31);
#pragma unroll
        for (int h = 0; h < NH; h += 2) {
          const unsigned int hA = (unsigned int)hi_bits(rsub(v[h], u[h])) & ownM[h] & fill;
          const unsigned int hB =
              h + 1 < NH ? (unsigned int)hi_bits(rsub(v[h + 1 < NH ? h + 1 : 0], u[h + 1 < NH ? h + 1 : 0])) &
                               ownM[h + 1 < NH ? h + 1 : 0] & fill
                         : 0u;
          hmax[s >> 1] = max3u(hmax[s >> 1], hA, hB);
        }
      } else if (CK != 0 && (CK == 2 || s >= S - 2)) {
        const bool inb = (unsigned)(r - R0) < (unsigned)(R1 - R0);
        const int slot = CK == 2 ? (s >> 1) : 0;
#pragma unroll
        for (int h = 0; h < NH; ++h)
          dmax[slot] = umax64(dmax[slot], (inb && ownP[h]) ? delta_bits(v[h], u[h]) : 0ull);
      }
      (void)pcor;
      if (s < S - 1) {
#pragma unroll
        for (int h = 0; h < NH; ++h) C[s][PH][h] = v[h];
      } else {
        // finished row r: this stage's colour at q = O+2h; the other colour
        // from stage S-2's row r (one step old, at q = 1-O+2h)
        const bool inb = (unsigned)(r - R0) < (unsigned)(R1 - R0);
        R out[NC];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          out[O + 2 * h] = v[h];
          out[1 - O + 2 * h] = C[S - 2][P1][h];
        }
        if (LANE_OWN && NC % 4 == 0) {
#pragma unroll
          for (int k = 0; k < NC / 4; ++k)
            stg4_if(inb && ownP[0], orow + 4 * k, out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
        } else if (NC == 4) {
          // ghost band boundaries split a lane (odd T): one 4-wide store for
          // the fully owned lanes, pair stores only at the two strip edges
          stg4_if(inb && ownP[0] && ownP[1], orow, out[0], out[1], out[2], out[3]);
          stg2_if(inb && ownP[0] && !ownP[1], orow, out[0], out[1]);
          stg2_if(inb && ownP[1] && !ownP[0], orow + 2, out[2], out[3]);
        } else {
#pragma unroll
          for (int h = 0; h < NH; ++h) stg2_if(inb && ownP[h], orow + 2 * h, out[2 * h], out[2 * h + 1]);
        }
        orow += pitch;
      }
    }
    if (SE < S) {
      R x[NC];
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        x[h] = C[SE - 1][PH][h];
        x[NH + h] = C[SE >= 2 ? SE - 2 : 0][P2][h];
      }
      hand_st(hp, M6, x);
    }
  }

  template <int MK>
  __device__ __forceinline__ void batch(const WaveArgs<R>& a, int i, const R* rowp, R* hp) {
    step<MK, 0>(a, i, rowp, hp);
    step<MK, 1>(a, i + 1, rowp, hp);
    step<MK, 2>(a, i + 2, rowp, hp);
    step<MK, 3>(a, i + 3, rowp, hp);
    step<MK, 4>(a, i + 4, rowp, hp);
    step<MK, 5>(a, i + 5, rowp, hp);
  }

  // Batches [j0, j1) with masking level MK (one loop per level, so each loop
  // keeps its own register assignment and no value is moved between levels).
  template <int MK>
  __device__ __forceinline__ void run_range(const WaveArgs<R>& a, int i_first, int j0, int j1) {
    constexpr bool front = SB == 0;
    constexpr bool split = !(front && SE == S);
#pragma unroll 1
    for (int j = j0; j < j1; ++j) {
      const int m = 6 * j;
      if (CK == 4) {
        // probe rows of batch j: i_first+6j (stages s = M6) and i_first+6j-6 (s = M6+6)
        const int rp = i_first + m;
        pf[0] = (unsigned)(rp - R0) < (unsigned)(R1 - R0) ? 0xffffffffu : 0u;
        pf[1] = (unsigned)(rp - 6 - R0) < (unsigned)(R1 - R0) ? 0xffffffffu : 0u;
      }
      const R* rowp = nullptr;
      R* hp = split ? hand + (j & 1) * (6 * 32 * NC) : nullptr;
      if (front) {
        mbar_wait(bar_s + 8u * (j & 1), (uint32_t)((j >> 1) & 1));
        rowp = ring + (j & 1) * 6 * WC;
        if (split) named_bar_sync(bar_empty + (j & 1), 64);
      } else {
        named_bar_sync(bar_full + (j & 1), 64);
      }
      batch<MK>(a, i_first + m, rowp, hp);
      if (front) {
        if (split) named_bar_arrive(bar_full + (j & 1), 64);
        __syncwarp();
        // every lane's reads of this half of the ring completed (their values
        // were consumed in the batch) before lane 0 refills it
        if (lane == 0 && j + 2 < nbatch) issue_batch_tma(j + 2);
      } else if (j + 2 < nbatch) {
        named_bar_arrive(bar_empty + (j & 1), 64);
      }
    }
  }

  __device__ __forceinline__ void run(const WaveArgs<R>& a, int i_first) {
    constexpr bool front = SB == 0, back = SE == S;
    constexpr bool split = !(front && back);
    if (split && !front) {  // back warp: both handoff buffers start empty
      named_bar_arrive(bar_empty + 0, 64);
      if (nbatch > 1) named_bar_arrive(bar_empty + 1, 64);
    }
    // Batch j updates rows i_first+6j-(S-1) .. i_first+6j+5; they are all in
    // [1, rows] for jA <= j < jB, where only an edge strip's columns need
    // masking.  The first and last batches of the top/bottom bands mask rows.
    const int jA = min(nbatch, max(0, -floordiv6(i_first - S)));            // ceil((S - i_first) / 6)
    const int jB = max(jA, min(nbatch, floordiv6(rows - 5 - i_first) + 1));
    run_range<2>(a, i_first, 0, jA);
    if (col_mask)
      run_range<1>(a, i_first, jA, jB);
    else
      run_range<0>(a, i_first, jA, jB);
    run_range<2>(a, i_first, jB, nbatch);
  }
};

// One warp (or warp pair) = one (strip, band) tile; tiles never synchronise.
template <typename R, int T, int NST, int CK, int SB, int SE, int NC>
__device__ __forceinline__ void wave_tile(const WaveArgs<R>& a, const CUtensorMap* tm, unsigned char* wbase, R* hand,
                                          int bar_id, int lane, int sw, int R0, int R1, int i_first, int nsteps,
                                          unsigned long long (&dm)[kMaxT]) {
  using Pipe = WavePipe<R, T, NST, CK, SB, SE, NC>;
  constexpr int WC = Pipe::WC, NH = Pipe::NH;
  Pipe P;
#pragma unroll
  for (int t = 0; t < P.NSLOT; ++t) {
    if (CK == 1 || CK == 2) P.dmax[t] = 0ull;
    if (CK >= 3) P.hmax[t] = 0u;
  }
  P.ring = reinterpret_cast<const R*>(wbase);
  P.ring_s = smem_u32(wbase);
  P.bar_s = P.ring_s + NST * WC * sizeof(R);
  static_assert(NST == 14, "ring layout: 2 batches of 6 rows + 2 prologue rows");
  P.hand = hand;
  P.bar_full = bar_id;
  P.bar_empty = bar_id + 2;
  P.lane = lane;
  P.rows = (int)a.rows;
  P.R0 = R0;
  P.R1 = R1;
  const long long c0 = (long long)sw + NC * lane;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    const int c = (int)c0 + q;
    P.upd[q] = (c >= 1) && (c <= (int)a.cols);
  }
  P.col_mask = (sw >= 1 && sw + WC - 1 <= (int)a.cols) ? 0 : 1;
  // Ownership by position: the strip minus its 2T ghost columns per side.
  // The ghost bands are 2T wide and strips start at even columns, so they
  // cover whole column pairs (q = 2h, 2h+1; whole lanes when NC divides 2T);
  // cell q = O+2h is in pair h.  Owned-by-position columns of different
  // strips are disjoint.  Ring and padding columns inside it are never
  // updated: they carry their source value through every stage, so storing
  // them rewrites the value they hold and their |delta| is 0.  Stores and
  // maxima therefore need no per-column test against [1, cols].
  {
    const int g_lo = sw + 2 * T, g_hi = sw + WC - 2 * T;
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      const int cp = (int)c0 + 2 * h;
      P.ownP[h] = cp >= g_lo && cp + 1 < g_hi;
      P.ownM[h] = P.ownP[h] ? 0x7fffffffu : 0u;
    }
  }
  // row finished by stage S-1 at step 0 is i_first - (S-1)
  P.orow = a.dst + (long long)(i_first - (2 * T - 1) - a.g0) * a.pitch + c0;
#pragma unroll
  for (int s = 0; s < 2 * T - 1; ++s)
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int h = 0; h < NH; ++h) P.C[s][k][h] = R(0);
  P.pitch = a.pitch;
  P.tm = tm;
  P.tm2 = tm + 1;
  P.tm_x = kColPad + sw;
  P.tm_y = i_first - 1 - (int)a.g0;
  P.nbatch = nsteps / 6;
  if (SB == 0) {
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) mbar_init(P.bar_s + 8u * k, 1u);
      mbar_fence_init();
    }
    __syncwarp();
    if (lane == 0) {
      P.issue_prologue();
      P.issue_batch_tma(0);
      if (P.nbatch > 1) P.issue_batch_tma(1);
    }
    mbar_wait(P.bar_s + 16u, 0u);
    P.ld_row(P.ring + 12 * WC, P.F[0]);  // row i_first - 1
    P.ld_row(P.ring + 13 * WC, P.F[1]);  // row i_first
  }
  P.run(a, i_first);
#pragma unroll
  for (int t = 0; t < P.NSLOT; ++t) dm[t] = CK >= 3 ? (unsigned long long)P.hmax[t] : P.dmax[(CK == 1 || CK == 2) ? t : 0];
}

// Register budget per configuration: resident CTAs (4 warps each) per SM.
// NC = 4: split kernels hold half the stages per warp and aim for 4 CTAs;
// wider lanes hold NC/4 times the registers and trade warps for ILP.
#ifndef SOR_WAVE_MINB34
#define SOR_WAVE_MINB34 3
#endif
#ifndef SOR_WAVE_MINB_SPLIT
#define SOR_WAVE_MINB_SPLIT 4
#endif
__host__ __device__ constexpr int wave_min_blocks(int T, bool split, int NC) {
  return NC == 8 ? 2 : NC == 6 ? 3 : split ? SOR_WAVE_MINB_SPLIT : (T <= 2 ? 4 : SOR_WAVE_MINB34);
}
// Split point of a warp pair: the front warp runs stages [0, K), the back
// warp [K, 2T).  The front also streams the source rows (TMA waits, LDS) and
// was measured to be the slower warp at K = T, so it gets fewer stages.
// (Measured on B200, C3/C5: T = 4 -> K = 3 is 2-4% faster than K = 4, K = 2
// slower; T = 3 -> K = 3 beats K = 2; T = 2 needs K = 2.)
#ifndef SOR_WAVE_K4
#define SOR_WAVE_K4 3
#endif
__host__ __device__ constexpr int wave_split_stage(int T) { return T == 4 ? SOR_WAVE_K4 : T; }
// warps (tiles, or warp pairs in split mode) per CTA
__host__ __device__ constexpr int wave_tiles_per_cta(bool split) { return split ? kWaveWarps / 2 : kWaveWarps; }
template <typename R, int NST, bool SPLIT, int NC>
__host__ __device__ constexpr int wave_smem_bytes() {
  return SPLIT ? (kWaveWarps / 2) * wave_smem_per_pair<R, NST, NC>() : kWaveWarps * wave_smem_per_warp<R, NST, NC>();
}

// Warp pairs: the front warp (stages [0, K), source stream) and the back warp
// ([K, 2T), stores) do unequal work.  A CTA's warp w runs on sub-partition
// (SMSP) w % 4 of its SM, so with fixed roles every resident CTA would put its
// fronts on the same two SMSPs and its backs on the other two.  The roles of
// a CTA are therefore swapped when its hardware warp slot (%warpid of warp 0,
// 4 slots per CTA) is odd, so each SMSP hosts fronts and backs of different
// CTAs (SOR_WAVE_MIX=0 at build time: fixed roles).
#ifndef SOR_WAVE_MIX
#define SOR_WAVE_MIX 0
#endif

template <typename R, int T, int NST, int CK, bool SPLIT, int NC, bool LINK>
__global__ void __launch_bounds__(kWaveWarps * 32, wave_min_blocks(T, SPLIT, NC))
    wave_kernel(WaveArgs<R> a, IterCtl ctl, const __grid_constant__ WaveMaps tm) {
  const int bid = (int)blockIdx.x - ctl.defer;
  extern __shared__ __align__(128) unsigned char wave_smem[];
  constexpr int WC = wave_cols<NC>();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int slot = SPLIT ? warp >> 1 : warp;  // tile slot within the CTA
  int role = SPLIT ? warp & 1 : 0;            // 0 front (or whole), 1 back
  if (SPLIT && SOR_WAVE_MIX) {
    __shared__ int cta_swap;
    if (threadIdx.x == 0) {
      unsigned wid;
      asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
      cta_swap = (int)((wid >> 2) & 1u);
    }
    __syncthreads();
    role ^= cta_swap;
  }
  const int gw = bid * wave_tiles_per_cta(SPLIT) + slot;
  // the tile table is written once by the host: read it before waiting on the
  // previous launch, so its latency overlaps that wait and the stop read
  const bool has_tile = bid >= 0 && gw < a.ntiles;
  const int4 tile = has_tile ? a.tiles[gw] : make_int4(0, 0, 0, 0);
  // Programmatic dependent launch (single slab): the next launch in the
  // stream may be scheduled as soon as every CTA of this one has started;
  // everything this launch reads (source plane, stop flag, maxima) is written
  // by the previous launch, so wait for its completion first.  Both are no-ops
  // for an ordinary launch.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the previous launch wrote the source plane through the generic proxy;
  // this launch reads it with TMA (async proxy)
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (ctl.st && ctl.solve) {
    if (ctl.defer && blockIdx.x == 0) {  // the decision block: stop test of the previous pass
      if (threadIdx.x == 0 && ctl.prev_valid && !ld_stop(ctl.st))
        finalize_pass(ctl.st, ctl, ctl.prev_k_last, ctl.prev_T, ctl.prev_ck, ctl.prev_set, ctl.prev_seq);
      return;
    }
    // one read per CTA: with a deferred stop test the flag can change while
    // this launch runs, and the warps of a pair must agree (named barriers)
    __shared__ int cta_stop;
    if (threadIdx.x == 0) cta_stop = ld_stop(ctl.st);
    __syncthreads();
    if (cta_stop) return;
  }
  unsigned long long dm[kMaxT] = {};
  if (has_tile) {
    const int sw = a.s0 + tile.x * (WC - 4 * T);
    const int R0 = tile.y;
    const int R1 = tile.z;
    // step m (front row i_first+m) feeds stage 2T-1 row i_first+m-2T+1;
    // i_first even; nsteps a multiple of 6 (ring phase x parity)
    const int i_first = (R0 - (2 * T - 1)) & ~1;
    const int nsteps = (R1 + 2 * T - 1 - i_first + 5) / 6 * 6;
    if (LINK && role == 0) tile_halo_wait(a, sw, WC, R0, R1, 2 * T, lane, ctl.st);
    if (SPLIT) {
      unsigned char* pbase = wave_smem + slot * wave_smem_per_pair<R, NST, NC>();
      R* hand = reinterpret_cast<R*>(pbase + wave_smem_per_warp<R, NST, NC>());
      const int bar_id = 1 + 4 * slot;  // named barriers 1..8 (0 is __syncthreads)
      constexpr int K = wave_split_stage(T);
      if (role == 0)
        wave_tile<R, T, NST, CK, 0, K, NC>(a, tm.m, pbase, hand, bar_id, lane, sw, R0, R1, i_first, nsteps, dm);
      else
        wave_tile<R, T, NST, CK, K, 2 * T, NC>(a, tm.m, pbase, hand, bar_id, lane, sw, R0, R1, i_first, nsteps, dm);
    } else {
      unsigned char* wbase = wave_smem + warp * wave_smem_per_warp<R, NST, NC>();
      wave_tile<R, T, NST, CK, 0, 2 * T, NC>(a, tm.m, wbase, nullptr, 0, lane, sw, R0, R1, i_first, nsteps, dm);
    }
  }
  if (LINK && (!SPLIT || role == 1)) {
    // re-read the tile (nothing of it stays live across the stream loop)
    const int gw2 = ((int)blockIdx.x - ctl.defer) * wave_tiles_per_cta(SPLIT) + (SPLIT ? (int)(threadIdx.x >> 6) : (int)(threadIdx.x >> 5));
    if ((int)blockIdx.x >= ctl.defer && gw2 < a.ntiles) {
      const int4 t2 = a.tiles[gw2];
      tile_halo_push<R, NC>(a, a.s0 + t2.x * (WC - 4 * T), WC, 2 * T, t2.x, t2.y, t2.z, (int)(threadIdx.x & 31));
    }
  }
  (void)role;
  if (CK != 0) {
    // warp max -> CTA max in shared memory -> one atomic per CTA and slot
    constexpr int NS = CK >= 2 ? T : 1;
    __shared__ unsigned long long cta_max[kWaveWarps][NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const unsigned long long m =
          CK >= 3 ? ((unsigned long long)__reduce_max_sync(0xffffffffu, (unsigned int)dm[t]) << 32)
                  : warp_max_u64(dm[t]);
      if (lane == 0) cta_max[warp][t] = m;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int t = 0; t < NS; ++t) {
        unsigned long long m = 0ull;
#pragma unroll
        for (int w = 0; w < kWaveWarps; ++w) m = umax64(m, cta_max[w][t]);
        contribute(ctl, t, m);
      }
      maybe_finalize(ctl);
    }
  }
}

// ---------------------------------------------------------------- persistent (K6)
// L2-resident grids (C2: two 8 MB planes): the launch, ramp and drain of one
// wave launch per pass cost more than the pass itself.  One cooperative
// launch runs `npasses` T-deep passes; the CTAs meet at a grid barrier
// between passes (the paper's per-phase barrier [P:314, P:317] once per T
// iterations), alternating the planes.  Each pass is the wave kernel's tile
// pass (same tiles, same stages), so the result is bitwise the same.
__device__ __forceinline__ void mbar_inval(uint32_t bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// All CTAs of a cooperative launch: arrive, then wait until `target` CTAs
// arrived in total (the counter only grows during a launch).
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    while (ld_acquire_gpu_u32(ctr) < target) {
    }
  }
  __syncthreads();
  // the next pass reads rows other CTAs just wrote (generic proxy) with TMA
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <typename R, int T, int NST, bool SPLIT, int NC>
__global__ void __launch_bounds__(kWaveWarps * 32, wave_min_blocks(T, SPLIT, NC))
    wave_persist_kernel(WaveArgs<R> a, int npasses, unsigned* gbar, const __grid_constant__ WaveMaps tmA,
                        const __grid_constant__ WaveMaps tmB) {
  extern __shared__ __align__(128) unsigned char wave_smem[];
  constexpr int WC = wave_cols<NC>();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int slot = SPLIT ? warp >> 1 : warp;
  const int role = SPLIT ? warp & 1 : 0;
  const int gw = (int)blockIdx.x * wave_tiles_per_cta(SPLIT) + slot;
  const bool has_tile = gw < a.ntiles;
  const int4 tile = has_tile ? a.tiles[gw] : make_int4(0, 0, 0, 0);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");
  unsigned long long dm[kMaxT] = {};
  for (int p = 0; p < npasses; ++p) {
    WaveArgs<R> ap = a;
    if (p & 1) {
      ap.src = a.dst;
      ap.dst = const_cast<R*>(a.src);
    }
    const CUtensorMap* tm = (p & 1) ? tmB.m : tmA.m;
    if (has_tile) {
      const int sw = a.s0 + tile.x * (WC - 4 * T);
      const int R0 = tile.y, R1 = tile.z;
      const int i_first = (R0 - (2 * T - 1)) & ~1;
      const int nsteps = (R1 + 2 * T - 1 - i_first + 5) / 6 * 6;
      unsigned char* base = SPLIT ? wave_smem + slot * wave_smem_per_pair<R, NST, NC>()
                                  : wave_smem + warp * wave_smem_per_warp<R, NST, NC>();
      if (SPLIT) {
        R* hand = reinterpret_cast<R*>(base + wave_smem_per_warp<R, NST, NC>());
        const int bar_id = 1 + 4 * slot;
        constexpr int K = wave_split_stage(T);
        if (role == 0)
          wave_tile<R, T, NST, 0, 0, K, NC>(ap, tm, base, hand, bar_id, lane, sw, R0, R1, i_first, nsteps, dm);
        else
          wave_tile<R, T, NST, 0, K, 2 * T, NC>(ap, tm, base, hand, bar_id, lane, sw, R0, R1, i_first, nsteps, dm);
      } else {
        wave_tile<R, T, NST, 0, 0, 2 * T, NC>(ap, tm, base, nullptr, 0, lane, sw, R0, R1, i_first, nsteps, dm);
      }
      // the tile's mbarriers are initialised again by the next pass's tile
      if (role == 0 && lane == 0) {
        const uint32_t bar = smem_u32(base) + NST * WC * (uint32_t)sizeof(R);
#pragma unroll
        for (int k = 0; k < 3; ++k) mbar_inval(bar + 8u * k);
      }
    }
    if (p + 1 < npasses) grid_barrier(gbar, (unsigned)(p + 1) * gridDim.x);
  }
}

// ---------------------------------------------------------------- Jacobi (NEXT-2)
// Jacobi [P:95, S:179-187] on the same layout, tiles and TMA source ring as
// the wave kernel: X_k from X_{k-1} only, X = 0.25*((N+S)+(W+E)).  T
// iterations per HBM pass = T stages; stage s updates EVERY cell of row i-s
// from stage s-1's rows r-1, r, r+1 (4 values per lane per row, 3-row rings
// indexed by step mod 3).  The dependency cone grows one column per stage, so
// strips overlap by G = T rounded up to even ghost columns per side (even, so
// stores and ownership stay pair-aligned).  One warp per tile.
__host__ __device__ constexpr int jacobi_ghost(int T) { return T + (T & 1); }

template <typename R, int T, int NST, int CK>
struct JacobiPipe {
  static constexpr int S = T;
  static constexpr int NC = kWaveNC;
  static constexpr int WC = wave_cols<NC>();
  static constexpr int G = jacobi_ghost(T);
  static constexpr int NSLOT = CK == 2 ? T : 1;
  static constexpr uint32_t ROWB = WC * sizeof(R);
  R F[3][NC];                        // source rows, slot = step % 3 phase as in WavePipe
  R J[S > 1 ? S - 1 : 1][3][NC];     // stage outputs
  unsigned long long dmax[NSLOT];
  bool upd[NC];
  bool ownP[NC / 2];
  int rows, R0, R1;
  int col_mask;
  R* orow;
  const R* ring;
  uint32_t ring_s, bar_s;
  const CUtensorMap* tm;
  const CUtensorMap* tm2;
  int tm_x, tm_y;
  long long pitch;
  int nbatch;
  int lane;

  __device__ __forceinline__ void issue_batch_tma(int j) {
    const uint32_t bar = bar_s + 8u * (j & 1);
    mbar_expect_tx(bar, 6 * ROWB);
    tma_rows(ring_s + (j & 1) * 6 * ROWB, tm, tm_x, tm_y + 6 * j + 2, bar);
  }
  __device__ __forceinline__ void issue_prologue() {
    const uint32_t bar = bar_s + 16u;
    mbar_expect_tx(bar, 2 * ROWB);
    tma_rows(ring_s + 12 * ROWB, tm2, tm_x, tm_y, bar);
  }
  __device__ __forceinline__ void ld_row(const R* row, R (&x)[NC]) { ldsN<NC>(row + NC * lane, x); }

  template <int MK, int M6>
  __device__ __forceinline__ void step(const WaveArgs<R>& a, int i, const R* rowp) {
    constexpr int PH = M6 % 3;
    constexpr int P1 = (PH + 2) % 3;
    constexpr int P2 = (PH + 1) % 3;
    ld_row(rowp + M6 * WC, F[P1]);  // source row i+1
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int r = i - s;
      const int p = s > 0 ? s - 1 : 0;
      R n[NC], sv[NC], c[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        n[q] = s == 0 ? F[PH][q] : J[p][P2][q];   // row r-1
        sv[q] = s == 0 ? F[P1][q] : J[p][PH][q];  // row r+1
        c[q] = s == 0 ? F[P2][q] : J[p][P1][q];   // row r
      }
      const R wl = shfl_up1(c[NC - 1]);  // column c0-1 (left lane)
      const R er = shfl_dn1(c[0]);       // column c0+NC (right lane)
      R v[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        const R we = radd(q == 0 ? wl : c[q > 0 ? q - 1 : 0], q == NC - 1 ? er : c[q < NC - 1 ? q + 1 : 0]);
        v[q] = rmul(R(0.25), radd(radd(n[q], sv[q]), we));
        if (MK == 1) {
          v[q] = upd[q] ? v[q] : c[q];
        } else if (MK == 2) {
          const bool rowok = (unsigned)(r - 1) < (unsigned)rows;
          v[q] = (rowok && upd[q]) ? v[q] : c[q];
        }
      }
      if (CK == 2 || (CK == 1 && s == S - 1)) {
        const bool inb = (unsigned)(r - R0) < (unsigned)(R1 - R0);
        const int slot = CK == 2 ? s : 0;
#pragma unroll
        for (int q = 0; q < NC; ++q)
          dmax[slot] = umax64(dmax[slot], (inb && ownP[q >> 1]) ? delta_bits(v[q], c[q]) : 0ull);
      }
      if (s < S - 1) {
#pragma unroll
        for (int q = 0; q < NC; ++q) J[s][PH][q] = v[q];
      } else {
        const bool inb = (unsigned)(r - R0) < (unsigned)(R1 - R0);
        if (G % NC == 0) {
          stg4_if(inb && ownP[0], orow, v[0], v[1], v[2], v[3]);
        } else {
          stg4_if(inb && ownP[0] && ownP[1], orow, v[0], v[1], v[2], v[3]);
          stg2_if(inb && ownP[0] && !ownP[1], orow, v[0], v[1]);
          stg2_if(inb && ownP[1] && !ownP[0], orow + 2, v[2], v[3]);
        }
        orow += pitch;
      }
    }
  }

  template <int MK>
  __device__ __forceinline__ void run_range(const WaveArgs<R>& a, int i_first, int j0, int j1) {
#pragma unroll 1
    for (int j = j0; j < j1; ++j) {
      mbar_wait(bar_s + 8u * (j & 1), (uint32_t)((j >> 1) & 1));
      const R* rowp = ring + (j & 1) * 6 * WC;
      const int i = i_first + 6 * j;
      step<MK, 0>(a, i, rowp);
      step<MK, 1>(a, i + 1, rowp);
      step<MK, 2>(a, i + 2, rowp);
      step<MK, 3>(a, i + 3, rowp);
      step<MK, 4>(a, i + 4, rowp);
      step<MK, 5>(a, i + 5, rowp);
      __syncwarp();
      if (lane == 0 && j + 2 < nbatch) issue_batch_tma(j + 2);
    }
  }

  __device__ __forceinline__ void run(const WaveArgs<R>& a, int i_first) {
    // rows updated by batch j: i_first+6j-(S-1) .. i_first+6j+5 (see WavePipe::run)
    const int jA = min(nbatch, max(0, -floordiv6(i_first - S)));
    const int jB = max(jA, min(nbatch, floordiv6(rows - 5 - i_first) + 1));
    run_range<2>(a, i_first, 0, jA);
    if (col_mask)
      run_range<1>(a, i_first, jA, jB);
    else
      run_range<0>(a, i_first, jA, jB);
    run_range<2>(a, i_first, jB, nbatch);
  }
};

template <typename R, int T, int NST, int CK, bool LINK>
__global__ void __launch_bounds__(kWaveWarps * 32, T <= 2 ? 4 : 3)
    jacobi_kernel(WaveArgs<R> a, IterCtl ctl, const __grid_constant__ WaveMaps tm) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (ctl.st && ctl.solve) {
    if (ctl.defer && blockIdx.x == 0) {  // the decision block (see wave_kernel)
      if (threadIdx.x == 0 && ctl.prev_valid && !ld_stop(ctl.st))
        finalize_pass(ctl.st, ctl, ctl.prev_k_last, ctl.prev_T, ctl.prev_ck, ctl.prev_set, ctl.prev_seq);
      return;
    }
    __shared__ int cta_stop;
    if (threadIdx.x == 0) cta_stop = ld_stop(ctl.st);
    __syncthreads();
    if (cta_stop) return;
  }
  extern __shared__ __align__(128) unsigned char wave_smem[];
  using Pipe = JacobiPipe<R, T, NST, CK>;
  constexpr int WC = Pipe::WC, NC = Pipe::NC, G = Pipe::G;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gw = ((int)blockIdx.x - ctl.defer) * kWaveWarps + warp;
  unsigned long long dm[kMaxT] = {};
  if (gw < a.ntiles) {
    const int4 tile = a.tiles[gw];
    const int sw = a.s0 + tile.x * (WC - 2 * G);
    const int R0 = tile.y, R1 = tile.z;
    const int i_first = (R0 - (T - 1)) & ~1;
    const int nsteps = (R1 + T - 1 - i_first + 5) / 6 * 6;
    if (LINK) tile_halo_wait(a, sw, WC, R0, R1, T, lane, ctl.st);
    unsigned char* wbase = wave_smem + warp * wave_smem_per_warp<R, NST, NC>();
    Pipe P;
#pragma unroll
    for (int t = 0; t < Pipe::NSLOT; ++t) P.dmax[t] = 0ull;
    P.ring = reinterpret_cast<const R*>(wbase);
    P.ring_s = smem_u32(wbase);
    P.bar_s = P.ring_s + NST * WC * sizeof(R);
    P.lane = lane;
    P.rows = (int)a.rows;
    P.R0 = R0;
    P.R1 = R1;
    const long long c0 = (long long)sw + NC * lane;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int cc = (int)c0 + q;
      P.upd[q] = (cc >= 1) && (cc <= (int)a.cols);
    }
    P.col_mask = (sw >= 1 && sw + WC - 1 <= (int)a.cols) ? 0 : 1;
    {
      // ownership by position (see wave_tile): the strip minus G ghost columns per side
      const int g_lo = sw + G, g_hi = sw + WC - G;
#pragma unroll
      for (int h = 0; h < NC / 2; ++h) {
        const int cp = (int)c0 + 2 * h;
        P.ownP[h] = cp >= g_lo && cp + 1 < g_hi;
      }
    }
    P.orow = a.dst + (long long)(i_first - (T - 1) - a.g0) * a.pitch + c0;
#pragma unroll
    for (int s = 0; s < (T > 1 ? T - 1 : 1); ++s)
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int q = 0; q < NC; ++q) P.J[s][k][q] = R(0);
    P.pitch = a.pitch;
    P.tm = &tm.m[0];
    P.tm2 = &tm.m[1];
    P.tm_x = kColPad + sw;
    P.tm_y = i_first - 1 - (int)a.g0;
    P.nbatch = nsteps / 6;
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) mbar_init(P.bar_s + 8u * k, 1u);
      mbar_fence_init();
    }
    __syncwarp();
    if (lane == 0) {
      P.issue_prologue();
      P.issue_batch_tma(0);
      if (P.nbatch > 1) P.issue_batch_tma(1);
    }
    mbar_wait(P.bar_s + 16u, 0u);
    P.ld_row(P.ring + 12 * WC, P.F[0]);  // row i_first - 1
    P.ld_row(P.ring + 13 * WC, P.F[1]);  // row i_first
    P.run(a, i_first);
#pragma unroll
    for (int t = 0; t < Pipe::NSLOT; ++t) dm[t] = P.dmax[t];
  }
  if (LINK) {
    const int gw2 = ((int)blockIdx.x - ctl.defer) * kWaveWarps + (int)(threadIdx.x >> 5);
    if ((int)blockIdx.x >= ctl.defer && gw2 < a.ntiles) {
      const int4 t2 = a.tiles[gw2];
      tile_halo_push<R, NC>(a, a.s0 + t2.x * (WC - 2 * G), WC, G, t2.x, t2.y, t2.z, (int)(threadIdx.x & 31));
    }
  }
  if (CK != 0) {
    constexpr int NS = CK == 2 ? T : 1;
    __shared__ unsigned long long cta_max[kWaveWarps][NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const unsigned long long m = warp_max_u64(dm[t]);
      if (lane == 0) cta_max[warp][t] = m;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int t = 0; t < NS; ++t) {
        unsigned long long m = 0ull;
#pragma unroll
        for (int w = 0; w < kWaveWarps; ++w) m = umax64(m, cta_max[w][t]);
        contribute(ctl, t, m);
      }
      maybe_finalize(ctl);
    }
  }
}

// ---------------------------------------------------------------- 3-D (NEXT-3)
// 3-D red-black SOR [P:410]: (nz+2) x (ny+2) x (nx+2) grid with a Dirichlet
// shell; colour of (z, y, x) red iff z+y+x even, red phase first.  Per cell:
// s = ((N+S)+(W+E))+(U+D) (N/S = y-1/y+1, W/E = x-1/x+1, U/D = z-1/z+1),
// a = s/6 (correctly rounded division), r = a-u, u' = u + w*r.  One colour
// phase per launch, in place, one thread per cell of the colour (the K1 form
// of the 2-D path; 32 algorithmic bytes per update over the two phases).
// Layout: element (z, y, x) at base + (z*(ny+2) + y)*pitch + x.
template <typename R, bool CHECK>
__global__ void __launch_bounds__(256) k3d_half_sweep(R* base, long long pitch, int nz, int ny, int nx, int color,
                                                      R w, IterCtl ctl) {
  if (ctl.st && ctl.solve && ld_stop(ctl.st)) return;
  const int y = blockIdx.y + 1, z = blockIdx.z + 1;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int x = ((((z + y + 1) & 1) == color) ? 1 : 2) + 2 * (int)t;
  const long long plane = (long long)(ny + 2) * pitch;
  unsigned long long dmax = 0ull;
  if (x <= nx) {
    R* uc = base + (long long)z * plane + (long long)y * pitch + x;
    const R u = uc[0];
    const R s = radd(radd(radd(uc[-pitch], uc[pitch]), radd(uc[-1], uc[1])), radd(uc[-plane], uc[plane]));
    const R a = div6(s);
    const R un = radd(u, rmul(w, rsub(a, u)));
    if (CHECK) dmax = delta_bits(un, u);
    uc[0] = un;
  }
  if (CHECK) {
    dmax = warp_max_u64(dmax);
    __shared__ unsigned long long wmax[8];
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = dmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m = 0ull;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) m = umax64(m, wmax[k]);
      contribute(ctl, 0, m);
      maybe_finalize(ctl);
    }
  }
}

// Fused 3-D iteration (K3 form, one HBM pass per iteration, src -> dst).  A
// CTA owns a KX x KY tile of (y, x) columns and a chunk [z0, z1) of planes and
// marches up z; each thread holds a PAIR of x-adjacent columns of the
// (KY+4) x (KX+4) window (the tile and a 2-cell ring), so in every plane one
// of its two cells is red and the other black (no divergence between the
// colour phases).  Step z: the red half-sweep at plane z (tile + 1-cell ring,
// whose new reds the tile's blacks need) from the source planes z-1, z, z+1,
// then the black half-sweep at plane z-1 (tile only) from the new reds of
// planes z-2, z-1, z; plane z-1 of the tile is then final and stored.
// In-plane neighbours come from shared planes (source plane z and the reds of
// plane z-1, double-buffered by z parity), vertical ones from the thread's
// registers; one __syncthreads per plane.  The chunk's first step computes
// the reds of plane z0-1 (the neighbouring chunk owns them; both compute the
// same values from the source), so chunks never synchronise.  Bitwise equal
// to the two-phase sweep: every cell reads exactly the values the in-place
// red-then-black order gives it.
template <int KX, int KY>
struct K3Geo {
  static constexpr int WX = KX + 4, WY = KY + 4;  // window (columns, rows)
  static constexpr int WP = WX / 2;               // column pairs per window row
  static constexpr int NT = WP * WY;              // threads per CTA
};
#ifndef SOR_K3_X
#define SOR_K3_X 32
#endif
#ifndef SOR_K3_Y
#define SOR_K3_Y 16
#endif
#ifndef SOR_K3_PF
#define SOR_K3_PF 2
#endif
constexpr int kX3 = SOR_K3_X, kY3 = SOR_K3_Y;  // tile of the fused 3-D kernel

template <typename R, bool CHECK, int KX, int KY>
__global__ void __launch_bounds__(K3Geo<KX, KY>::NT)
    k3d_fused(const R* __restrict__ src, R* __restrict__ dst, long long pitch, int nz, int ny, int nx, int zc, R w,
              IterCtl ctl) {
  using G = K3Geo<KX, KY>;
  if (ctl.st && ctl.solve && ld_stop(ctl.st)) return;
  __shared__ R s_src[2][G::WY][G::WX];  // source plane z (by z parity)
  __shared__ R s_red[2][G::WY][G::WX];  // plane z after its red phase (by z parity)
  const int tp = threadIdx.x % G::WP, ty = threadIdx.x / G::WP;
  const int tx0 = 2 * tp;  // window column of the pair's first cell
  const int x0 = blockIdx.x * KX - 2 + tx0, y = blockIdx.y * KY - 2 + ty;
  const int z0 = 1 + blockIdx.z * zc, z1 = min(nz + 1, z0 + zc);  // owned planes [z0, z1)
  bool inside[2], interior[2], ring1[2], tile[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int x = x0 + e, tx = tx0 + e;
    inside[e] = x >= 0 && x <= nx + 1 && y >= 0 && y <= ny + 1;
    interior[e] = x >= 1 && x <= nx && y >= 1 && y <= ny;
    ring1[e] = tx >= 1 && tx <= KX + 2 && ty >= 1 && ty <= KY + 2;
    tile[e] = tx >= 2 && tx < KX + 2 && ty >= 2 && ty < KY + 2;
  }
  const bool both = inside[0] && inside[1];
  const long long plane = (long long)(ny + 2) * pitch;
  const long long col = (long long)y * pitch + x0;
  // the pair of plane z (zero outside the grid); one 16-B load when both
  // cells are inside (x0 even: aligned)
  auto ld = [&](int z, R (&v)[2]) {
    v[0] = v[1] = R(0);
    if (z < 0 || z > nz + 1) return;
    const R* p = src + (long long)z * plane + col;
    if (both) {
      if (sizeof(R) == 8) {
        const double2 d = *reinterpret_cast<const double2*>(p);
        v[0] = (R)d.x;
        v[1] = (R)d.y;
      } else {
        const float2 d = *reinterpret_cast<const float2*>(p);
        v[0] = (R)d.x;
        v[1] = (R)d.y;
      }
    } else {
      if (inside[0]) v[0] = p[0];
      if (inside[1]) v[1] = p[1];
    }
  };
  constexpr int kPF = SOR_K3_PF;  // source planes in flight ahead of the step
  R q[kPF][2];
  R sm1[2], s0[2], n2[2], n1[2];
  ld(z0 - 2, sm1);
  ld(z0 - 1, s0);
  n2[0] = n2[1] = n1[0] = n1[1] = R(0);
#pragma unroll
  for (int k = 0; k < kPF; ++k) ld(z0 + k, q[k]);
  unsigned long long dmax = 0ull;
  auto step = [&](int z, R (&qs)[2]) {
    R sp1[2] = {qs[0], qs[1]};  // plane z+1
    ld(z + 1 + kPF, qs);
    const int pz = z & 1;
    s_src[pz][ty][tx0] = s0[0];
    s_src[pz][ty][tx0 + 1] = s0[1];
    __syncthreads();
    // red phase at plane z: the pair's cell e with (z + y + x0 + e) even
    const bool e1 = ((z + y + x0) & 1) != 0;  // the red cell is the pair's second
    R nz0[2] = {s0[0], s0[1]};
    {
      const int tx = tx0 + (e1 ? 1 : 0);
      const bool upd = e1 ? (ring1[1] && interior[1]) : (ring1[0] && interior[0]);
      if (z >= 1 && z <= nz && upd) {
        const R sv = e1 ? s0[1] : s0[0];
        const R s = radd(radd(radd(s_src[pz][ty - 1][tx], s_src[pz][ty + 1][tx]),
                              radd(s_src[pz][ty][tx - 1], s_src[pz][ty][tx + 1])),
                         radd(e1 ? sm1[1] : sm1[0], e1 ? sp1[1] : sp1[0]));
        const R v = radd(sv, rmul(w, rsub(div6(s), sv)));
        nz0[0] = e1 ? nz0[0] : v;
        nz0[1] = e1 ? v : nz0[1];
        if (CHECK && z >= z0 && z < z1 && (e1 ? tile[1] : tile[0])) dmax = umax64(dmax, delta_bits(v, sv));
      }
    }
    s_red[pz][ty][tx0] = nz0[0];
    s_red[pz][ty][tx0 + 1] = nz0[1];
    // black phase at plane z-1: the pair's cell with (z-1 + y + x) odd, i.e.
    // the red index of plane z; its neighbours are reds: in-plane ones of
    // plane z-1 (shared, written last step), vertical ones of planes z-2, z
    if (z - 1 >= z0) {
      const int tx = tx0 + (e1 ? 1 : 0);
      R out[2] = {n1[0], n1[1]};
      if (e1 ? (tile[1] && interior[1]) : (tile[0] && interior[0])) {
        const int qz = pz ^ 1;
        const R ub = e1 ? n1[1] : n1[0];
        const R s = radd(radd(radd(s_red[qz][ty - 1][tx], s_red[qz][ty + 1][tx]),
                              radd(s_red[qz][ty][tx - 1], s_red[qz][ty][tx + 1])),
                         radd(e1 ? n2[1] : n2[0], e1 ? nz0[1] : nz0[0]));
        const R v = radd(ub, rmul(w, rsub(div6(s), ub)));
        out[0] = e1 ? out[0] : v;
        out[1] = e1 ? v : out[1];
        if (CHECK) dmax = umax64(dmax, delta_bits(v, ub));
      }
      R* o = dst + (long long)(z - 1) * plane + col;
      if (tile[0] && tile[1] && both) {
        if (sizeof(R) == 8)
          *reinterpret_cast<double2*>(o) = make_double2((double)out[0], (double)out[1]);
        else
          *reinterpret_cast<float2*>(o) = make_float2((float)out[0], (float)out[1]);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (tile[e] && inside[e]) o[e] = out[e];
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      n2[e] = n1[e];
      n1[e] = nz0[e];
      sm1[e] = s0[e];
      s0[e] = sp1[e];
    }
  };
  for (int z = z0 - 1; z <= z1; z += kPF) {
#pragma unroll
    for (int k = 0; k < kPF; ++k)
      if (z + k <= z1) step(z + k, q[k]);
  }
  if (CHECK) {
    dmax = warp_max_u64(dmax);
    __shared__ unsigned long long wmax[(G::NT + 31) / 32];
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = dmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m = 0ull;
      for (int k = 0; k < (int)((blockDim.x + 31) >> 5); ++k) m = umax64(m, wmax[k]);
      contribute(ctl, 0, m);
      maybe_finalize(ctl);
    }
  }
}

// ---------------------------------------------------------------- K5
// Whole grid (rows+2) x (cols+2) in shared memory; Algorithm 1's loop on one
// CTA.  __syncthreads() is the phase barrier [P:314, P:317].  Used for small
// grids (BJ configs[0]) where launch latency dominates.
constexpr int kK5Cells = 13;  // cells of one colour per thread (1024 threads; <= 200 KB grids)

template <typename R>
__global__ void __launch_bounds__(1024) k5_small_solve(R* base, long long pitch, long long g0,
                                                       int rows, int cols, R w, int solve,
                                                       long long n_iter, double tol,
                                                       long long K, int measure_last,
                                                       DevState* st) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* u = reinterpret_cast<R*>(smem_raw);
  const int ld = cols + 2;
  const int ncell = (rows + 2) * ld;
  for (int c = threadIdx.x; c < ncell; c += blockDim.x) {
    const int i = c / ld, j = c % ld;
    u[c] = base[(i - g0) * pitch + j];
  }
  // each thread's cells of each colour, as shared-memory offsets (-1: none),
  // computed once (Code 2's stride-2 enumeration)
  const int half = (cols + 1) / 2;  // max cells of one colour per row
  const int per_phase = rows * half;
  int off[2][kK5Cells];
#pragma unroll
  for (int color = 0; color < 2; ++color)
#pragma unroll
    for (int k = 0; k < kK5Cells; ++k) {
      const int c = (int)threadIdx.x + k * (int)blockDim.x;
      off[color][k] = -1;
      if (c < per_phase) {
        const int i = 1 + c / half;
        const int j = ((((i + 1) & 1) == color) ? 1 : 2) + 2 * (c % half);
        if (j <= cols) off[color][k] = i * ld + j;
      }
    }
  // per-warp maxima, double-buffered by iteration parity: iteration k writes
  // slot k&1 and every thread reads all of it after the barrier, so no
  // barrier is needed before the next check overwrites the other slot
  __shared__ unsigned long long wmax[2][32];
  __syncthreads();
  long long k = 1, checks = 0;
  double last = 0.0;
  int converged = 0;
  for (; k <= n_iter; ++k) {
    const int check = solve ? (k % K == 0) : (measure_last && k == n_iter);
    unsigned long long dmax = 0ull;
#pragma unroll
    for (int color = 0; color < 2; ++color) {
#pragma unroll
      for (int q = 0; q < kK5Cells; ++q) {
        const int o = off[color][q];
        if (o >= 0) {
          const R uo = u[o];
          const R un = sor_update(radd(u[o - ld], u[o + ld]), radd(u[o - 1], u[o + 1]), uo, w);
          if (check) dmax = umax64(dmax, delta_bits(un, uo));
          u[o] = un;
        }
      }
      __syncthreads();  // the phase barrier [P:314, P:317]
    }
    if (check) {
      dmax = warp_max_u64(dmax);
      if ((threadIdx.x & 31) == 0) wmax[k & 1][threadIdx.x >> 5] = dmax;
      __syncthreads();
      // every warp folds the warp maxima lane-parallel (one load per lane)
      const int lane = threadIdx.x & 31;
      unsigned long long m = lane < (int)(blockDim.x >> 5) ? wmax[k & 1][lane] : 0ull;
      m = warp_max_u64(m);
      last = __longlong_as_double((long long)m);
      ++checks;
      if (solve && last < tol) {  // every thread decides the same (strict <)
        converged = 1;
        break;
      }
    }
  }
  if (threadIdx.x == 0) {
    st->checks += checks;
    if (checks) st->max_change = last;
    if (converged) {
      st->converged = 1;
      st->conv_iter = k;
    }
    st->iters_done = k > n_iter ? n_iter : k;
    st->stop = 1;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ncell; c += blockDim.x) {
    const int i = c / ld, j = c % ld;
    base[(i - g0) * pitch + j] = u[c];
  }
}

// ---------------------------------------------------------------- layout
// fp64 -> fp32 round-to-nearest (reading #17) and exact widening, row blocks.
static __global__ void narrow_rows(const double* __restrict__ src, long long src_ld, float* dst,
                            long long dst_ld, long long nrows, long long ncols) {
  for (long long r = blockIdx.y; r < nrows; r += gridDim.y)
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < ncols;
         c += (long long)gridDim.x * blockDim.x)
      dst[r * dst_ld + c] = __double2float_rn(src[r * src_ld + c]);
}
static __global__ void widen_rows(const float* __restrict__ src, long long src_ld, double* dst,
                           long long dst_ld, long long nrows, long long ncols) {
  for (long long r = blockIdx.y; r < nrows; r += gridDim.y)
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < ncols;
         c += (long long)gridDim.x * blockDim.x)
      dst[r * dst_ld + c] = (double)src[r * src_ld + c];
}
// Non-finite detector for sor_create's validation of device-resident input.
static __global__ void count_nonfinite(const double* __restrict__ p, long long n, unsigned int* out) {
  unsigned int bad = 0;
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(p[c]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(out, 1u);
}

}  // namespace sorb
