// sor3d_tma.cuh — NEXT-3 one-pass 3-D red-black iteration (the 2-D
// update of Eq. 1 [P:97-100] with the six face neighbours, reading N3-1 of
// s = ((N+S)+(W+E))+(U+D), a = s/6 correctly rounded, u' = u +
// w*(a - u); red iff z+y+x even, red phase first [P:149, P:198]).
//
// One HBM pass per iteration, src -> dst (16 algorithmic bytes per update in
// fp64).  A CTA owns a KX x KY tile of (y, x) columns and a chunk [z0, z1) of
// planes and marches up z.  The source planes arrive by 3-D tensor TMA
// (cp.async.bulk.tensor.3d, one (KX+6) x (KY+4) box per plane: the tile, a
// 2-cell ring and one alignment column) into a ring of NP shared slots, three
// planes ahead of use, one mbarrier per slot.  Per plane z:
//   red(z)    over the tile + 1-cell ring (the tile's blacks need those reds):
//             in-plane neighbours and own value from slot z, U/D from slots
//             z-1, z+1 (all old blacks); the new red is written IN PLACE
//             into slot z (blacks of slot z stay old: later reds of plane
//             z+1 read them as their U neighbour).
//   black(z-1) over the tile: in-plane neighbours = the new reds of slot
//             z-1 (written last step), own old value from slot z-1, U/D =
//             the thread's reds of planes z-2 and z (registers: the same
//             (y, x) column); the finished pair of plane z-1 goes to dst.
// The black phase of a plane needs only reds of earlier planes, so one
// __syncthreads covers two planes: the interval at z runs red(z), red(z+1),
// black(z-2), black(z-1).  Thread t owns a pair of x-adjacent columns
// (one red and one black per plane, so every thread works every step) and
// reads its rows as 16-byte pairs.  A warp holds two ring-1 rows of the same
// parity, so which cell of a pair is red is warp-uniform; steps are unrolled
// in pairs and that position is a compile-time constant (no selects).  The chunk's first step computes the reds
// of plane z0-1 from the source (the neighbouring chunk computes the same
// values), so chunks never synchronise.  Bitwise equal to the two-phase
// sweep: every cell reads exactly the values the in-place red-then-black
// order gives it.
#pragma once

#include <type_traits>

#include "sor_kernels.cuh"

namespace sorb {

constexpr int kT3X = 30, kT3Y = 14;           // tile (x, y)
constexpr int kT3WX = kT3X + 6, kT3WY = kT3Y + 4;  // window: columns [x0-3, x0+33), rows [y0-2, y0+16)
// The TMA box starts on a 16-B boundary (a 3-D box whose first column is not
// 16-B aligned faults with an illegal instruction on B200: fp32 windows
// starting at x0-3 did): the box starts up to 16/size-2 elements left of
// x0-3 and is that much wider, rounded to 16 B.
template <typename R>
__host__ __device__ constexpr int t3_wxb() {
  return (kT3WX + (16 / (int)sizeof(R) - 2) + (16 / (int)sizeof(R)) - 1) / (16 / (int)sizeof(R)) *
         (16 / (int)sizeof(R));
}
constexpr int kT3NP = 8;                       // shared plane slots
constexpr int kT3Pairs = (kT3X + 2) / 2;       // column pairs of the ring-1 region (16: a half warp)
constexpr int kT3Threads = kT3Pairs * (kT3Y + 2);  // 256: 8 warps, each two ring-1 rows of one parity

// elements per shared slot: one box, rounded up to 128 B (TMA destinations
// are 128-B aligned)
template <typename R>
__host__ __device__ constexpr int t3_slot_elems() {
  return (t3_wxb<R>() * kT3WY * (int)sizeof(R) + 127) / 128 * 128 / (int)sizeof(R);
}
template <typename R>
__host__ __device__ constexpr int t3_smem_bytes() {
  return kT3NP * t3_slot_elems<R>() * (int)sizeof(R) + 128;
}

__device__ __forceinline__ void tma_box3(uint32_t dst, const CUtensorMap* tm, int x, int y, int z, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(tm), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}

template <typename R>
struct Pair2;
template <>
struct Pair2<double> {
  __device__ static void ld(const double* p, double& a, double& b) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    a = v.x;
    b = v.y;
  }
  __device__ static void st(double* p, double a, double b) { *reinterpret_cast<double2*>(p) = make_double2(a, b); }
};
template <>
struct Pair2<float> {
  __device__ static void ld(const float* p, float& a, float& b) {
    const float2 v = *reinterpret_cast<const float2*>(p);
    a = v.x;
    b = v.y;
  }
  __device__ static void st(float* p, float a, float b) { *reinterpret_cast<float2*>(p) = make_float2(a, b); }
};

// s/6 as div6 (reading N3-1, N3-2) with a cheaper range test (the high
// word decides).  Normal range (|s| >=
// 0x1.8p-1020, finite): the FMA-corrected quotient; zero, inf, NaN: s
// itself (exact); tiny non-zero: div6_tiny.
template <typename R>
__device__ __forceinline__ R div6_v(R s);
template <>
__device__ __forceinline__ double div6_v(double s) {
  const double yi = 1.0 / 6.0;
  const double q0 = __dmul_rn(s, yi);
  const double r = __fma_rn(-q0, 6.0, s);
  const double q1 = __fma_rn(r, yi, q0);
  const unsigned hi = (unsigned)__double2hiint(s) & 0x7fffffffu, lo = (unsigned)__double2loint(s);
  const bool normal = hi - 0x00380000u <= 0x7fefffffu - 0x00380000u;
  double q = normal ? q1 : s;
  if (hi < 0x00380000u && (hi | lo) != 0u) q = div6_tiny(s);
  return q;
}
template <>
__device__ __forceinline__ float div6_v(float s) {
  const float yi = 1.0f / 6.0f;
  const float q0 = __fmul_rn(s, yi);
  const float r = __fmaf_rn(-q0, 6.0f, s);
  const float q1 = __fmaf_rn(r, yi, q0);
  const unsigned a = __float_as_uint(s) & 0x7fffffffu;
  const bool normal = a - 0x01c00000u <= 0x7f7fffffu - 0x01c00000u;
  float q = normal ? q1 : s;
  if (a < 0x01c00000u && a != 0u) q = div6_tiny(s);
  return q;
}

// Per-thread constants of k3d_tma (all loop-invariant predicates precomputed).
template <typename R>
struct T3Thread {
  int off;        // window offset of the pair: wr * WX + wc
  bool trow;      // a tile row (black phase)
  bool upd[2];    // cell e of the pair is interior (in-plane)
  bool chk[2];    // ... and in a tile column (max-change)
  bool st2, st0, st1;  // store of the finished pair: both cells as one 16-B vector, cell 0, cell 1
};

// A row pair of a slot: cells 0, 1 of the thread's pair in window row wr+dr.
template <typename R>
struct T3Row {
  R a, b;
  __device__ __forceinline__ R at(int e) const { return e ? b : a; }
};
template <typename R>
__device__ __forceinline__ T3Row<R> t3_row(const R* sl, int off) {
  T3Row<R> r;
  Pair2<R>::ld(sl + off, r.a, r.b);
  return r;
}

// Eq. 1 in 3-D for the pair's cell E of a plane: in-plane rows N (above), C
// (own row), S (below), the neighbour outside the pair, vertical U, D.
template <typename R, int E>
__device__ __forceinline__ R t3_update(const T3Row<R>& N, const T3Row<R>& C, const T3Row<R>& S, R outside, R uU,
                                       R uD, R w) {
  const R uW = E ? C.a : outside, uE = E ? outside : C.b;
  const R s = radd(radd(radd(N.at(E), S.at(E)), radd(uW, uE)), radd(uU, uD));
  const R u = C.at(E);
  return radd(u, rmul(w, rsub(div6_v(s), u)));
}

// black(zb) at column E over the tile from slot rows N, C, S (its new reds
// and its own old value) and vertical reds rU (zb-1), rD (zb+1) of the same
// column; the finished pair of plane zb goes to out.
template <typename R, bool CHECK, int E>
__device__ __forceinline__ void t3_black(const T3Thread<R>& t, R w, const T3Row<R>& N, const T3Row<R>& C,
                                         const T3Row<R>& S, R outside, R rU, R rD, R* out,
                                         unsigned long long& dmax) {
  const R v = t3_update<R, E>(N, C, S, outside, rU, rD, w);
  const R u = C.at(E);
  const R b = t.upd[E] ? v : u;
  if (CHECK && t.upd[E] && t.chk[E]) dmax = umax64(dmax, delta_bits(v, u));
  // the finished pair: black b at E, red (slot) at 1-E
  const R o0 = E ? C.a : b, o1 = E ? b : C.b;
  if (t.st2) Pair2<R>::st(out, o0, o1);
  if (t.st0) out[0] = o0;
  if (t.st1) out[1] = o1;
}

template <typename R, bool CHECK>
__global__ void __launch_bounds__(kT3Threads, sizeof(R) == 8 ? 4 : 5)
    k3d_tma(const __grid_constant__ CUtensorMap tm, R* __restrict__ dst, long long pitch, int nz, int ny, int nx,
            int zc, R w, IterCtl ctl) {
  extern __shared__ __align__(128) unsigned char t3_smem[];
  if (ctl.st && ctl.solve && ld_stop(ctl.st)) return;
  constexpr int SP = t3_slot_elems<R>();  // elements per slot
  R* slot = reinterpret_cast<R*>(t3_smem);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(t3_smem + kT3NP * SP * sizeof(R));
  const int tid = threadIdx.x;
  const int warp = tid >> 5, half = (tid >> 4) & 1, p = tid & 15;
  // ring-1 row of the thread: warp w holds rows base, base + 2 (one parity)
  const int ty = (warp >> 1) * 4 + (warp & 1) + 2 * half;
  const int x0 = 1 + (int)blockIdx.x * kT3X, y0 = 1 + (int)blockIdx.y * kT3Y;
  const int z0 = 1 + (int)blockIdx.z * zc, z1 = min(nz + 1, z0 + zc);  // owned planes [z0, z1)
  const int wr = 1 + ty, wc = 2 + 2 * p;        // window row / first column of the pair
  const int y = y0 - 2 + wr, xa = x0 - 3 + wc;  // global row / first column
  T3Thread<R> t;
  // box origin: x0-3 rounded down to 16 B; the window starts xd columns into it
  const int xs = (x0 - 3) & ~(16 / (int)sizeof(R) - 1), xd = (x0 - 3) - xs;
  t.off = wr * t3_wxb<R>() + wc + xd;
  t.trow = wr >= 2 && wr < 2 + kT3Y;
  const bool yin = y >= 1 && y <= ny;
  const bool tcol0 = wc >= 3 && wc < 3 + kT3X, tcol1 = wc + 1 >= 3 && wc + 1 < 3 + kT3X;
  t.upd[0] = yin && xa >= 1 && xa <= nx;
  t.upd[1] = yin && xa + 1 >= 1 && xa + 1 <= nx;
  t.chk[0] = tcol0;
  t.chk[1] = tcol1;
  {
    const bool k0 = yin && tcol0 && xa >= 1 && xa <= nx, k1 = yin && tcol1 && xa + 1 <= nx;
    t.st2 = k0 && k1 && (xa & 1) == 0;
    t.st0 = k0 && !t.st2;
    t.st1 = k1 && !t.st2;
  }
  const uint32_t bar0 = smem_u32(bars);
  // Two planes per barrier.  The interval at z computes red(z), red(z+1) (old
  // blacks only) and black(z-2), black(z-1) (the reds of planes z-2, z-1 were
  // written in earlier intervals; the vertical reds are the thread's own).
  // Intervals z = z0-1, z0+1, ... while z-2 <= z1-1; planes z0-2 .. z+2.
  const int nint = (z1 + 1 - (z0 - 1)) / 2 + 1;
  const int nq = 2 * nint + 3;  // planes q = z - z0 + 2 in [0, nq)
  if (tid == 0) {
    for (int s = 0; s < kT3NP; ++s) mbar_init(bar0 + 8u * s, 1);
    mbar_fence_init();
  }
  __syncthreads();
  constexpr uint32_t kBytes = (uint32_t)(t3_wxb<R>() * kT3WY * sizeof(R));  // one box
  auto issue = [&](int q) {  // plane z0-2+q into its slot
    const uint32_t b = bar0 + 8u * (q % kT3NP);
    mbar_expect_tx(b, kBytes);
    tma_box3(smem_u32(slot + (q % kT3NP) * SP), &tm, xs, y0 - 2, z0 - 2 + q, b);
  };
  if (tid == 0)  // planes 0..NP-4; interval q issues q+NP-4, q+NP-3 (into the slots of q-4, q-3)
    for (int q = 0; q < min(kT3NP - 3, nq); ++q) issue(q);
  // the thread's reds (value after the red phase) of planes z-3, z-2, z-1
  R r3 = R(0), r2 = R(0), r1 = R(0);
  unsigned long long dmax = 0ull;
  const long long zstride = (long long)(ny + 2) * pitch;
  // pointer to the pair in plane z-2 of dst, advanced by two planes per interval
  R* out = dst + (long long)(z0 - 3) * zstride + (long long)y * pitch + xa;
  // the pair's red column in plane z0-1 (warp-uniform)
  const int E0 = (z0 - 1 + y + xa) & 1;
  const int zr_lo = max(1, z0 - 1), zr_hi = min(nz, z1 + 1);  // planes with a red phase
  auto interval = [&](int z, auto e_const) {
    constexpr int E = decltype(e_const)::value;  // red column of plane z
    const int q = z - z0 + 2;
    __syncthreads();  // earlier reds are written; slots of planes z-4, z-3 are free
    if (tid == 0) {
      fence_proxy_async_smem();  // slots being refilled were written by the generic proxy
      if (q + kT3NP - 4 < nq) issue(q + kT3NP - 4);
      if (q + kT3NP - 3 < nq) issue(q + kT3NP - 3);
    }
    // planes z+1, z+2 (z-2 .. z arrived for earlier intervals or the first)
    mbar_wait(bar0 + 8u * ((q + 1) % kT3NP), (uint32_t)(((q + 1) / kT3NP) & 1));
    mbar_wait(bar0 + 8u * ((q + 2) % kT3NP), (uint32_t)(((q + 2) / kT3NP) & 1));
    if (q == 1) {
      mbar_wait(bar0 + 8u * 0, 0u);
      mbar_wait(bar0 + 8u * 1, 0u);
    }
    constexpr int WX = t3_wxb<R>();
    R* sl[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) sl[k] = slot + ((q - 2 + k + kT3NP) % kT3NP) * SP;  // planes z-2 .. z+2
    // Rows are loaded once per interval and shared between the phases that
    // read them: slot z-1's own row is red(z)'s U and black(z-1)'s centre,
    // slot z's own row is red(z)'s centre and red(z+1)'s U (column E^1, which
    // red(z) does not write), slot z+1's own row is red(z)'s D and red(z+1)'s
    // centre (read before red(z+1) writes its column).
    const int o = t.off;
    const T3Row<R> Bc = t3_row(sl[1], o);
    const T3Row<R> Cn = t3_row(sl[2], o - WX), Cc = t3_row(sl[2], o), Cs = t3_row(sl[2], o + WX);
    const T3Row<R> Dn = t3_row(sl[3], o - WX), Dc = t3_row(sl[3], o), Ds = t3_row(sl[3], o + WX);
    const R Co = sl[2][o + (E == 0 ? -1 : 2)];
    const R Do = sl[3][o + (E == 0 ? 2 : -1)];
    const R Fc = sl[4][o + (E ^ 1)];
    // red(z): column E
    R rz = Cc.at(E);
    {
      const R v = t3_update<R, E>(Cn, Cc, Cs, Co, Bc.at(E), Dc.at(E), w);
      const bool upd = (unsigned)(z - zr_lo) <= (unsigned)(zr_hi - zr_lo) && t.upd[E];
      if (upd) {
        sl[2][o + E] = v;
        if (CHECK && z >= z0 && z < z1 && t.trow && t.chk[E]) dmax = umax64(dmax, delta_bits(v, rz));
        rz = v;
      }
    }
    // red(z+1): column E^1
    R rz1 = Dc.at(E ^ 1);
    {
      const R v = t3_update<R, E ^ 1>(Dn, Dc, Ds, Do, Cc.at(E ^ 1), Fc, w);
      const bool upd = (unsigned)(z + 1 - zr_lo) <= (unsigned)(zr_hi - zr_lo) && t.upd[E ^ 1];
      if (upd) {
        sl[3][o + (E ^ 1)] = v;
        if (CHECK && z + 1 >= z0 && z + 1 < z1 && t.trow && t.chk[E ^ 1]) dmax = umax64(dmax, delta_bits(v, rz1));
        rz1 = v;
      }
    }
    if (t.trow) {
      // black(z-2): column E^1 (red column of plane z-1), reds z-3, z-1
      if (z - 2 >= z0 && z - 2 < z1) {
        const T3Row<R> An = t3_row(sl[0], o - WX), Ac = t3_row(sl[0], o), As = t3_row(sl[0], o + WX);
        const R Ao = sl[0][o + (E == 0 ? 2 : -1)];
        t3_black<R, CHECK, E ^ 1>(t, w, An, Ac, As, Ao, r3, r1, out, dmax);
      }
      // black(z-1): column E, reds z-2, z
      if (z - 1 >= z0 && z - 1 < z1) {
        const T3Row<R> Bn = t3_row(sl[1], o - WX), Bs = t3_row(sl[1], o + WX);
        const R Bo = sl[1][o + (E == 0 ? -1 : 2)];
        t3_black<R, CHECK, E>(t, w, Bn, Bc, Bs, Bo, r2, rz, out + zstride, dmax);
      }
    }
    out += 2 * zstride;
    r3 = r1;
    r2 = rz;
    r1 = rz1;
  };
  for (int z = z0 - 1; z - 2 <= z1 - 1; z += 2) {
    if (E0 == 0)
      interval(z, std::integral_constant<int, 0>());
    else
      interval(z, std::integral_constant<int, 1>());
  }
  if (CHECK) {
    dmax = warp_max_u64(dmax);
    __shared__ unsigned long long wmax[(kT3Threads + 31) / 32];
    if ((tid & 31) == 0) wmax[tid >> 5] = dmax;
    __syncthreads();
    if (tid == 0) {
      unsigned long long m = 0ull;
      for (int k = 0; k < (kT3Threads + 31) / 32; ++k) m = umax64(m, wmax[k]);
      contribute(ctl, 0, m);
      maybe_finalize(ctl);
    }
  }
}

}  // namespace sorb
