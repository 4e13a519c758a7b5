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
constexpr int kT3Threads = kT3Pairs * (kT3Y + 2) / 2;  // 128: each thread two adjacent ring-1 rows

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

// Per-thread constants of k3d_tma (all loop-invariant predicates precomputed):
// the thread owns the same column pair in two adjacent window rows a, b.
template <typename R>
struct T3Thread {
  int off;          // window offset of the pair in row a: wr_a * WX + wc (row b: + WX)
  bool trow[2];     // row a / b is a tile row (black phase)
  bool upd[2][2];   // [row][cell] interior (in-plane)
  bool chk[2];      // cell in a tile column (max-change)
  bool st2[2], st0[2], st1[2];  // [row] store of the finished pair: 16-B vector, cell 0, cell 1
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

// black(zb) of row `r` at column E over the tile from slot rows N, C, S (its
// new reds and its own old value) and vertical reds rU (zb-1), rD (zb+1) of
// the same column; the finished pair of plane zb goes to out (tile rows only).
template <typename R, bool CHECK, int E>
__device__ __forceinline__ void t3_black(const T3Thread<R>& t, int r, R w, const T3Row<R>& N, const T3Row<R>& C,
                                         const T3Row<R>& S, R outside, R rU, R rD, R* out,
                                         unsigned long long& dmax) {
  const R v = t3_update<R, E>(N, C, S, outside, rU, rD, w);
  const R u = C.at(E);
  const bool upd = t.upd[r][E];
  const R b = upd ? v : u;
  if (CHECK && upd && t.trow[r] && t.chk[E]) dmax = umax64(dmax, delta_bits(v, u));
  // the finished pair: black b at E, red (slot) at 1-E
  const R o0 = E ? C.a : b, o1 = E ? b : C.b;
  if (t.st2[r]) Pair2<R>::st(out, o0, o1);
  if (t.st0[r]) out[0] = o0;
  if (t.st1[r]) out[1] = o1;
}

// red(z) of row `r` at column E, in place into slot sl at offset o.
template <typename R, bool CHECK, int E>
__device__ __forceinline__ R t3_red(const T3Thread<R>& t, int r, bool red_z, bool red_own, R w, R* sl, int o,
                                    const T3Row<R>& N, const T3Row<R>& C, const T3Row<R>& S, R outside, R uU,
                                    R uD, unsigned long long& dmax) {
  const R u = C.at(E);
  const R v = t3_update<R, E>(N, C, S, outside, uU, uD, w);
  const bool upd = red_z && t.upd[r][E];
  if (upd) sl[o + E] = v;
  if (CHECK && upd && red_own && t.trow[r] && t.chk[E]) dmax = umax64(dmax, delta_bits(v, u));
  return upd ? v : u;
}

template <typename R, bool CHECK>
__global__ void __launch_bounds__(kT3Threads, sizeof(R) == 8 ? 5 : 8)
    k3d_tma(const __grid_constant__ CUtensorMap tm, R* __restrict__ dst, long long pitch, int nz, int ny, int nx,
            int zc, R w, IterCtl ctl) {
  extern __shared__ __align__(128) unsigned char t3_smem[];
  if (ctl.st && ctl.solve && ld_stop(ctl.st)) return;
  constexpr int SP = t3_slot_elems<R>();  // elements per slot
  R* slot = reinterpret_cast<R*>(t3_smem);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(t3_smem + kT3NP * SP * sizeof(R));
  const int tid = threadIdx.x;
  const int p = tid & 15, rp = tid >> 4;  // column pair; rows 2rp, 2rp+1 of the ring-1 region
  const int x0 = 1 + (int)blockIdx.x * kT3X, y0 = 1 + (int)blockIdx.y * kT3Y;
  const int z0 = 1 + (int)blockIdx.z * zc, z1 = min(nz + 1, z0 + zc);  // owned planes [z0, z1)
  const int wra = 1 + 2 * rp, wc = 2 + 2 * p;     // window row a (row b = wra + 1) / first column
  const int ya = y0 - 2 + wra, xa = x0 - 3 + wc;  // global row a / first column
  T3Thread<R> t;
  // box origin: x0-3 rounded down to 16 B; the window starts xd columns into it
  const int xs = (x0 - 3) & ~(16 / (int)sizeof(R) - 1), xd = (x0 - 3) - xs;
  t.off = wra * t3_wxb<R>() + wc + xd;
  const bool tcol0 = wc >= 3 && wc < 3 + kT3X, tcol1 = wc + 1 >= 3 && wc + 1 < 3 + kT3X;
  t.chk[0] = tcol0;
  t.chk[1] = tcol1;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int wr = wra + r, y = ya + r;
    const bool yin = y >= 1 && y <= ny;
    t.trow[r] = wr >= 2 && wr < 2 + kT3Y;
    t.upd[r][0] = yin && xa >= 1 && xa <= nx;
    t.upd[r][1] = yin && xa + 1 >= 1 && xa + 1 <= nx;
    const bool k0 = t.trow[r] && yin && tcol0 && xa >= 1 && xa <= nx;
    const bool k1 = t.trow[r] && yin && tcol1 && xa + 1 <= nx;
    t.st2[r] = k0 && k1 && (xa & 1) == 0;
    t.st0[r] = k0 && !t.st2[r];
    t.st1[r] = k1 && !t.st2[r];
  }
  const uint32_t bar0 = smem_u32(bars);
  // Two planes per barrier.  The interval at z computes red(z), red(z+1) (old
  // blacks only) and black(z-2), black(z-1) (the reds of planes z-2, z-1 were
  // written in earlier intervals; the vertical reds are the thread's own).
  // Intervals z = z0-1, z0+1, ... while z-2 <= z1-1; planes z0-2 .. z+2.
  const int nint = (z1 + 1 - (z0 - 1)) / 2 + 1;
  // planes q = z - z0 + 2 in [0, nq): the last interval (q = 2 nint - 1) reads
  // up to q + 2, and every issued plane is waited for before the CTA exits
  const int nq = 2 * nint + 2;
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
  // the thread's reds (value after the red phase) of planes z-3, z-2, z-1, rows a, b
  R r3a = R(0), r2a = R(0), r1a = R(0), r3b = R(0), r2b = R(0), r1b = R(0);
  unsigned long long dmax = 0ull;
  const long long zstride = (long long)(ny + 2) * pitch;
  // pointer to the pair of row a in plane z-2 of dst, advanced by two planes per interval
  R* out = dst + (long long)(z0 - 3) * zstride + (long long)ya * pitch + xa;
  // row a's red column in plane z0-1 (block-uniform; row b's is the other one)
  const int E0 = (z0 - 1 + ya + xa) & 1;
  const int zr_lo = max(1, z0 - 1), zr_hi = min(nz, z1 + 1);  // planes with a red phase
  auto interval = [&](int z, auto e_const) {
    constexpr int E = decltype(e_const)::value;  // red column of row a in plane z
    constexpr int F = E ^ 1;                     // ... of row b (and of row a in plane z+1)
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
    // Rows are loaded once per interval and shared between the phases and the
    // two rows that read them (see the 1-row notes: a row's red column is the
    // only cell of it a red phase writes, and no phase reads that cell of a
    // slot another phase of the interval writes).
    const int oa = t.off, ob = oa + WX;
    const bool rz_ok = (unsigned)(z - zr_lo) <= (unsigned)(zr_hi - zr_lo);
    const bool rz1_ok = (unsigned)(z + 1 - zr_lo) <= (unsigned)(zr_hi - zr_lo);
    const T3Row<R> Ba = t3_row(sl[1], oa), Bb = t3_row(sl[1], ob);
    const T3Row<R> Cn = t3_row(sl[2], oa - WX), Ca = t3_row(sl[2], oa), Cb = t3_row(sl[2], ob),
                   Cs = t3_row(sl[2], ob + WX);
    const T3Row<R> Dn = t3_row(sl[3], oa - WX), Da = t3_row(sl[3], oa), Db = t3_row(sl[3], ob),
                   Ds = t3_row(sl[3], ob + WX);
    const R Fa = sl[4][oa + F], Fb = sl[4][ob + E];
    const R Coa = sl[2][oa + (E == 0 ? -1 : 2)], Cob = sl[2][ob + (F == 0 ? -1 : 2)];
    const R Doa = sl[3][oa + (F == 0 ? -1 : 2)], Dob = sl[3][ob + (E == 0 ? -1 : 2)];
    // red(z): row a column E, row b column F
    const R rza = t3_red<R, CHECK, E>(t, 0, rz_ok, z >= z0 && z < z1, w, sl[2], oa, Cn, Ca, Cb, Coa, Ba.at(E),
                                      Da.at(E), dmax);
    const R rzb = t3_red<R, CHECK, F>(t, 1, rz_ok, z >= z0 && z < z1, w, sl[2], ob, Ca, Cb, Cs, Cob, Bb.at(F),
                                      Db.at(F), dmax);
    // red(z+1): row a column F, row b column E
    const R rz1a = t3_red<R, CHECK, F>(t, 0, rz1_ok, z + 1 >= z0 && z + 1 < z1, w, sl[3], oa, Dn, Da, Db, Doa,
                                       Ca.at(F), Fa, dmax);
    const R rz1b = t3_red<R, CHECK, E>(t, 1, rz1_ok, z + 1 >= z0 && z + 1 < z1, w, sl[3], ob, Da, Db, Ds, Dob,
                                       Cb.at(E), Fb, dmax);
    // black(z-2): row a column F, row b column E (the red columns of plane z-1); reds z-3, z-1
    if (z - 2 >= z0 && z - 2 < z1) {
      const T3Row<R> An = t3_row(sl[0], oa - WX), Aa = t3_row(sl[0], oa), Ab = t3_row(sl[0], ob),
                     As = t3_row(sl[0], ob + WX);
      const R Aoa = sl[0][oa + (F == 0 ? -1 : 2)], Aob = sl[0][ob + (E == 0 ? -1 : 2)];
      t3_black<R, CHECK, F>(t, 0, w, An, Aa, Ab, Aoa, r3a, r1a, out, dmax);
      t3_black<R, CHECK, E>(t, 1, w, Aa, Ab, As, Aob, r3b, r1b, out + pitch, dmax);
    }
    // black(z-1): row a column E, row b column F; reds z-2, z
    if (z - 1 >= z0 && z - 1 < z1) {
      const T3Row<R> Bn = t3_row(sl[1], oa - WX), Bs = t3_row(sl[1], ob + WX);
      const R Boa = sl[1][oa + (E == 0 ? -1 : 2)], Bob = sl[1][ob + (F == 0 ? -1 : 2)];
      t3_black<R, CHECK, E>(t, 0, w, Bn, Ba, Bb, Boa, r2a, rza, out + zstride, dmax);
      t3_black<R, CHECK, F>(t, 1, w, Ba, Bb, Bs, Bob, r2b, rzb, out + zstride + pitch, dmax);
    }
    out += 2 * zstride;
    r3a = r1a;
    r2a = rza;
    r1a = rz1a;
    r3b = r1b;
    r2b = rzb;
    r1b = rz1b;
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
