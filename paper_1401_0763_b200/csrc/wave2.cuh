// wave2.cuh — skew-2 wavefront variant of the temporally blocked wave kernel
// (K4).  Same tiles, layout, arithmetic and max-change modes
// as wave_kernel (sor_kernels.cuh); only the schedule of the stages differs.
//
// wave_kernel's stage s updates row i-s at step m (front row i), so within a
// step stage s needs stage s-1's row of the SAME step: every step is a serial
// chain of 2T stages (a shuffle, then six dependent FP64 operations each).
// Here stage s updates row i-2s: the rows r-1, r, r+1 it needs from stage s-1
// were produced at steps m-3, m-2, m-1, and its own old value (stage s-2's row
// r) at step m-4, so the 2T stages of a step are independent and the
// scheduler can overlap them.  Rings hold the outputs of the last four steps
// (slot = step mod 4); the stages of a step run in DESCENDING order, so stage
// s+2 reads slot m mod 4 of stage s (step m-4) before stage s overwrites it.
// Source rows arrive in 4-row TMA boxes; the loop is unrolled over one ring
// period (4 steps x 2 row parities fold into the same period).  The result is
// bitwise that of wave_kernel (every cell reads the same operand values).
#pragma once

#include "sor_kernels.cuh"

namespace sorb {

constexpr int kW2Batch = 4;  // steps (source rows) per TMA box / unrolled loop body
// RING = source batches in flight (TMA look-ahead): 3 for one-wave launches
// (C3: +3 %), 2 otherwise (C5, T < 4: the smaller footprint is faster)
template <int RING>
__host__ __device__ constexpr int wave2_slots() { return RING * kW2Batch + 3; }  // + 3 prologue rows (rel -2, -1, 0)

template <typename R, int NC, int RING>
__host__ __device__ constexpr int wave2_smem_per_warp() {
  return (wave2_slots<RING>() * wave_cols<NC>() * (int)sizeof(R) + (RING + 1) * 8 + 127) / 128 * 128;
}
template <typename R, int NC>
__host__ __device__ constexpr int wave2_handoff_bytes() {
  return 2 * kW2Batch * 32 * NC * (int)sizeof(R);  // 2 batches x 4 steps x 32 lanes x NC values
}
template <typename R, int NC, int RING>
__host__ __device__ constexpr int wave2_smem_per_pair() {
  return wave2_smem_per_warp<R, NC, RING>() + wave2_handoff_bytes<R, NC>();
}
template <typename R, bool SPLIT, int NC, int RING>
__host__ __device__ constexpr int wave2_smem_bytes() {
  return SPLIT ? (kWaveWarps / 2) * wave2_smem_per_pair<R, NC, RING>() : kWaveWarps * wave2_smem_per_warp<R, NC, RING>();
}
#ifndef SOR_WAVE2_K4
#define SOR_WAVE2_K4 3
#endif
__host__ __device__ constexpr int wave2_split_stage(int T) { return T == 4 ? SOR_WAVE2_K4 : T; }

// Warp pipeline: stages [SB, SE) of S = 2T.  Step t (relative to the tile's
// first front row i_first, even): the front row is rel t; stage s updates row
// rel t-2s, colour s&1, cells q = O + 2h with O = (s + t) & 1.
template <typename R, int T, int CK, int SB, int SE, int NC, int RING>
struct WavePipe2 {
  static constexpr int kW2Ring = RING;
  static constexpr int S = 2 * T;
  static constexpr int NH = NC / 2;
  static constexpr int WC = wave_cols<NC>();
  static constexpr int NSLOT = CK >= 2 ? T : 1;
  static constexpr bool LANE_OWN = (2 * T) % NC == 0;
  static constexpr uint32_t ROWB = WC * sizeof(R);
  static constexpr int CH = 16 / (int)sizeof(R);
  // CK 4 probes the red stages on rows with rel % 8 == 0: rel % 4 == 0 is
  // static per step and stage (rel = t - 2s), the batch parity selects half
  __host__ __device__ static constexpr bool probe_row(int M, int s) { return (((M - 2 * s) % 4) + 4) % 4 == 0; }
  R F[4][NC];                 // source rows, slot = rel mod 4 (front warp)
  R C[S > 1 ? S - 1 : 1][4][NH];  // stage outputs, slot = step mod 4
  unsigned long long dmax[CK == 1 || CK == 2 ? NSLOT : 1];
  unsigned int hmax[CK >= 3 ? NSLOT : 1];
  unsigned int ownM[NH];
  unsigned int pf;            // CK 4: all-ones iff this batch's probe rows are owned (see run_range)
  bool upd[NC];
  bool ownP[NH];
  int rows, R0, R1, i_first;
  int col_mask;
  R* orow;
  const R* ring;
  uint32_t ring_s, bar_s;
  const CUtensorMap* tm;      // 4-row boxes
  const CUtensorMap* tm3;     // 3-row box (prologue)
  int tm_x, tm_y;             // storage (column, row) of (s_w, rel -2)
  long long pitch;
  int nbatch;
  int lane;
  R* hand;
  int bar_full, bar_empty;

  __device__ __forceinline__ void issue_batch_tma(int j) {
    const int b = j % kW2Ring;
    const uint32_t bar = bar_s + 8u * b;
    mbar_expect_tx(bar, kW2Batch * ROWB);
    tma_rows(ring_s + b * kW2Batch * ROWB, tm, tm_x, tm_y + kW2Batch * j + 3, bar);  // rows rel 4j+1..4j+4
  }
  __device__ __forceinline__ void issue_prologue() {
    const uint32_t bar = bar_s + 8u * kW2Ring;
    mbar_expect_tx(bar, 3 * ROWB);
    tma_rows(ring_s + kW2Ring * kW2Batch * ROWB, tm3, tm_x, tm_y, bar);  // rows rel -2, -1, 0
  }
  __device__ __forceinline__ void ld_row(const R* row, R (&x)[NC]) { ldsN<NC>(row + NC * lane, x); }
  __device__ __forceinline__ void hand_st(R* hp, int M, const R (&x)[NC]) {
#pragma unroll
    for (int k = 0; k < NC / CH; ++k) {
      R* q = hp + ((M * (NC / CH) + k) * 32 + lane) * CH;
      if (sizeof(R) == 8)
        *reinterpret_cast<double2*>(q) = make_double2((double)x[2 * k], (double)x[2 * k + 1]);
      else
        *reinterpret_cast<float4*>(q) = make_float4((float)x[4 * k], (float)x[4 * k + 1], (float)x[4 * k + 2],
                                                    (float)x[4 * k + 3]);
    }
  }
  __device__ __forceinline__ void hand_ld(const R* hp, int M, R (&x)[NC]) {
#pragma unroll
    for (int k = 0; k < NC / CH; ++k) {
      const R* q = hp + ((M * (NC / CH) + k) * 32 + lane) * CH;
      if (sizeof(R) == 8) {
        const double2 v = *reinterpret_cast<const double2*>(q);
        x[2 * k] = (R)v.x;
        x[2 * k + 1] = (R)v.y;
      } else {
        const float4 v = *reinterpret_cast<const float4*>(q);
        x[4 * k] = (R)v.x;
        x[4 * k + 1] = (R)v.y;
        x[4 * k + 2] = (R)v.z;
        x[4 * k + 3] = (R)v.w;
      }
    }
  }

  // One stage at step t = 4j + M: row rel t - 2s.  `uext` (stage SB of the back
  // warp) is the old value handed over by the front warp.
  template <int MK, int M, int s>
  __device__ __forceinline__ void stage(const WaveArgs<R>& a, int t, const R* uext) {
    constexpr int O = (s + M) & 1;
    constexpr int Q1 = (M + 3) & 3;  // slot of step t-1
    constexpr int Q2 = (M + 2) & 3;  // t-2
    constexpr int Q3 = (M + 1) & 3;  // t-3
    const int r = i_first + t - 2 * s;
    R n[NH], sv[NH], w[NH], u[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      if (s == 0) {
        // source rows rel t-1, t+1 (N/S), rel t (W/E and self)
        n[h] = F[(M + 3) & 3][O + 2 * h];
        sv[h] = F[(M + 1) & 3][O + 2 * h];
        w[h] = F[M][1 - O + 2 * h];
        u[h] = F[M][O + 2 * h];
      } else {
        const int p = s > 0 ? s - 1 : 0;
        n[h] = C[p][Q3][h];   // row r-1 (step t-3)
        sv[h] = C[p][Q1][h];  // row r+1 (step t-1)
        w[h] = C[p][Q2][h];   // row r (step t-2), other colour
        if (s == SB && SB > 0) {
          u[h] = uext[h];                      // stage s-2's row r (step t-4), from the front
        } else if (s == 1) {
          u[h] = F[(M + 2) & 3][O + 2 * h];  // source row rel t-2
        } else {
          const int pp = s >= 2 ? s - 2 : 0;
          u[h] = C[pp][M][h];                  // stage s-2's row r (step t-4), not yet overwritten
        }
      }
    }
    const R nb = (O == 0) ? shfl_up1(w[NH - 1]) : shfl_dn1(w[0]);
    R v[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      const R we = (O == 0) ? radd(h == 0 ? nb : w[h > 0 ? h - 1 : 0], w[h])
                            : radd(w[h], h == NH - 1 ? nb : w[h < NH - 1 ? h + 1 : 0]);
      v[h] = sor_update(radd(n[h], sv[h]), we, u[h], a.w);
      if (MK == 1) {
        v[h] = upd[O + 2 * h] ? v[h] : u[h];
      } else if (MK == 2) {
        const bool rowok = (unsigned)(r - 1) < (unsigned)rows;
        v[h] = (rowok && upd[O + 2 * h]) ? v[h] : u[h];
      }
    }
    if (CK == 4 && (s & 1) == 0 && probe_row(M, s)) {
      if (pf)  // even batches only: probe rows with rel % 8 == 0
#pragma unroll
      for (int h = 0; h < NH; ++h)
        hmax[s >> 1] = max(hmax[s >> 1], (unsigned int)hi_bits(rsub(v[h], u[h])) & ownM[h] & pf &
                                             ((unsigned)(r - R0) < (unsigned)(R1 - R0) ? 0xffffffffu : 0u));
    } else if (CK == 3) {
      const unsigned int fill = (unsigned)(r - R0) < (unsigned)(R1 - R0) ? 0xffffffffu : 0u;
#pragma unroll
      for (int h = 0; h < NH; ++h)
        hmax[s >> 1] = max(hmax[s >> 1], (unsigned int)hi_bits(rsub(v[h], u[h])) & ownM[h] & fill);
    } else if (CK != 0 && (CK == 2 || s >= S - 2)) {
      const bool inb = (unsigned)(r - R0) < (unsigned)(R1 - R0);
      const int slot = CK == 2 ? (s >> 1) : 0;
#pragma unroll
      for (int h = 0; h < NH; ++h)
        dmax[slot] = umax64(dmax[slot], (inb && ownP[h]) ? delta_bits(v[h], u[h]) : 0ull);
    }
    if (s < S - 1) {
#pragma unroll
      for (int h = 0; h < NH; ++h) C[s][M][h] = v[h];
    } else {
      // finished row r: this colour at q = O+2h, the other from stage S-2's
      // row r (step t-2, positions 1-O+2h)
      const bool inb = (unsigned)(r - R0) < (unsigned)(R1 - R0);
      R out[NC];
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        out[O + 2 * h] = v[h];
        out[1 - O + 2 * h] = C[S - 2][Q2][h];
      }
      if (LANE_OWN && NC % 4 == 0) {
#pragma unroll
        for (int k = 0; k < NC / 4; ++k)
          stg4_if(inb && ownP[0], orow + 4 * k, out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
      } else if (NC == 4) {
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

  // Stages [lo, hi) in descending order.
  template <int MK, int M, int s, int lo>
  __device__ __forceinline__ void stages_desc(const WaveArgs<R>& a, int t, const R* uext) {
    if constexpr (s >= lo) {
      stage<MK, M, s>(a, t, uext);
      stages_desc<MK, M, s - 1, lo>(a, t, uext);
    }
  }

  template <int MK, int M>
  __device__ __forceinline__ void step(const WaveArgs<R>& a, int t, const R* rowp, R* hp) {
    if (SB == 0) {
      ld_row(rowp + M * WC, F[(M + 1) & 3]);  // source row rel t+1
      if (SE < S) {
        // front of a pair: the back's first stage SE needs stage SE-1's rows
        // of steps t-1..t-3 (handed over as they are produced) and stage
        // SE-2's row of step t-4 (its old value, slot M before stage SE-2
        // overwrites it this step)
        stages_desc<MK, M, SE - 1, SE - 1>(a, t, nullptr);
        R x[NC];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          x[h] = C[SE - 1][M][h];
          x[NH + h] = C[SE >= 2 ? SE - 2 : 0][M][h];
        }
        hand_st(hp, M, x);
        stages_desc<MK, M, SE - 2, 0>(a, t, nullptr);
      } else {
        stages_desc<MK, M, SE - 1, 0>(a, t, nullptr);
      }
    } else {
      R x[NC];
      hand_ld(hp, M, x);
      // stages above SB first: stage SB+1 reads slot M of the received ring
      // (step t-4) before this step's row is stored there
      stages_desc<MK, M, SE - 1, SB + 1>(a, t, nullptr);
#pragma unroll
      for (int h = 0; h < NH; ++h) C[SB - 1][M][h] = x[h];
      R ue[NH];
#pragma unroll
      for (int h = 0; h < NH; ++h) ue[h] = x[NH + h];
      stage<MK, M, SB>(a, t, ue);
    }
  }

  template <int MK>
  __device__ __forceinline__ void batch(const WaveArgs<R>& a, int t, const R* rowp, R* hp) {
    step<MK, 0>(a, t, rowp, hp);
    step<MK, 1>(a, t + 1, rowp, hp);
    step<MK, 2>(a, t + 2, rowp, hp);
    step<MK, 3>(a, t + 3, rowp, hp);
  }

  template <int MK>
  __device__ __forceinline__ void run_range(const WaveArgs<R>& a, int j0, int j1) {
    constexpr bool front = SB == 0;
    constexpr bool split = !(front && SE == S);
#pragma unroll 1
    for (int j = j0; j < j1; ++j) {
      const int t = kW2Batch * j;
      // CK 4: probe rows (rel % 8 == 0) only in even batches; ownership is
      // tested per row in stage()
      if (CK == 4) pf = (j & 1) ? 0u : 0xffffffffu;
      const R* rowp = nullptr;
      R* hp = split ? hand + (j & 1) * (kW2Batch * 32 * NC) : nullptr;
      if (front) {
        const int b = j % kW2Ring;
        mbar_wait(bar_s + 8u * b, (uint32_t)((j / kW2Ring) & 1));
        rowp = ring + b * kW2Batch * WC;
        if (split) named_bar_sync(bar_empty + (j & 1), 64);
      } else {
        named_bar_sync(bar_full + (j & 1), 64);
      }
      batch<MK>(a, t, rowp, hp);
      if (front) {
        if (split) named_bar_arrive(bar_full + (j & 1), 64);
        __syncwarp();
        if (lane == 0 && j + kW2Ring < nbatch) issue_batch_tma(j + kW2Ring);
      } else if (j + 2 < nbatch) {
        named_bar_arrive(bar_empty + (j & 1), 64);
      }
    }
  }

  __device__ __forceinline__ void run(const WaveArgs<R>& a) {
    constexpr bool front = SB == 0, back = SE == S;
    constexpr bool split = !(front && back);
    if (split && !front) {
      named_bar_arrive(bar_empty + 0, 64);
      if (nbatch > 1) named_bar_arrive(bar_empty + 1, 64);
    }
    // batch j updates rows i_first + 4j - 2(S-1) .. i_first + 4j + 3; they
    // are all in [1, rows] for jA <= j < jB
    const int lo_need = 1 - i_first + 2 * (S - 1);  // 4j >= lo_need
    const int jA = min(nbatch, max(0, lo_need > 0 ? (lo_need + 3) / 4 : 0));
    const int hi_lim = rows - 3 - i_first;          // 4j <= hi_lim
    const int jB = max(jA, min(nbatch, hi_lim >= 0 ? hi_lim / 4 + 1 : 0));
    run_range<2>(a, 0, jA);
    if (col_mask)
      run_range<1>(a, jA, jB);
    else
      run_range<0>(a, jA, jB);
    run_range<2>(a, jB, nbatch);
  }
};

template <typename R, int T, int CK, int SB, int SE, int NC, int RING>
__device__ __forceinline__ void wave2_tile(const WaveArgs<R>& a, const CUtensorMap* tm4, const CUtensorMap* tm3,
                                           unsigned char* wbase, R* hand, int bar_id, int lane, int sw, int R0, int R1,
                                           int i_first, int nsteps, unsigned long long (&dm)[kMaxT]) {
  using Pipe = WavePipe2<R, T, CK, SB, SE, NC, RING>;
  constexpr int kW2Ring = RING;
  constexpr int WC = Pipe::WC, NH = Pipe::NH;
  Pipe P;
#pragma unroll
  for (int t = 0; t < P.NSLOT; ++t) {
    if (CK == 1 || CK == 2) P.dmax[t] = 0ull;
    if (CK >= 3) P.hmax[t] = 0u;
  }
  P.ring = reinterpret_cast<const R*>(wbase);
  P.ring_s = smem_u32(wbase);
  P.bar_s = P.ring_s + wave2_slots<RING>() * WC * sizeof(R);
  P.hand = hand;
  P.bar_full = bar_id;
  P.bar_empty = bar_id + 2;
  P.lane = lane;
  P.rows = (int)a.rows;
  P.R0 = R0;
  P.R1 = R1;
  P.i_first = i_first;
  const long long c0 = (long long)sw + NC * lane;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    const int c = (int)c0 + q;
    P.upd[q] = (c >= 1) && (c <= (int)a.cols);
  }
  P.col_mask = (sw >= 1 && sw + WC - 1 <= (int)a.cols) ? 0 : 1;
  {
    const int g_lo = sw + 2 * T, g_hi = sw + WC - 2 * T;
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      const int cp = (int)c0 + 2 * h;
      P.ownP[h] = cp >= g_lo && cp + 1 < g_hi;
      P.ownM[h] = P.ownP[h] ? 0x7fffffffu : 0u;
    }
  }
  // row finished by stage S-1 at step 0 is rel -2(S-1)
  P.orow = a.dst + (long long)(i_first - 2 * (2 * T - 1) - a.g0) * a.pitch + c0;
#pragma unroll
  for (int s = 0; s < 2 * T - 1; ++s)
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int h = 0; h < NH; ++h) P.C[s][k][h] = R(0);
  P.pitch = a.pitch;
  P.tm = tm4;
  P.tm3 = tm3;
  P.tm_x = kColPad + sw;
  P.tm_y = i_first - 2 - (int)a.g0;
  P.nbatch = nsteps / kW2Batch;
  if (SB == 0) {
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < kW2Ring + 1; ++k) mbar_init(P.bar_s + 8u * k, 1u);
      mbar_fence_init();
    }
    __syncwarp();
    if (lane == 0) {
      P.issue_prologue();
      for (int j = 0; j < kW2Ring && j < P.nbatch; ++j) P.issue_batch_tma(j);
    }
    mbar_wait(P.bar_s + 8u * kW2Ring, 0u);
    const R* pro = P.ring + kW2Ring * kW2Batch * WC;
    P.ld_row(pro, P.F[2]);           // rel -2 -> slot 2
    P.ld_row(pro + WC, P.F[3]);      // rel -1 -> slot 3
    P.ld_row(pro + 2 * WC, P.F[0]);  // rel 0  -> slot 0
  }
  P.run(a);
#pragma unroll
  for (int t = 0; t < P.NSLOT; ++t)
    dm[t] = CK >= 3 ? (unsigned long long)P.hmax[t] : P.dmax[(CK == 1 || CK == 2) ? t : 0];
}

// The kernel: wave_kernel's launch protocol (PDL, stop test, deferred
// decision, max reduction) around wave2_tile.  Tensor maps: m[0] 4-row and
// m[1] 3-row boxes (wave2 maps of the source plane).
template <typename R, int T, int CK, bool SPLIT, int NC, bool LINK, int RING>
__global__ void __launch_bounds__(kWaveWarps * 32, wave_min_blocks(T, SPLIT, NC))
    wave2_kernel(WaveArgs<R> a, IterCtl ctl, const __grid_constant__ WaveMaps tm) {
  const int bid = (int)blockIdx.x - ctl.defer;
  extern __shared__ __align__(128) unsigned char wave_smem[];
  constexpr int WC = wave_cols<NC>();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int slot = SPLIT ? warp >> 1 : warp;
  const int role = SPLIT ? warp & 1 : 0;
  const int gw = bid * wave_tiles_per_cta(SPLIT) + slot;
  const bool has_tile = bid >= 0 && gw < a.ntiles;
  const int4 tile = has_tile ? a.tiles[gw] : make_int4(0, 0, 0, 0);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (ctl.st && ctl.solve) {
    if (ctl.defer && blockIdx.x == 0) {
      if (threadIdx.x == 0 && ctl.prev_valid && !ld_stop(ctl.st))
        finalize_pass(ctl.st, ctl, ctl.prev_k_last, ctl.prev_T, ctl.prev_ck, ctl.prev_set, ctl.prev_seq);
      return;
    }
    __shared__ int cta_stop;
    if (threadIdx.x == 0) cta_stop = ld_stop(ctl.st);
    __syncthreads();
    if (cta_stop) return;
  }
  unsigned long long dm[kMaxT] = {};
  if (has_tile) {
    const int sw = a.s0 + tile.x * (WC - 4 * T);
    const int R0 = tile.y, R1 = tile.z;
    const int i_first = (R0 - (2 * T - 1)) & ~1;
    const int nsteps = (R1 - i_first + 2 * (2 * T - 1) + kW2Batch - 1) / kW2Batch * kW2Batch;
    if (LINK && role == 0) tile_halo_wait(a, sw, WC, R0, R1, 2 * T, lane, ctl.st);
    if (SPLIT) {
      unsigned char* pbase = wave_smem + slot * wave2_smem_per_pair<R, NC, RING>();
      R* hand = reinterpret_cast<R*>(pbase + wave2_smem_per_warp<R, NC, RING>());
      const int bar_id = 1 + 4 * slot;
      constexpr int K = wave2_split_stage(T);
      if (role == 0)
        wave2_tile<R, T, CK, 0, K, NC, RING>(a, &tm.m[0], &tm.m[1], pbase, hand, bar_id, lane, sw, R0, R1, i_first, nsteps,
                                       dm);
      else
        wave2_tile<R, T, CK, K, 2 * T, NC, RING>(a, &tm.m[0], &tm.m[1], pbase, hand, bar_id, lane, sw, R0, R1, i_first,
                                           nsteps, dm);
    } else {
      unsigned char* wbase = wave_smem + warp * wave2_smem_per_warp<R, NC, RING>();
      wave2_tile<R, T, CK, 0, 2 * T, NC, RING>(a, &tm.m[0], &tm.m[1], wbase, nullptr, 0, lane, sw, R0, R1, i_first, nsteps,
                                         dm);
    }
  }
  if (LINK && (!SPLIT || role == 1)) {
    const int gw2 = ((int)blockIdx.x - ctl.defer) * wave_tiles_per_cta(SPLIT) +
                    (SPLIT ? (int)(threadIdx.x >> 6) : (int)(threadIdx.x >> 5));
    if ((int)blockIdx.x >= ctl.defer && gw2 < a.ntiles) {
      const int4 t2 = a.tiles[gw2];
      tile_halo_push<R, NC>(a, a.s0 + t2.x * (WC - 4 * T), WC, 2 * T, t2.x, t2.y, t2.z, (int)(threadIdx.x & 31));
    }
  }
  if (CK != 0) {
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

// K6 with the skew-2 tiles: `npasses` T-deep passes in one cooperative
// launch, grid barrier between passes (see wave_persist_kernel).
template <typename R, int T, bool SPLIT, int NC>
__global__ void __launch_bounds__(kWaveWarps * 32, wave_min_blocks(T, SPLIT, NC))
    wave2_persist_kernel(WaveArgs<R> a, int npasses, unsigned* gbar, const __grid_constant__ WaveMaps tmA,
                         const __grid_constant__ WaveMaps tmB) {
  constexpr int RING = 2;
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
      const int nsteps = (R1 - i_first + 2 * (2 * T - 1) + kW2Batch - 1) / kW2Batch * kW2Batch;
      unsigned char* base = SPLIT ? wave_smem + slot * wave2_smem_per_pair<R, NC, RING>()
                                  : wave_smem + warp * wave2_smem_per_warp<R, NC, RING>();
      if (SPLIT) {
        R* hand = reinterpret_cast<R*>(base + wave2_smem_per_warp<R, NC, RING>());
        const int bar_id = 1 + 4 * slot;
        constexpr int K = wave2_split_stage(T);
        if (role == 0)
          wave2_tile<R, T, 0, 0, K, NC, RING>(ap, &tm[0], &tm[1], base, hand, bar_id, lane, sw, R0, R1, i_first, nsteps,
                                              dm);
        else
          wave2_tile<R, T, 0, K, 2 * T, NC, RING>(ap, &tm[0], &tm[1], base, hand, bar_id, lane, sw, R0, R1, i_first,
                                                  nsteps, dm);
      } else {
        wave2_tile<R, T, 0, 0, 2 * T, NC, RING>(ap, &tm[0], &tm[1], base, nullptr, 0, lane, sw, R0, R1, i_first, nsteps,
                                                dm);
      }
      if (role == 0 && lane == 0) {
        const uint32_t bar = smem_u32(base) + wave2_slots<RING>() * WC * (uint32_t)sizeof(R);
#pragma unroll
        for (int k = 0; k < RING + 1; ++k) mbar_inval(bar + 8u * k);
      }
    }
    if (p + 1 < npasses) grid_barrier(gbar, (unsigned)(p + 1) * gridDim.x);
  }
}

}  // namespace sorb
