// wave_launch.cuh — launchers of the wave (K3/K4) and Jacobi kernels, one
// explicit instantiation per (dtype, depth) translation unit (wave_*.cu,
// jacobi_inst.cu) so the library builds in parallel.
#pragma once

#include "sor_internal.h"
#include "wave2.cuh"

namespace sorh {

template <typename R>
constexpr int wave_nst() { return 14; }

template <typename R, int T, int CK, bool SPLIT, int NC, bool LINK>
int launch_wave_TS(sor_grid* g, const Slab& s, R w, const IterCtl& ctl, bool fused_fin) {
  constexpr int NST = wave_nst<R>();
  constexpr int smem = wave_smem_bytes<R, NST, SPLIT, NC>();
  constexpr int per_cta = wave_tiles_per_cta(SPLIT);
  static int occ_dev[kMaxDev] = {};  // resident CTAs/SM for this instance, per device
  int& occ = occ_dev[g->device % kMaxDev];
  if (occ == 0) {
    CU(cudaFuncSetAttribute(wave_kernel<R, T, NST, CK, SPLIT, NC, LINK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wave_kernel<R, T, NST, CK, SPLIT, NC, LINK>, kWaveWarps * 32, smem);
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
  TRY(wave_tiles(g, s, slab_idx, 2 * T, 2 * T, wave_cols<NC>(), occ * per_cta, SPLIT, a.s0, &tt,
                 ctl.defer ? per_cta : 0));
  a.tiles = tt.first;
  a.ntiles = tt.second;
  a.link = make_link(g, s, g->cur, g->nxt(g->cur));
  record_layout(g, g->nxt(g->cur), a.s0, wave_cols<NC>(), 2 * T, strips_of(g, a.s0, wave_cols<NC>(), 2 * T));
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
  // PDL only for one-wave launches (wave_pdl)
  // the deferred decision block (block 0) exits at once: still one wave
  cfg.numAttrs = wave_pdl(g, blocks - (ctl.defer ? 1u : 0u), occ) ? 1 : 0;
  CU(cudaLaunchKernelEx(&cfg, wave_kernel<R, T, NST, CK, SPLIT, NC, LINK>, a, c, s.tmap[g->cur]));
  g->st.kernel_launches += 1;
  return SOR_OK;
}

// The skew-2 schedule (wave2.cuh): the same tiles and launch protocol.
template <typename R, int T, int CK, bool LINK, int RING>
int launch_wave2_TR(sor_grid* g, const Slab& s, R w, const IterCtl& ctl, bool fused_fin) {
  constexpr bool SPLIT = T >= 2;
  constexpr int NC = kWaveNC;
  constexpr int smem = wave2_smem_bytes<R, SPLIT, NC, RING>();
  constexpr int per_cta = wave_tiles_per_cta(SPLIT);
  static int occ_dev[kMaxDev] = {};
  int& occ = occ_dev[g->device % kMaxDev];
  if (occ == 0) {
    CU(cudaFuncSetAttribute(wave2_kernel<R, T, CK, SPLIT, NC, LINK, RING>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wave2_kernel<R, T, CK, SPLIT, NC, LINK, RING>, kWaveWarps * 32, smem);
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
  TRY(wave_tiles(g, s, slab_idx, 2 * T, 2 * T, wave_cols<NC>(), occ * per_cta, SPLIT, a.s0, &tt,
                 ctl.defer ? per_cta : 0));
  a.tiles = tt.first;
  a.ntiles = tt.second;
  a.link = make_link(g, s, g->cur, g->nxt(g->cur));
  record_layout(g, g->nxt(g->cur), a.s0, wave_cols<NC>(), 2 * T, strips_of(g, a.s0, wave_cols<NC>(), 2 * T));
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
  // the deferred decision block (block 0) exits at once: still one wave
  cfg.numAttrs = wave_pdl(g, blocks - (ctl.defer ? 1u : 0u), occ) ? 1 : 0;
  CU(cudaLaunchKernelEx(&cfg, wave2_kernel<R, T, CK, SPLIT, NC, LINK, RING>, a, c, s.tmap2[g->cur]));
  g->st.kernel_launches += 1;
  return SOR_OK;
}

template <typename R, int T, int CK, bool LINK>
int launch_wave2_T(sor_grid* g, const Slab& s, R w, const IterCtl& ctl, bool fused_fin) {
  // a deeper TMA look-ahead pays for one-wave launches at T = 4 (C3-sized
  // slabs); multi-wave launches (C4, C5) and T < 4 keep the smaller ring
  const double cells = (double)(s.g_hi - s.g_lo) * (double)g->cols;
  if (T >= 4 && cells <= 64.0 * (1 << 20)) return launch_wave2_TR<R, T, CK, LINK, 3>(g, s, w, ctl, fused_fin);
  return launch_wave2_TR<R, T, CK, LINK, 2>(g, s, w, ctl, fused_fin);
}

template <typename R, int T, int CK, bool LINK>
int launch_wave_T(sor_grid* g, const Slab& s, R w, const IterCtl& ctl, bool fused_fin) {
  // 4 columns per lane: wider lanes (NC = 6, 8; bitwise equal) measured
  // slower on B200 at every T (fewer resident warps outweigh the extra ILP).
  // T >= 2: warp pairs (split).
  return launch_wave_TS<R, T, CK, (T >= 2), kWaveNC, LINK>(g, s, w, ctl, fused_fin);
}

// K6: `npasses` T-deep passes in one cooperative launch (L2-resident grids;
// see wave_persist_kernel).  Returns SOR_E_UNSUPPORTED if the tiles do not fit
// in one wave of co-resident CTAs (the caller then launches pass by pass).
template <typename R, int T, bool W2>
int launch_wave_persist_S(sor_grid* g, const Slab& s, R w, int npasses, unsigned* gbar) {
  constexpr int NST = wave_nst<R>();
  constexpr bool SPLIT = T >= 2;
  constexpr int NC = kWaveNC;
  constexpr int smem = W2 ? wave2_smem_bytes<R, SPLIT, NC, 2>() : wave_smem_bytes<R, NST, SPLIT, NC>();
  auto kern = W2 ? wave2_persist_kernel<R, T, SPLIT, NC> : wave_persist_kernel<R, T, NST, SPLIT, NC>;
  constexpr int per_cta = wave_tiles_per_cta(SPLIT);
  static int occ_dev[kMaxDev] = {};
  int& occ = occ_dev[g->device % kMaxDev];
  if (occ == 0) {
    CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kWaveWarps * 32, smem);
    if (occ <= 0) occ = 1;
  }
  WaveArgs<R> a;
  a.src = col0<R>(s.plane[0]);
  a.dst = col0<R>(s.plane[1]);
  a.pitch = g->pitch;
  a.g0 = s.g0;
  a.rows = g->rows;
  a.cols = g->cols;
  a.r_lo = s.g_lo;
  a.r_hi = s.g_hi;
  a.w = w;
  a.s0 = -4 * ((2 * T + 3) / 4);
  // tiles per SM: half the one-wave budget of an ordinary launch (taller
  // bands, less warm-up per pass; measured best on C2 at T = 3, 4:
  // profiles/r2_c2_persistent.txt); SOR_PERSIST_TPS overrides
  static int tps = -1;
  if (tps < 0) {
    const char* e = getenv("SOR_PERSIST_TPS");
    tps = e ? atoi(e) : 0;
  }
  const int budget = tps > 0 ? std::min(tps, occ * per_cta) : std::max(1, occ * per_cta / 2);
  std::pair<int4*, int> tt{nullptr, 0};
  TRY(wave_tiles(g, s, 0, 2 * T, 2 * T, wave_cols<NC>(), budget, SPLIT, a.s0, &tt));
  a.tiles = tt.first;
  a.ntiles = tt.second;
  const unsigned blocks = (unsigned)((a.ntiles + per_cta - 1) / per_cta);
  if (blocks > (unsigned)(occ * g->nsm)) return SOR_E_UNSUPPORTED;
  // planes alternate pass by pass starting from the current one
  const int p0 = g->cur, p1 = g->nxt(g->cur);
  a.src = col0<R>(s.plane[p0]);
  a.dst = col0<R>(s.plane[p1]);
  CU(cudaMemsetAsync(gbar, 0, sizeof(unsigned), g->stream));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kWaveWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = g->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = W2 ? cudaLaunchKernelEx(&cfg, kern, a, npasses, gbar, s.tmap2[p0], s.tmap2[p1])
                           : cudaLaunchKernelEx(&cfg, kern, a, npasses, gbar, s.tmap[p0], s.tmap[p1]);
  if (e == cudaErrorCooperativeLaunchTooLarge) {
    cudaGetLastError();  // not co-resident now (other work on the device): pass-by-pass launches instead
    return SOR_E_UNSUPPORTED;
  }
  CU(e);
  g->st.kernel_launches += 1;
  return SOR_OK;
}

template <typename R, int T>
int launch_wave_persist(sor_grid* g, const Slab& s, R w, int npasses, unsigned* gbar) {
  if constexpr (T >= 2) {
    if (use_wave2(g, T)) return launch_wave_persist_S<R, T, true>(g, s, w, npasses, gbar);
  }
  return launch_wave_persist_S<R, T, false>(g, s, w, npasses, gbar);
}

// Jacobi pass (NEXT-2): jacobi_kernel on the wave tiles with ghost G and T stages.
template <typename R, int T, int CK, bool LINK>
int launch_jacobi_T(sor_grid* g, const Slab& s, const IterCtl& ctl, bool fused_fin) {
  constexpr int NST = wave_nst<R>();
  constexpr int smem = kWaveWarps * wave_smem_per_warp<R, NST, kWaveNC>();
  constexpr int G = jacobi_ghost(T);
  static int occ_dev[kMaxDev] = {};
  int& occ = occ_dev[g->device % kMaxDev];
  if (occ == 0) {
    CU(cudaFuncSetAttribute(jacobi_kernel<R, T, NST, CK, LINK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, jacobi_kernel<R, T, NST, CK, LINK>, kWaveWarps * 32, smem);
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
  TRY(wave_tiles(g, s, slab_idx, G, T, wave_cols<kWaveNC>(), occ * kWaveWarps, false, a.s0, &tt,
                 ctl.defer ? kWaveWarps : 0));
  a.tiles = tt.first;
  a.ntiles = tt.second;
  a.link = make_link(g, s, g->cur, g->nxt(g->cur));
  record_layout(g, g->nxt(g->cur), a.s0, wave_cols<kWaveNC>(), G, strips_of(g, a.s0, wave_cols<kWaveNC>(), G));
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
  // the deferred decision block (block 0) exits at once: still one wave
  cfg.numAttrs = wave_pdl(g, blocks - (ctl.defer ? 1u : 0u), occ) ? 1 : 0;
  CU(cudaLaunchKernelEx(&cfg, jacobi_kernel<R, T, NST, CK, LINK>, a, c, s.tmap[g->cur]));
  g->st.kernel_launches += 1;
  return SOR_OK;
}

}  // namespace sorh
