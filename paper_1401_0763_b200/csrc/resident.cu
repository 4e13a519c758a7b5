// resident.cu — K7 launchers (see resident.cuh): the grid register-resident
// across the SMs.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "resident.cuh"
#include "sor_internal.h"

namespace sorh {

namespace {

constexpr int kResNC = 4;  // columns per lane: a window is 128 columns wide
constexpr int kResWW = 32 * kResNC;

struct ResShape {
  int rpw, cps;
};
// Instances, in order of preference for the multi-CTA form: two CTAs per SM
// with 2 rows per warp (twice the warps per SM: the updates of one warp run
// as dependent chains, so latency is hidden by warps), else one CTA per SM.
constexpr ResShape kMultiShapes[] = {{4, 1}, {6, 1}, {2, 2}};
constexpr ResShape kSingleShapes[] = {{4, 1}, {6, 1}, {8, 1}};
int res_max_warps(int rpw, int cps) { return res_max_threads(rpw, cps) / 32; }

struct ResPlan {
  int nbx = 1, nby = 1, rpw = 4, cps = 1, nw = 1, nc = kResNC;
};

int env_int(const char* name) {
  const char* e = getenv(name);
  return e ? atoi(e) : 0;
}

// Block grid and window shape.  Multi-CTA: the window (block + G ring, origin
// rounded down to even) must fit 128 columns x rpw*nw rows, every block must
// be at least G cells in each direction (its ring then lies in the 8
// neighbouring blocks' frames), and all blocks must be co-resident (cps per
// SM; the neighbour waits cannot deadlock).  As many blocks as that allows:
// the time of a pass is that of one window.
bool res_plan(const sor_grid* g, int T, bool single, ResPlan* out) {
  static const int force_rpw = env_int("SOR_RES_RPW");  // A/B of the instances
  if (single) {
    // <= 64 interior columns: 2 columns per lane, window = interior columns
    // (+ one row above the ring so the colour pattern stays compile-time)
    if (g->cols <= 64 && (g->rows + 3 + 3) / 4 <= res_max_warps(4, 1)) {
      *out = ResPlan{1, 1, 4, 1, (int)((g->rows + 3 + 3) / 4), 2};
      return true;
    }
    if (g->cols + 2 > kResWW) return false;
    for (const ResShape& sh : kSingleShapes) {
      const int nw = (int)((g->rows + 2 + sh.rpw - 1) / sh.rpw);
      if (nw <= res_max_warps(sh.rpw, 1)) {
        *out = ResPlan{1, 1, sh.rpw, 1, nw};
        return true;
      }
    }
    return false;
  }
  const int G = 2 * T;
  const int64_t bw_max = kResWW - 2 * G - 1;  // window origin rounded down to even
  if (bw_max < G) return false;
  const int nbx = (int)((g->cols + bw_max - 1) / bw_max);
  if (g->cols / nbx < G) return false;
  for (const ResShape& sh : kMultiShapes) {
    if (force_rpw && sh.rpw != force_rpw) continue;
    const int nby = (int)std::min<int64_t>((int64_t)g->nsm * sh.cps / nbx, g->rows / G);
    if (nby < 1 || nbx * nby < 2) continue;
    const int64_t bh = (g->rows + nby - 1) / nby;
    const int nw = (int)((bh + 2 * G + 1 + sh.rpw - 1) / sh.rpw);
    if (nw <= res_max_warps(sh.rpw, sh.cps)) {
      *out = ResPlan{nbx, nby, sh.rpw, sh.cps, nw};
      return true;
    }
  }
  return false;
}

template <typename R, int RPW, int CPS, int NC = kResNC>
int res_launch(sor_grid* g, const ResPlan& p, const ResArgs<R>& a, bool coop) {
  auto kern = resident_kernel<R, NC, RPW, CPS>;
  const int threads = 32 * p.nw;
  const size_t smem = (size_t)2 * p.nw * 2 * (NC / 2) * 32 * sizeof(R);
  static bool attr_dev[kMaxDev] = {};
  if (!attr_dev[g->device % kMaxDev]) {
    CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(res_max_warps(RPW, CPS) * 2 * 2 * (NC / 2) * 32 * sizeof(R))));
    attr_dev[g->device % kMaxDev] = true;
  }
  if (coop) {  // every block must be resident at once (they wait on each other)
    int occ = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
    static const int verbose = env_int("SOR_RES_VERBOSE");
    if (verbose)
      fprintf(stderr, "K7 plan %dx%d blocks, rpw %d cps %d nw %d, occupancy %d/SM\n", p.nbx, p.nby, p.rpw, p.cps,
              p.nw, occ);
    if (occ * g->nsm < p.nbx * p.nby) return SOR_E_UNSUPPORTED;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p.nbx * p.nby));
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = g->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = coop ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (coop && e == cudaErrorCooperativeLaunchTooLarge) {
    cudaGetLastError();  // not all blocks can be resident now: the caller falls back to the wave path
    return SOR_E_UNSUPPORTED;
  }
  CU(e);
  g->st.kernel_launches += 1;
  return SOR_OK;
}

template <typename R>
int res_dispatch(sor_grid* g, const ResPlan& p, const ResArgs<R>& a, bool coop) {
  if (p.nc == 2) return res_launch<R, 4, 1, 2>(g, p, a, coop);
  if (p.cps == 2) return res_launch<R, 2, 2>(g, p, a, coop);
  switch (p.rpw) {
    case 4: return res_launch<R, 4, 1>(g, p, a, coop);
    case 6: return res_launch<R, 6, 1>(g, p, a, coop);
    default: return res_launch<R, 8, 1>(g, p, a, coop);
  }
}

template <typename R>
ResArgs<R> res_args(sor_grid* g, R w) {
  const Slab& s = g->slabs[0];
  ResArgs<R> a{};
  a.pitch = g->pitch;
  a.g0 = s.g0;
  a.rows = (int)g->rows;
  a.cols = (int)g->cols;
  a.w = w;
  a.ctl.st = g->dstate;
  return a;
}

}  // namespace

bool resident_fits(const sor_grid* g, int T, bool single) {
  ResPlan p;
  return res_plan(g, T, single, &p);
}

template <typename R>
int launch_resident_iterate(sor_grid* g, R w, int64_t iters, int T, bool check_last) {
  static const int force_t = std::min(kMaxT, std::max(0, env_int("SOR_RESIDENT_T")));  // A/B only
  if (force_t) T = force_t;
  ResPlan p;
  if (!single_part(g) || iters < 1 || !res_plan(g, T, false, &p)) return SOR_E_UNSUPPORTED;
  if (iters > (int64_t)T * (1 << 30)) return SOR_E_UNSUPPORTED;
  const int npasses = (int)((iters + T - 1) / T);
  if (!g->rflags) {
    CU(cudaMalloc(&g->rflags, (size_t)16 * 8 * 2 * g->nsm));
    CU(cudaMemsetAsync(g->rflags, 0, (size_t)16 * 8 * 2 * g->nsm, g->stream));
    g->rseq = 0;
  }
  const Slab& s = g->slabs[0];
  ResArgs<R> a = res_args<R>(g, w);
  const int p0 = g->cur, p1 = g->nxt(g->cur);
  a.pa = col0<R>(s.plane[p0]);
  a.pb = col0<R>(s.plane[p1]);
  a.nbx = p.nbx;
  a.nby = p.nby;
  a.T = T;
  a.G = 2 * T;
  a.npasses = npasses;
  a.t_last = (int)(iters - (int64_t)(npasses - 1) * T);
  a.flags = g->rflags;
  a.seq0 = g->rseq;
  a.check_last = check_last ? 1 : 0;
  if (check_last) {
    a.ctl.k_last = iters;
    a.ctl.maxit = iters;
    a.ctl.K = 1;
    a.ctl.T = 1;
    a.ctl.ck = 1;
    a.ctl.finalize = 1;
    a.ctl.nparts = (unsigned)(p.nbx * p.nby);
  }
  // development aid: per-pass phase timestamps appended to SOR_RES_TRACE
  static const char* trace_path = getenv("SOR_RES_TRACE");
  static unsigned long long* dtrace = nullptr;
  const size_t ntr = (size_t)2 * g->nsm * 64 * 8;
  if (trace_path) {
    if (!dtrace) CU(cudaMalloc(&dtrace, ntr * 8));
    CU(cudaMemsetAsync(dtrace, 0, ntr * 8, g->stream));
    a.trace = dtrace;
  }
  TRY(res_dispatch<R>(g, p, a, true));
  if (trace_path) {
    std::vector<unsigned long long> h(ntr);
    CU(cudaMemcpyAsync(h.data(), dtrace, ntr * 8, cudaMemcpyDeviceToHost, g->stream));
    CU(cudaStreamSynchronize(g->stream));
    FILE* f = fopen(trace_path, "ab");
    if (f) {
      const int hdr[4] = {p.nbx, p.nby, npasses, T};
      fwrite(hdr, sizeof(hdr), 1, f);
      fwrite(h.data(), 8, ntr, f);
      fclose(f);
    }
  }
  g->rseq += (uint64_t)npasses;
  if (npasses & 1) g->cur = p1;
  g->st.half_sweeps += 2 * iters;
  g->st.hbm_passes += npasses;
  if (check_last) g->st.checks += 1;
  g->seq += (unsigned long long)npasses;
  return SOR_OK;
}

template <typename R>
int launch_resident_single(sor_grid* g, R w, int solve, int64_t n_iter, double tol, int64_t K, int check_last) {
  ResPlan p;
  if (!single_part(g) || !res_plan(g, 1, true, &p)) return SOR_E_UNSUPPORTED;
  const Slab& s = g->slabs[0];
  ResArgs<R> a = res_args<R>(g, w);
  a.pa = a.pb = col0<R>(s.plane[g->cur]);  // in place
  a.nbx = a.nby = 1;
  a.T = 1;
  a.G = 1;
  a.npasses = 1;
  a.t_last = 1;
  a.solve = solve;
  a.n_iter = n_iter;
  a.K = K;
  a.tol = tol;
  a.check_last = check_last;
  return res_dispatch<R>(g, p, a, false);
}

template int launch_resident_iterate<double>(sor_grid*, double, int64_t, int, bool);
template int launch_resident_iterate<float>(sor_grid*, float, int64_t, int, bool);
template int launch_resident_single<double>(sor_grid*, double, int, int64_t, double, int64_t, int);
template int launch_resident_single<float>(sor_grid*, float, int, int64_t, double, int64_t, int);

}  // namespace sorh
