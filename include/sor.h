/*
 * sor.h — C ABI of the B200-native red-black SOR hot path (libsor.so).
 *
 * Method: S. Mittal, "A Study of Successive Over-relaxation Method
 * Parallelization Over Modern HPC Languages", arXiv 1401.0763.
 * Citation key: P:n = /root/reference/PAPER.md line n (section in brackets);
 * "reading #k" = DESIGN.md §3 (the interpretation adopted where the paper is
 * silent or garbled, shared with the oracle but not its code).
 *
 * What one iteration computes (every entry point below runs exactly this):
 *   red phase   [§3.1; Alg. 1 P:313]: for every interior cell
 *               with (i+j) even, Eq. 1 [§2.1, P:97-100] in the canonical form
 *               s = (uN+uS)+(uW+uE); a = 0.25*s; r = a - u; u' = u + w*r
 *               (readings #2-#4; no FMA contraction, no reassociation);
 *   black phase [P:198, P:316]: the same for (i+j) odd, reading the new reds;
 *   max-change  [P:103, Alg. 1 P:319-325]: max over interior cells of
 *               |u' - u| (reading #5), on checked iterations only.
 * Indices are on the global padded grid: row 0 is the north ring,
 * cell (1,1) is red (reading #11).  The ring is Dirichlet data, never written.
 *
 * Conventions shared by every call:
 *   - Grid arrays are row-major (rows+2) x (cols+2) fp64 INCLUDING the ring
 *     (reading #1: rows, cols count interior cells).  Pointers may be host
 *     memory (pageable or pinned) or device memory of the handle's GPU (e.g.
 *     a torch tensor's data_ptr); the library detects which.  Caller buffers
 *     are borrowed only for the duration of the call; the caller keeps
 *     ownership.
 *   - Return value: SOR_OK (0) on success, SOR_NOT_CONVERGED (1) when a solve
 *     reached maxit (outputs and grid still valid), negative sor_status on
 *     error.  On a negative status, sor_last_error() returns a thread-local
 *     message.  Invalid arguments (SOR_E_INVAL) leave the handle unchanged.
 *     A CUDA or NCCL failure (SOR_E_CUDA / SOR_E_NCCL) makes the handle
 *     sticky-failed: later calls return SOR_E_STATE until sor_destroy.
 *   - Calls are synchronous: they return after the device work completed.
 *     A handle is not thread-safe; distinct handles are independent.
 *   - There is no CPU fallback: without a usable sm_100 GPU, sor_create*
 *     returns SOR_E_CUDA.
 */
#ifndef SOR_H
#define SOR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sor_grid sor_grid; /* opaque; owns all device memory, stream, events, comm */

typedef enum { SOR_F64 = 0, SOR_F32 = 1 } sor_dtype;

typedef enum {
  SOR_OK = 0,
  SOR_NOT_CONVERGED = 1,
  SOR_E_INVAL = -1,
  SOR_E_NOMEM = -2,
  SOR_E_CUDA = -3,
  SOR_E_NCCL = -4,
  SOR_E_STATE = -5,
  SOR_E_UNSUPPORTED = -6
} sor_status;

/* Kernel variants (selected explicitly; there is no auto-dispatch).  All give
 * bitwise-identical results.                                  */
#define SOR_MAX_T 6  /* deepest temporal blocking (iterations per HBM pass); > 4: one slab, SOR only */

typedef enum {
  SOR_KERNEL_NATURAL = 1,  /* K1: one launch per colour phase, in place, natural layout */
  SOR_KERNEL_FUSED = 3,    /* K3: red+black fused in one HBM pass, src->dst ping-pong  */
  SOR_KERNEL_TEMPORAL = 4, /* K4: T iterations per HBM pass (temporal blocking)         */
  SOR_KERNEL_SMALL = 5,    /* K5: whole grid in one CTA (registers if <= 126 columns,   */
                           /*     else shared memory), one launch                        */
  SOR_KERNEL_RESIDENT = 6  /* K7: grid register-resident across the SMs, one CTA per SM  */
} sor_kernel;

/* Create a single-GPU handle on the current CUDA device.
 *   N / rows, cols : interior size, >= 1 each (reading #1).
 *   init           : (rows+2)*(cols+2) fp64, row-major, host or device; ring =
 *                    Dirichlet data, interior = initial guess; all finite.
 *   dt             : storage AND arithmetic type.  SOR_F32 rounds init to
 *                    nearest once; w and 0.25 are rounded once (reading #17).
 * Default kernel: SOR_KERNEL_FUSED.  Returns SOR_E_INVAL (NULL out/init,
 * rows/cols < 1, non-finite init), SOR_E_NOMEM, SOR_E_CUDA.                 */
int sor_create(sor_grid** out, int64_t N, const double* init, sor_dtype dt);
int sor_create_rect(sor_grid** out, int64_t rows, int64_t cols, const double* init,
                    sor_dtype dt);

/* Multi-GPU, one process per GPU (row slabs, §8(e)): rank r of nranks owns a
 * contiguous block of interior rows (sizes differ by <= 1) — the
 * P workers of Algorithm 1 each updating their own cells [P:313-317, P:378].
 * Two transports, the same kernels and bitwise the same results:
 *
 * sor_create_dist_ipc (the product path, one node): ranks map each other's
 *   planes over CUDA IPC; a wave pass's edge tiles store their first/last
 *   rows straight into the neighbours' halo rows (NVLink peer stores) and
 *   release a per-strip flag; the edge tiles of the neighbours' next pass
 *   acquire it, interior tiles never wait, so no global barrier or copy
 *   separates passes [the paper's per-phase barrier, P:203, P:314-317,
 *   P:394, becomes neighbour-only flags].  Checked passes join the per-rank
 *   max-changes through the same mappings (publish / acquire), decided
 *   speculatively by the next pass's block 0 as on one GPU.  `ipc_id` is the
 *   128-byte id from sor_ipc_unique_id() on rank 0, broadcast by the caller;
 *   the ranks meet in a POSIX shared-memory segment of that name (also their
 *   host barrier for create / reset / download / the start of every call).
 *   Ranks that share one GPU (a test configuration) run in lockstep: a host
 *   barrier after every pass, because kernels of different processes on one
 *   device are time-sliced and must never wait on each other.
 * sor_create_dist (fallback): halo rows by NCCL send/recv after every pass
 *   and the max-change by an NCCL allreduce-max; `nccl_id` = the 128-byte
 *   ncclUniqueId from sor_nccl_unique_id() on rank 0.
 *
 * `device` is the CUDA ordinal for this rank.  `init` is read on rank 0
 * only (the full (rows+2)*(cols+2) array, host or device); other ranks may
 * pass NULL — rank 0 scatters the slabs (a non-finite init fails every
 * rank).  Requires rows >= 8*nranks and at most 8 ranks for IPC.  All later
 * calls on a dist handle are collective: every rank calls them with
 * identical arguments (a mismatch times out, making the handle failed).     */
int sor_create_dist(sor_grid** out, int64_t rows, int64_t cols, const double* init,
                    sor_dtype dt, int rank, int nranks, int device, const void* nccl_id);
int sor_nccl_unique_id(void* out128);
int sor_create_dist_ipc(sor_grid** out, int64_t rows, int64_t cols, const double* init,
                        sor_dtype dt, int rank, int nranks, int device, const void* ipc_id);
int sor_ipc_unique_id(void* out128);

/* Virtual slabs on ONE GPU (test/diagnostic mode): the same slab
 * decomposition, halo layout and kernels as the dist handles with `nslabs`
 * slabs in one process; halo rows move by the same device-initiated pushes
 * and flags as sor_create_dist_ipc (SOR_VIRTUAL_COPY=1 in the environment:
 * by device-to-device copies after every pass instead).                    */
int sor_create_virtual(sor_grid** out, int64_t rows, int64_t cols, const double* init,
                       sor_dtype dt, int nslabs);

/* Select the kernel variant.  temporal_depth T (iterations per HBM pass) is
 * used by SOR_KERNEL_TEMPORAL and SOR_KERNEL_RESIDENT, 1 <= T <= SOR_MAX_T
 * (T = 1 equals FUSED; multi-slab grids need slabs of >= 2T rows; T = 5, 6
 * only on single-slab handles (SOR_E_UNSUPPORTED otherwise), and Jacobi calls
 * on a handle set deeper than 4 return SOR_E_UNSUPPORTED).
 * SOR_KERNEL_SMALL requires a single-slab grid that fits in shared memory;
 * SOR_KERNEL_NATURAL is not available on dist-IPC handles (SOR_E_UNSUPPORTED).
 * SOR_KERNEL_RESIDENT (K7, for small grids; the paper's per-phase barrier
 * [P:203, P:314, P:317] becomes a CTA barrier and neighbour-only flags):
 * sor_iterate on a single-slab grid that fits one 2-D block per SM (window of
 * block + 2T ring <= 128 columns x ~80-90 rows: up to ~1.2 M cells) runs all
 * its passes of T iterations in one cooperative launch, blocks exchanging only
 * the 2T-deep frames with their 8 neighbours between passes; a grid of at most
 * 126 columns and ~94 rows runs (iterate and solve) on one CTA with the stop
 * test on the device.  Anything else runs as SOR_KERNEL_TEMPORAL with depth T.
 * Jacobi calls run as SOR_KERNEL_TEMPORAL.
 * Returns SOR_E_INVAL / SOR_E_UNSUPPORTED without changing the handle.      */
int sor_set_kernel(sor_grid* g, int kernel, int temporal_depth);

/* Run exactly `iters` >= 0 iterations with relaxation factor 0 < omega < 2
 * (P:100).  If last_max_change != NULL it receives max|u'-u| of the last
 * iteration (0 if iters == 0).  The grid persists across calls.             */
int sor_iterate(sor_grid* g, double omega, int64_t iters, double* last_max_change);

/* Algorithm 1: for k = 1..maxit, one iteration; if k % check_every
 * == 0 the max-change of iteration k is computed and the call stops as soon
 * as it is < tol (strict).  Requires 0 < omega < 2, tol > 0 finite,
 * maxit >= 1, 1 <= check_every <= maxit.  Outputs (nullable):
 *   iters_out      : iterations executed in THIS call (the converging one
 *                    included; maxit if not converged);
 *   max_change_out : the last checked max-change (fp64).
 * Returns SOR_OK if converged, SOR_NOT_CONVERGED if maxit was reached.      */
int sor_solve(sor_grid* g, double omega, double tol, int64_t maxit, int64_t check_every,
              int64_t* iters_out, double* max_change_out);

/* Jacobi (NEXT-2) on the same handle and layout: iteration
 * k sets every interior cell of X_k to 0.25*((N+S)+(W+E)) of X_{k-1} (the
 * operation order of reading #3; no relaxation factor).  Same contracts,
 * outputs and errors as sor_iterate / sor_solve (without omega); the max-
 * change is |X_k - X_{k-1}| per cell.  Runs on SOR_KERNEL_FUSED (T = 1) and
 * SOR_KERNEL_TEMPORAL (T Jacobi iterations per HBM pass); other kernels
 * return SOR_E_UNSUPPORTED.  SOR and Jacobi calls may be mixed on a handle. */
int sor_jacobi_iterate(sor_grid* g, int64_t iters, double* last_max_change);
int sor_jacobi_solve(sor_grid* g, double tol, int64_t maxit, int64_t check_every, int64_t* iters_out,
                     double* max_change_out);

/* NEXT-4: the parallel SOR variants the paper names beside red-black SOR
 * [§3.1, P:147] ("multi-color SOR", "block-parallel SOR"; no algorithm is
 * given there: DESIGN.md §3 readings N4-1 / N4-2 define them), on the same
 * handle and layout.  Every update is Eq. 1 [P:97-100] in the canonical
 * order, in place, reading the latest values.
 *   SOR_VARIANT_MULTICOLOR: colour(i, j) = (ca*i + cb*j) mod nc (storage
 *     indices, non-negative residue); one iteration = colour phases 0, 1,
 *     ..., nc-1.  Needs 2 <= nc <= 8 (else SOR_E_UNSUPPORTED) and ca, cb not
 *     multiples of nc (else SOR_E_INVAL: 5-point neighbours would share a
 *     colour).  (1, 1, 2) is red-black SOR.
 *   SOR_VARIANT_BLOCK: block x block blocks anchored at cell (1, 1), red iff
 *     bi+bj even; the red blocks, then the black blocks, natural (row-major)
 *     order inside a block.  Needs 1 <= block <= 32 (else
 *     SOR_E_UNSUPPORTED).  block = 1 is red-black SOR.
 * Single-GPU handles only (virtual / dist: SOR_E_UNSUPPORTED); the handle's
 * sor_kernel setting is not used.  Contracts, outputs and errors otherwise as
 * sor_iterate / sor_solve; `v` is read during the call only.  Stats:
 * half_sweeps counts colour phases (nc or 2 per iteration).                */
typedef enum { SOR_VARIANT_MULTICOLOR = 1, SOR_VARIANT_BLOCK = 2 } sor_variant_kind;
typedef struct {
  int32_t kind;       /* sor_variant_kind                    */
  int32_t ca, cb, nc; /* multi-colour: colour (ca*i+cb*j) mod nc */
  int32_t block;      /* block: block side B                 */
} sor_variant;
int sor_variant_iterate(sor_grid* g, const sor_variant* v, double omega, int64_t iters, double* last_max_change);
int sor_variant_solve(sor_grid* g, const sor_variant* v, double omega, double tol, int64_t maxit,
                      int64_t check_every, int64_t* iters_out, double* max_change_out);

/* 3-D red-black SOR (NEXT-3; the paper's future work): a separate
 * single-GPU handle over an nz x ny x nx interior with a Dirichlet shell.
 * `init` = caller-owned (nz+2)*(ny+2)*(nx+2) fp64 array, row-major with z
 * slowest (shell = boundary data, interior = initial guess), host or device,
 * copied during the call; 1 <= nz, ny <= 65535.  Colour of (z, y, x): red iff
 * z+y+x even, red phase first; per cell s = ((N+S)+(W+E))+(U+D), a = s/6
 * (correctly rounded), u' = u + omega*(a - u) (reading N3-1).
 * iterate / solve / download / errors as the 2-D calls, exact maxima.
 * Kernels (sor3d_set_kernel): SOR_KERNEL_NATURAL (two in-place colour
 * phases) or SOR_KERNEL_FUSED (the default: one HBM pass per iteration, a
 * z-plane wavefront over TMA-staged planes, src -> dst, two planes per CTA
 * barrier); bitwise equal.  The handle lives on the CUDA device current at
 * sor3d_create; later calls run there whatever device is current and
 * restore the caller's device on return (as the 2-D handles do).           */
typedef struct sor3d_grid sor3d_grid;
int sor3d_create(sor3d_grid** out, int64_t nz, int64_t ny, int64_t nx, const double* init, sor_dtype dt);
int sor3d_iterate(sor3d_grid* g, double omega, int64_t iters, double* last_max_change);
int sor3d_solve(sor3d_grid* g, double omega, double tol, int64_t maxit, int64_t check_every, int64_t* iters_out,
                double* max_change_out);
int sor3d_download(sor3d_grid* g, double* out);
int sor3d_set_kernel(sor3d_grid* g, int kernel);
int sor3d_last_elapsed_ms(const sor3d_grid* g, double* ms);
void sor3d_destroy(sor3d_grid* g);

/* Copy the current iterate into `out` ((rows+2)*(cols+2) fp64, host or
 * device; fp32 grids are widened exactly).  Dist: collective; rank 0
 * receives the whole grid, other ranks' `out` may be NULL (ignored).       */
int sor_download(sor_grid* g, double* out);

/* Copy global rows [row_a, row_b) (0 <= row_a < row_b <= rows+2, ring rows
 * included) of the current iterate into `out` ((row_b-row_a)*(cols+2) fp64,
 * host or device).  Dist: collective like sor_download (rank 0 receives).   */
int sor_download_rows(sor_grid* g, int64_t row_a, int64_t row_b, double* out);

/* Re-load the grid from `init` (same contract as sor_create), keeping the
 * handle's allocation, kernel choice and stream.  Dist: collective, `init`
 * read on rank 0 only (NULL allowed elsewhere).                             */
int sor_reset(sor_grid* g, const double* init);

/* Use an external CUDA stream (cudaStream_t, e.g. torch's current stream) for
 * all work of this handle; NULL restores the handle's own stream.           */
int sor_set_stream(sor_grid* g, void* cuda_stream);

/* CUDA-event time (ms) of the device work of the last iterate/solve call.   */
int sor_last_elapsed_ms(const sor_grid* g, double* ms);

typedef struct {
  int64_t kernel_launches;  /* library kernels launched by the last iterate/solve call */
  int64_t half_sweeps;      /* colour phases executed (2 per iteration); Jacobi: sweeps */
  int64_t halo_exchanges;   /* halo exchange rounds (dist / virtual)                  */
  int64_t checks;           /* convergence checks evaluated                           */
  int64_t hbm_passes;       /* full read+write passes over the grid                    */
  int32_t kernel;           /* active sor_kernel                                       */
  int32_t temporal_depth;
  int32_t nslabs;           /* slabs held by this handle (virtual) or 1               */
  int32_t rank, nranks;
  int64_t row_lo, row_hi;   /* owned global interior rows [row_lo, row_hi) of slab 0  */
  int64_t pitch_elems;      /* device row pitch in elements                           */
  int64_t exact_reruns;     /* solve: passes re-run to decide the stop test exactly    */
} sor_stats;
int sor_get_stats(const sor_grid* g, sor_stats* out);

/* Host logic shared by the dist and virtual modes (also usable without a
 * GPU): rank p of P owns interior rows [*lo, *hi), 1-based, contiguous,
 * sizes differ by at most 1.  Returns SOR_E_INVAL if P < 1,
 * p outside [0,P) or rows < P.                                              */
int sor_partition_rows(int64_t rows, int P, int p, int64_t* lo, int64_t* hi);

/* Release everything owned by the handle.  NULL-safe.                       */
void sor_destroy(sor_grid* g);

/* Thread-local text for the last non-OK status on this thread.             */
const char* sor_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SOR_H */
