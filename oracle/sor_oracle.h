/*
 * sor_oracle.h — CPU oracle for red-black SOR (arXiv 1401.0763).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1401_0763_b200/) never links, imports or calls it,
 * and shares no code, header, table or constant generator with it.
 *
 * Citation key: P:n = PAPER.md line n; S:n = SPEC.md line n; "reading #k" =
 * DESIGN.md §3 / SURVEY.md §8(c) interpretation k.
 *
 * Grid convention (reading #1): `rows` x `cols` INTERIOR cells; storage is the
 * full (rows+2) x (cols+2) row-major array including the Dirichlet ring
 * (row 0 = north).  The ring is never written.
 * Colour (reading #11): cell (i,j) is red iff (row_off + i + j) is even,
 * where row_off is the global index of the array's row 0 (0 for a full grid;
 * used only to run a slab of a larger grid with its halo rows as the ring).
 *
 * Parity status: every function below is pinned by
 * tests/test_oracle_pins.py EXCEPT where its comment says "parity unpinned".
 */
#ifndef SOR_ORACLE_H
#define SOR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_DONE = 0, ORC_NOT_CONVERGED = 1, ORC_E_INVAL = -1 };

typedef struct {
  int32_t status;       /* ORC_DONE (iterate done / solve converged), ORC_NOT_CONVERGED */
  int64_t iters;        /* iterations executed (1-based index of converging one, else maxit) */
  double max_change;    /* last CHECKED max |X_k - X_{k-1}|; widened to f64 */
  int64_t half_sweeps;  /* barrier counter: 2 per iteration */
  int64_t checks;       /* number of convergence checks performed */
} orc_report;

/* Eq. 1 for one cell in the canonical operation order (reading #2-#4):
 *   s = (N+S)+(W+E); a = 0.25*s; r = a-u; u' = u + w*r.                        */
double orc_cell_update_f64(double n, double s, double w_, double e, double u, double omega);
float  orc_cell_update_f32(float n, float s, float w_, float e, float u, double omega);

/* Algorithm 1, single thread, fused |delta| (reading #5):
 * mode 0 = iterate exactly `n_iter` iterations; if `measure_last` the last
 *          iteration's max|delta| is returned in rep->max_change.
 * mode 1 = solve: check every K iterations, converged iff max < tol
 *          (strict), stop at n_iter (= MaxIterations).         */
int orc_sor_run_f64(double* u, int64_t rows, int64_t cols, int64_t row_off, double omega,
                    int mode, int64_t n_iter, double tol, int64_t K, int measure_last,
                    orc_report* rep);
int orc_sor_run_f32(float* u, int64_t rows, int64_t cols, int64_t row_off, double omega,
                    int mode, int64_t n_iter, double tol, int64_t K, int measure_last,
                    orc_report* rep);

/* One colour phase (half-sweep) of updateGridRed/updateGridBlack,
 * colour c = 0 red, 1 black.  If m != NULL, max|delta| of the phase is folded
 * into *m.  Exposed so tests can run individual phases.          */
void orc_half_sweep_f64(double* u, int64_t rows, int64_t cols, int64_t row_off, int c,
                        double omega, double* m);

/* Algorithm 1 literally: snapshot copy of gridData at iter % K == 0,
 * both phases, then serial max over all cells of |gridData - gridDataOld|
 * (P:319-325).  Solve mode only.  Pin P13: equals orc_sor_run_f64 bitwise.   */
int orc_sor_run_snapshot_f64(double* u, int64_t rows, int64_t cols, double omega,
                             int64_t maxit, double tol, int64_t K, orc_report* rep);

/* P workers on contiguous row blocks with a barrier after each
 * colour phase and the serial max combine.
 * Pin P14: bitwise equal to orc_sor_run_f64 for any P.                      */
int orc_sor_run_threads_f64(double* u, int64_t rows, int64_t cols, double omega, int mode,
                            int64_t n_iter, double tol, int64_t K, int measure_last,
                            int nthreads, orc_report* rep);
int orc_sor_run_threads_f32(float* u, int64_t rows, int64_t cols, double omega, int mode,
                            int64_t n_iter, double tol, int64_t K, int measure_last,
                            int nthreads, orc_report* rep);

/* Contiguous near-equal row partition: worker p of P gets rows
 * [lo, hi) of 1..rows (1-based, interior); sizes differ by at most 1.       */
void orc_partition_rows(int64_t rows, int P, int p, int64_t* lo, int64_t* hi);

/* Jacobi: X_k computed from X_{k-1} only, X = (N+S+W+E)/4
 * in the same operation order; check every iteration, stop when max < tol. */
int orc_jacobi_f64(double* u, int64_t rows, int64_t cols, int64_t maxit, double tol,
                   orc_report* rep);

/* Jacobi in the same two modes as orc_sor_run (NEXT-2): iteration k computes
 * every interior cell of X_k from X_{k-1} only, X = 0.25*((N+S)+(W+E)) in the
 * order of reading #3, |delta| = |X_k - X_{k-1}| by
 * subtraction (reading #5); mode 1 checks every K iterations and
 * stops when the checked max < tol (strict).  f32: storage and
 * arithmetic in float, 0.25 exact.  half_sweeps counts 1 per iteration.     */
int orc_jacobi_run_f64(double* u, int64_t rows, int64_t cols, int mode, int64_t n_iter, double tol,
                       int64_t K, int measure_last, orc_report* rep);
int orc_jacobi_run_f32(float* u, int64_t rows, int64_t cols, int mode, int64_t n_iter, double tol,
                       int64_t K, int measure_last, orc_report* rep);

/* 3-D red-black SOR (NEXT-3; the paper's future work): an nz x ny x nx
 * interior with a Dirichlet shell, storage (nz+2)*(ny+2)*(nx+2) row-major
 * (z slowest).  Colour of (z, y, x): red iff z+y+x even (reading #11 in 3-D);
 * red phase first.  Per cell (reading N3-1): s = ((N+S)+(W+E))+(U+D) with
 * N/S = y-1/y+1, W/E = x-1/x+1, U/D = z-1/z+1; a = s / 6 (correctly rounded
 * division: the average of the six neighbours); r = a - u; u' = u + w*r.
 * Modes, cadence and |delta| as orc_sor_run.                                */
int orc_sor3d_run_f64(double* u, int64_t nz, int64_t ny, int64_t nx, double omega, int mode,
                      int64_t n_iter, double tol, int64_t K, int measure_last, orc_report* rep);
int orc_sor3d_run_f32(float* u, int64_t nz, int64_t ny, int64_t nx, double omega, int mode,
                      int64_t n_iter, double tol, int64_t K, int measure_last, orc_report* rep);

/* NEXT-4 (readings N4-1, N4-2): multi-colour SOR (kind 0: colour
 * (p1*i + p2*j) mod p3, phases 0..p3-1; p1, p2 not multiples of p3) and
 * block red-black SOR (kind 1: p1 x p1 blocks, chessboard of blocks, red
 * first, natural order inside a block).  Modes, cadence, |delta| and the
 * stop test as orc_sor_run; half_sweeps counts colour phases (p3 or 2 per
 * iteration).  f32: float storage and arithmetic.                          */
int orc_variant_run_f64(double* u, int64_t rows, int64_t cols, int kind, int64_t p1, int64_t p2,
                        int64_t p3, double omega, int mode, int64_t n_iter, double tol, int64_t K,
                        int measure_last, orc_report* rep);
int orc_variant_run_f32(float* u, int64_t rows, int64_t cols, int kind, int64_t p1, int64_t p2,
                        int64_t p3, double omega, int mode, int64_t n_iter, double tol, int64_t K,
                        int measure_last, orc_report* rep);

/* Brute force for the 3-D pin (test only): the 7-point Dirichlet system by
 * dense Gaussian elimination; nz*ny*nx <= 1728.                             */
int orc_dense_solve3d_f64(double* u, int64_t nz, int64_t ny, int64_t nx);

/* Brute force (test only): solve the 5-point Dirichlet system
 * 4u_ij - sum(interior neighbours) = sum(ring neighbours) by dense Gaussian
 * elimination with partial pivoting; writes the interior of `u` in place.
 * Returns 0, or -1 if rows*cols > 4096.                                      */
int orc_dense_solve_f64(double* u, int64_t rows, int64_t cols);

#ifdef __cplusplus
}
#endif
#endif
