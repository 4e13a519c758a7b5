/*
 * sor_oracle.c — plain, slow, obviously-correct CPU oracle for red-black SOR
 * (S. Mittal, arXiv 1401.0763).  TEST INFRASTRUCTURE ONLY (see sor_oracle.h):
 * never linked into the product library, shares no code with it.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared (no -ffast-math:
 * FTZ/DAZ must stay off so fp32 subnormals are kept, reading #17).
 *
 * The code follows the paper in its own order:
 *   Eq. 1           X_k = w*Xbar_k + (1-w)*X_{k-1}, written in the
 *                              BJ form u + w*(a - u) (reading #2) with
 *                              Xbar = 0.25*((N+S)+(W+E)) (readings #3, #4);
 *   colouring          red iff (i+j) even (reading #11);
 *   phase order        red phase, then black phase using the new reds;
 *   loop form (Fig. 2)  stride-2 loops, no per-cell parity test (A5);
 *   Algorithm 1    iteration loop, check every K,
 *                              maxChange = max |X_k - X_{k-1}|,
 *                              converged iff maxChange < eps.
 */
#define _POSIX_C_SOURCE 200809L
#include "sor_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* One cell, Eq. 1 in the canonical order.  T-typed temporaries round every
 * intermediate to T (x86-64 SSE: FLT_EVAL_METHOD == 0; contraction off).    */
#define DEFINE_CELL(T, SUF)                                                   \
  T orc_cell_update_##SUF##_impl(T n, T s_, T w_, T e, T u, T w) {            \
    const T q = (T)0.25;                                                      \
    T s = (n + s_) + (w_ + e);                                                \
    T a = q * s;                                                              \
    T r = a - u;                                                              \
    return u + w * r;                                                         \
  }
DEFINE_CELL(double, f64)
DEFINE_CELL(float, f32)

double orc_cell_update_f64(double n, double s, double w_, double e, double u, double omega) {
  return orc_cell_update_f64_impl(n, s, w_, e, u, omega);
}
float orc_cell_update_f32(float n, float s, float w_, float e, float u, double omega) {
  return orc_cell_update_f32_impl(n, s, w_, e, u, (float)omega);
}

/* ------------------------------------------------------------------------ */
/* One colour phase over interior rows [i_lo, i_hi) (1-based, inclusive of
 * nothing outside 1..rows).  Code 2 form: for each row the first
 * column of colour c, then stride 2.  Delta = |u' - u| by subtraction
 * (reading #5); max keeps NaN (reading #25).                                 */
#define DEFINE_PHASE(T, SUF, ABS)                                             \
  static void phase_##SUF(T* u, int64_t cols, int64_t row_off, int64_t i_lo,  \
                          int64_t i_hi, int c, T w, int check, T* m) {        \
    const int64_t ld = cols + 2;                                              \
    const T q = (T)0.25;                                                      \
    for (int64_t i = i_lo; i < i_hi; ++i) {                                   \
      const int64_t j0 = (((row_off + i + 1) & 1) == c) ? 1 : 2;             \
      T* up = u + (i - 1) * ld;                                               \
      T* uc = u + i * ld;                                                     \
      T* dn = u + (i + 1) * ld;                                               \
      for (int64_t j = j0; j <= cols; j += 2) {                               \
        T s = (up[j] + dn[j]) + (uc[j - 1] + uc[j + 1]);                      \
        T a = q * s;                                                          \
        T r = a - uc[j];                                                      \
        T un = uc[j] + w * r;                                                 \
        if (check) {                                                          \
          T d = ABS(un - uc[j]);                                              \
          if (d > *m || d != d) *m = d;                                       \
        }                                                                     \
        uc[j] = un;                                                           \
      }                                                                       \
    }                                                                         \
  }
DEFINE_PHASE(double, f64, fabs)
DEFINE_PHASE(float, f32, fabsf)

void orc_half_sweep_f64(double* u, int64_t rows, int64_t cols, int64_t row_off, int c,
                        double omega, double* m) {
  double mm = m ? *m : 0.0;
  phase_f64(u, cols, row_off, 1, rows + 1, c, omega, m != NULL, &mm);
  if (m) *m = mm;
}

static int check_args(int64_t rows, int64_t cols, double omega, int mode, int64_t n_iter,
                      double tol, int64_t K) {
  if (rows < 1 || cols < 1) return 0;
  if (!(omega > 0.0 && omega < 2.0)) return 0;
  if (mode == 1) {
    if (!(tol > 0.0) || !isfinite(tol) || n_iter < 1 || K < 1 || K > n_iter) return 0;
  } else if (mode == 0) {
    if (n_iter < 0) return 0;
  } else {
    return 0;
  }
  return 1;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 1 main routine, single thread.                      */
#define DEFINE_RUN(T, SUF)                                                    \
  int orc_sor_run_##SUF(T* u, int64_t rows, int64_t cols, int64_t row_off,    \
                        double omega, int mode, int64_t n_iter, double tol,   \
                        int64_t K, int measure_last, orc_report* rep) {       \
    memset(rep, 0, sizeof(*rep));                                             \
    if (!check_args(rows, cols, omega, mode, n_iter, tol, K)) {               \
      rep->status = ORC_E_INVAL;                                              \
      return ORC_E_INVAL;                                                     \
    }                                                                         \
    const T w = (T)omega;                                                     \
    rep->status = mode == 1 ? ORC_NOT_CONVERGED : ORC_DONE;                   \
    for (int64_t k = 1; k <= n_iter; ++k) {                /* P:301 */        \
      int check = mode == 1 ? (k % K == 0)                 /* P:304 */        \
                            : (measure_last && k == n_iter);                  \
      T m = (T)0;                                                             \
      phase_##SUF(u, cols, row_off, 1, rows + 1, 0, w, check, &m); /* red */  \
      phase_##SUF(u, cols, row_off, 1, rows + 1, 1, w, check, &m); /* black*/ \
      rep->half_sweeps += 2;                                                  \
      rep->iters = k;                                                         \
      if (check) {                                                            \
        rep->checks += 1;                                                     \
        rep->max_change = (double)m;                                          \
        if (mode == 1 && (double)m < tol) {                /* P:327 */        \
          rep->status = ORC_DONE;                                             \
          break;                                                              \
        }                                                                     \
      }                                                                       \
    }                                                                         \
    return rep->status;                                                       \
  }
DEFINE_RUN(double, f64)
DEFINE_RUN(float, f32)

/* ------------------------------------------------------------------------ */
/* Algorithm 1 with its literal snapshot copy. */
int orc_sor_run_snapshot_f64(double* u, int64_t rows, int64_t cols, double omega,
                             int64_t maxit, double tol, int64_t K, orc_report* rep) {
  memset(rep, 0, sizeof(*rep));
  if (!check_args(rows, cols, omega, 1, maxit, tol, K)) {
    rep->status = ORC_E_INVAL;
    return ORC_E_INVAL;
  }
  const int64_t n = (rows + 2) * (cols + 2);
  double* old = (double*)malloc((size_t)n * sizeof(double));
  if (!old) {
    rep->status = ORC_E_INVAL;
    return ORC_E_INVAL;
  }
  rep->status = ORC_NOT_CONVERGED;
  for (int64_t iter = 1; iter <= maxit; ++iter) {
    int should_check = (iter % K == 0);
    if (should_check) memcpy(old, u, (size_t)n * sizeof(double));
    double unused = 0.0;
    phase_f64(u, cols, 0, 1, rows + 1, 0, omega, 0, &unused);
    phase_f64(u, cols, 0, 1, rows + 1, 1, omega, 0, &unused);
    rep->half_sweeps += 2;
    rep->iters = iter;
    if (should_check) {
      double maxChange = 0.0;
      for (int64_t c = 0; c < n; ++c) {
        double d = fabs(u[c] - old[c]);
        if (d > maxChange || d != d) maxChange = d;
      }
      rep->checks += 1;
      rep->max_change = maxChange;
      if (maxChange < tol) {
        rep->status = ORC_DONE;
        break;
      }
    }
  }
  free(old);
  return rep->status;
}

/* ------------------------------------------------------------------------ */
/* P workers with a barrier after each phase.                    */
void orc_partition_rows(int64_t rows, int P, int p, int64_t* lo, int64_t* hi) {
  const int64_t base = rows / P, rem = rows % P;
  const int64_t start = 1 + p * base + (p < rem ? p : rem);
  *lo = start;
  *hi = start + base + (p < rem ? 1 : 0);
}

typedef struct {
  void* u;
  int64_t rows, cols;
  double omega;
  int mode;
  int64_t n_iter;
  double tol;
  int64_t K;
  int measure_last;
  int P;
  int is_f32;
  pthread_barrier_t bar;
  double* partial_max; /* one per worker, combined serially */
  volatile int stop;
  orc_report* rep;
} tjob;

typedef struct {
  tjob* job;
  int p;
} targ;

static void* worker(void* vp) {
  targ* ta = (targ*)vp;
  tjob* jb = ta->job;
  int64_t lo, hi;
  orc_partition_rows(jb->rows, jb->P, ta->p, &lo, &hi);
  for (int64_t k = 1; k <= jb->n_iter; ++k) {
    int check = jb->mode == 1 ? (k % jb->K == 0) : (jb->measure_last && k == jb->n_iter);
    if (jb->is_f32) {
      float m = 0.0f, w = (float)jb->omega;
      phase_f32((float*)jb->u, jb->cols, 0, lo, hi, 0, w, check, &m);
      pthread_barrier_wait(&jb->bar);
      phase_f32((float*)jb->u, jb->cols, 0, lo, hi, 1, w, check, &m);
      jb->partial_max[ta->p] = (double)m;
    } else {
      double m = 0.0;
      phase_f64((double*)jb->u, jb->cols, 0, lo, hi, 0, jb->omega, check, &m);
      pthread_barrier_wait(&jb->bar);
      phase_f64((double*)jb->u, jb->cols, 0, lo, hi, 1, jb->omega, check, &m);
      jb->partial_max[ta->p] = m;
    }
    pthread_barrier_wait(&jb->bar);
    if (ta->p == 0) {
      orc_report* rep = jb->rep;
      rep->half_sweeps += 2;
      rep->iters = k;
      if (check) {
        double m = 0.0;                       /* serial combine */
        for (int q = 0; q < jb->P; ++q) {
          double d = jb->partial_max[q];
          if (d > m || d != d) m = d;
        }
        rep->checks += 1;
        rep->max_change = m;
        if (jb->mode == 1 && m < jb->tol) {
          rep->status = ORC_DONE;
          jb->stop = 1;
        }
      }
    }
    pthread_barrier_wait(&jb->bar);
    if (jb->stop) break;
  }
  return NULL;
}

static int run_threads(void* u, int is_f32, int64_t rows, int64_t cols, double omega, int mode,
                       int64_t n_iter, double tol, int64_t K, int measure_last, int nthreads,
                       orc_report* rep) {
  memset(rep, 0, sizeof(*rep));
  if (!check_args(rows, cols, omega, mode, n_iter, tol, K) || nthreads < 1) {
    rep->status = ORC_E_INVAL;
    return ORC_E_INVAL;
  }
  if (nthreads > rows) nthreads = (int)rows;
  tjob jb;
  memset(&jb, 0, sizeof(jb));
  jb.u = u;
  jb.rows = rows;
  jb.cols = cols;
  jb.omega = omega;
  jb.mode = mode;
  jb.n_iter = n_iter;
  jb.tol = tol;
  jb.K = K;
  jb.measure_last = measure_last;
  jb.P = nthreads;
  jb.is_f32 = is_f32;
  jb.rep = rep;
  jb.partial_max = (double*)calloc((size_t)nthreads, sizeof(double));
  rep->status = mode == 1 ? ORC_NOT_CONVERGED : ORC_DONE;
  pthread_barrier_init(&jb.bar, NULL, (unsigned)nthreads);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  targ* ta = (targ*)malloc(sizeof(targ) * (size_t)nthreads);
  for (int p = 0; p < nthreads; ++p) {
    ta[p].job = &jb;
    ta[p].p = p;
    pthread_create(&th[p], NULL, worker, &ta[p]);
  }
  for (int p = 0; p < nthreads; ++p) pthread_join(th[p], NULL);
  pthread_barrier_destroy(&jb.bar);
  free(th);
  free(ta);
  free(jb.partial_max);
  return rep->status;
}

int orc_sor_run_threads_f64(double* u, int64_t rows, int64_t cols, double omega, int mode,
                            int64_t n_iter, double tol, int64_t K, int measure_last,
                            int nthreads, orc_report* rep) {
  return run_threads(u, 0, rows, cols, omega, mode, n_iter, tol, K, measure_last, nthreads, rep);
}
int orc_sor_run_threads_f32(float* u, int64_t rows, int64_t cols, double omega, int mode,
                            int64_t n_iter, double tol, int64_t K, int measure_last,
                            int nthreads, orc_report* rep) {
  return run_threads(u, 1, rows, cols, omega, mode, n_iter, tol, K, measure_last, nthreads, rep);
}

/* ------------------------------------------------------------------------ */
/* Jacobi: every interior cell from the previous iterate only.        */
/* Jacobi, both modes (NEXT-2): a plain copy of X_{k-1}, then
 * every interior cell of X_k from it, row by row.                           */
#define DEFINE_JACOBI(T, SUF)                                                     \
  int orc_jacobi_run_##SUF(T* u, int64_t rows, int64_t cols, int mode, int64_t n_iter, \
                           double tol, int64_t K, int measure_last, orc_report* rep) { \
    memset(rep, 0, sizeof(*rep));                                                 \
    if (!check_args(rows, cols, 1.0, mode, n_iter, tol, K)) {                     \
      rep->status = ORC_E_INVAL;                                                  \
      return ORC_E_INVAL;                                                         \
    }                                                                             \
    const int64_t ld = cols + 2, n = (rows + 2) * ld;                             \
    T* prev = (T*)malloc((size_t)n * sizeof(T));                                  \
    if (!prev) {                                                                  \
      rep->status = ORC_E_INVAL;                                                  \
      return ORC_E_INVAL;                                                         \
    }                                                                             \
    const T q = (T)0.25;                                                          \
    rep->status = mode == 1 ? ORC_NOT_CONVERGED : ORC_DONE;                       \
    for (int64_t k = 1; k <= n_iter; ++k) {                                       \
      int check = mode == 1 ? (k % K == 0) : (measure_last && k == n_iter);       \
      memcpy(prev, u, (size_t)n * sizeof(T));          /* X_{k-1} */             \
      T m = (T)0;                                                                 \
      for (int64_t i = 1; i <= rows; ++i)                                         \
        for (int64_t j = 1; j <= cols; ++j) {                                     \
          const T* c = prev + i * ld + j;                                         \
          T s = (c[-ld] + c[ld]) + (c[-1] + c[1]);     /* (N+S)+(W+E) */          \
          T a = q * s;                                                            \
          if (check) {                                                            \
            T d = (T)fabs((double)(a - c[0]));                                    \
            if (d > m || d != d) m = d;                                           \
          }                                                                       \
          u[i * ld + j] = a;                                                      \
        }                                                                         \
      rep->half_sweeps += 1;                                                      \
      rep->iters = k;                                                             \
      if (check) {                                                                \
        rep->checks += 1;                                                         \
        rep->max_change = (double)m;                                              \
        if (mode == 1 && (double)m < tol) {                                       \
          rep->status = ORC_DONE;                                                 \
          break;                                                                  \
        }                                                                         \
      }                                                                           \
    }                                                                             \
    free(prev);                                                                   \
    return rep->status;                                                           \
  }
DEFINE_JACOBI(double, f64)
DEFINE_JACOBI(float, f32)

/* 3-D red-black SOR (NEXT-3): one colour phase, then Algorithm 1's loop.   */
#define DEFINE_SOR3D(T, SUF, ABS)                                                 \
  static void phase3d_##SUF(T* u, int64_t nz, int64_t ny, int64_t nx, int c, T w, int check, T* m) { \
    const int64_t lx = nx + 2, lp = (ny + 2) * lx;                               \
    const T six = (T)6;                                                          \
    for (int64_t z = 1; z <= nz; ++z)                                            \
      for (int64_t y = 1; y <= ny; ++y) {                                        \
        const int64_t x0 = (((z + y + 1) & 1) == c) ? 1 : 2;  /* (z+y+x)%2 == c */ \
        for (int64_t x = x0; x <= nx; x += 2) {                                  \
          T* uc = u + z * lp + y * lx + x;                                       \
          T s = ((uc[-lx] + uc[lx]) + (uc[-1] + uc[1])) + (uc[-lp] + uc[lp]);   \
          T a = s / six;                                                         \
          T r = a - uc[0];                                                       \
          T un = uc[0] + w * r;                                                  \
          if (check) {                                                           \
            T d = ABS(un - uc[0]);                                               \
            if (d > *m || d != d) *m = d;                                        \
          }                                                                      \
          uc[0] = un;                                                            \
        }                                                                        \
      }                                                                          \
  }                                                                              \
  int orc_sor3d_run_##SUF(T* u, int64_t nz, int64_t ny, int64_t nx, double omega, int mode, \
                          int64_t n_iter, double tol, int64_t K, int measure_last, orc_report* rep) { \
    memset(rep, 0, sizeof(*rep));                                                \
    if (nz < 1 || !check_args(ny, nx, omega, mode, n_iter, tol, K)) {            \
      rep->status = ORC_E_INVAL;                                                 \
      return ORC_E_INVAL;                                                        \
    }                                                                            \
    const T w = (T)omega;                                                        \
    rep->status = mode == 1 ? ORC_NOT_CONVERGED : ORC_DONE;                      \
    for (int64_t k = 1; k <= n_iter; ++k) {                                      \
      int check = mode == 1 ? (k % K == 0) : (measure_last && k == n_iter);      \
      T m = (T)0;                                                                \
      phase3d_##SUF(u, nz, ny, nx, 0, w, check, &m);   /* red */                 \
      phase3d_##SUF(u, nz, ny, nx, 1, w, check, &m);   /* black */               \
      rep->half_sweeps += 2;                                                     \
      rep->iters = k;                                                            \
      if (check) {                                                               \
        rep->checks += 1;                                                        \
        rep->max_change = (double)m;                                             \
        if (mode == 1 && (double)m < tol) {                                      \
          rep->status = ORC_DONE;                                                \
          break;                                                                 \
        }                                                                        \
      }                                                                          \
    }                                                                            \
    return rep->status;                                                          \
  }
DEFINE_SOR3D(double, f64, fabs)
DEFINE_SOR3D(float, f32, fabsf)

int orc_jacobi_f64(double* u, int64_t rows, int64_t cols, int64_t maxit, double tol,
                   orc_report* rep) {
  memset(rep, 0, sizeof(*rep));
  if (rows < 1 || cols < 1 || maxit < 1 || !(tol > 0.0)) {
    rep->status = ORC_E_INVAL;
    return ORC_E_INVAL;
  }
  const int64_t ld = cols + 2, n = (rows + 2) * ld;
  double* v = (double*)malloc((size_t)n * sizeof(double));
  memcpy(v, u, (size_t)n * sizeof(double));
  rep->status = ORC_NOT_CONVERGED;
  for (int64_t k = 1; k <= maxit; ++k) {
    double m = 0.0;
    for (int64_t i = 1; i <= rows; ++i)
      for (int64_t j = 1; j <= cols; ++j) {
        double s = (u[(i - 1) * ld + j] + u[(i + 1) * ld + j]) + (u[i * ld + j - 1] + u[i * ld + j + 1]);
        double a = 0.25 * s;
        double d = fabs(a - u[i * ld + j]);
        if (d > m || d != d) m = d;
        v[i * ld + j] = a;
      }
    memcpy(u, v, (size_t)n * sizeof(double));
    rep->iters = k;
    rep->checks += 1;
    rep->max_change = m;
    if (m < tol) {
      rep->status = ORC_DONE;
      break;
    }
  }
  free(v);
  return rep->status;
}

/* ------------------------------------------------------------------------ */
/* Dense direct solve of the discrete Laplace system (brute force pin P3).   */
int orc_dense_solve_f64(double* u, int64_t rows, int64_t cols) {
  const int64_t n = rows * cols, ld = cols + 2;
  if (rows < 1 || cols < 1 || n > 4096) return -1;
  double* A = (double*)calloc((size_t)(n * n), sizeof(double));
  double* b = (double*)calloc((size_t)n, sizeof(double));
  if (!A || !b) {
    free(A);
    free(b);
    return -1;
  }
#define IDX(i, j) (((i) - 1) * cols + ((j) - 1))
  for (int64_t i = 1; i <= rows; ++i)
    for (int64_t j = 1; j <= cols; ++j) {
      const int64_t r = IDX(i, j);
      A[r * n + r] = 4.0;
      const int64_t ni[4] = {i - 1, i + 1, i, i};
      const int64_t nj[4] = {j, j, j - 1, j + 1};
      for (int t = 0; t < 4; ++t) {
        if (ni[t] < 1 || ni[t] > rows || nj[t] < 1 || nj[t] > cols)
          b[r] += u[ni[t] * ld + nj[t]];
        else
          A[r * n + IDX(ni[t], nj[t])] -= 1.0;
      }
    }
  for (int64_t c = 0; c < n; ++c) { /* forward elimination, partial pivoting */
    int64_t p = c;
    for (int64_t r = c + 1; r < n; ++r)
      if (fabs(A[r * n + c]) > fabs(A[p * n + c])) p = r;
    if (p != c) {
      for (int64_t k = 0; k < n; ++k) {
        double t = A[c * n + k];
        A[c * n + k] = A[p * n + k];
        A[p * n + k] = t;
      }
      double t = b[c];
      b[c] = b[p];
      b[p] = t;
    }
    for (int64_t r = c + 1; r < n; ++r) {
      double f = A[r * n + c] / A[c * n + c];
      if (f == 0.0) continue;
      for (int64_t k = c; k < n; ++k) A[r * n + k] -= f * A[c * n + k];
      b[r] -= f * b[c];
    }
  }
  for (int64_t c = n - 1; c >= 0; --c) { /* back substitution */
    double s = b[c];
    for (int64_t k = c + 1; k < n; ++k) s -= A[c * n + k] * b[k];
    b[c] = s / A[c * n + c];
  }
  for (int64_t i = 1; i <= rows; ++i)
    for (int64_t j = 1; j <= cols; ++j) u[i * ld + j] = b[IDX(i, j)];
#undef IDX
  free(A);
  free(b);
  return 0;
}


/* 3-D brute force: 6u - sum(interior neighbours) = sum(shell neighbours). */
int orc_dense_solve3d_f64(double* u, int64_t nz, int64_t ny, int64_t nx) {
  const int64_t n = nz * ny * nx;
  if (n > 1728) return -1;
  const int64_t lx = nx + 2, lp = (ny + 2) * lx;
  double* A = (double*)calloc((size_t)(n * (n + 1)), sizeof(double));
  if (!A) return -1;
#define IDX(z, y, x) (((z) - 1) * ny * nx + ((y) - 1) * nx + ((x) - 1))
  for (int64_t z = 1; z <= nz; ++z)
    for (int64_t y = 1; y <= ny; ++y)
      for (int64_t x = 1; x <= nx; ++x) {
        const int64_t r = IDX(z, y, x);
        double* row = A + r * (n + 1);
        row[r] = 6.0;
        const int64_t nb[6][3] = {{z, y - 1, x}, {z, y + 1, x}, {z, y, x - 1}, {z, y, x + 1}, {z - 1, y, x}, {z + 1, y, x}};
        for (int k = 0; k < 6; ++k) {
          const int64_t zz = nb[k][0], yy = nb[k][1], xx = nb[k][2];
          if (zz >= 1 && zz <= nz && yy >= 1 && yy <= ny && xx >= 1 && xx <= nx)
            row[IDX(zz, yy, xx)] -= 1.0;
          else
            row[n] += u[zz * lp + yy * lx + xx];
        }
      }
  for (int64_t c = 0; c < n; ++c) {  /* Gaussian elimination, partial pivoting */
    int64_t p = c;
    for (int64_t r = c + 1; r < n; ++r)
      if (fabs(A[r * (n + 1) + c]) > fabs(A[p * (n + 1) + c])) p = r;
    if (p != c)
      for (int64_t k = 0; k <= n; ++k) {
        double t = A[c * (n + 1) + k];
        A[c * (n + 1) + k] = A[p * (n + 1) + k];
        A[p * (n + 1) + k] = t;
      }
    for (int64_t r = c + 1; r < n; ++r) {
      const double f = A[r * (n + 1) + c] / A[c * (n + 1) + c];
      if (f != 0.0)
        for (int64_t k = c; k <= n; ++k) A[r * (n + 1) + k] -= f * A[c * (n + 1) + k];
    }
  }
  for (int64_t c = n - 1; c >= 0; --c) {
    double v = A[c * (n + 1) + n];
    for (int64_t k = c + 1; k < n; ++k) v -= A[c * (n + 1) + k] * A[k * (n + 1) + n];
    A[c * (n + 1) + n] = v / A[c * (n + 1) + c];
  }
  for (int64_t z = 1; z <= nz; ++z)
    for (int64_t y = 1; y <= ny; ++y)
      for (int64_t x = 1; x <= nx; ++x) u[z * lp + y * lx + x] = A[IDX(z, y, x) * (n + 1) + n];
#undef IDX
  free(A);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* NEXT-4: the two parallel SOR variants the paper names beside
 * red-black SOR, "multi-color SOR" and "block-parallel SOR".  The paper only
 * names them; the definitions below are readings N4-1 and N4-2 of DESIGN.md
 * §3 (the textbook orderings), written out plainly.  Every update is Eq. 1
 * in the canonical order of orc_cell_update (readings #2-#4),
 * in place, reading the latest values; |delta| = |u' - u| (reading #5);
 * Algorithm 1's loop, cadence and strict stop test as orc_sor_run.
 *
 * Multi-colour (N4-1): colour(i, j) = (ca*i + cb*j) mod nc (storage indices,
 * 1..rows x 1..cols; non-negative residue).  Valid iff ca, cb are not
 * multiples of nc, so 5-point neighbours never share a colour.  One
 * iteration = phases p = 0, 1, ..., nc-1; phase p updates every cell of
 * colour p.  (ca, cb, nc) = (1, 1, 2) is the paper's red-black SOR
 * (P:149).
 *
 * Block (N4-2): the interior is cut into B x B blocks anchored at cell (1, 1)
 * (block (bi, bj) = ((i-1)/B, (j-1)/B), clipped at the edges); blocks are
 * coloured like a chessboard, red iff bi+bj even.  One iteration = the red
 * blocks, then the black blocks; inside a block the cells are updated in
 * natural (lexicographic) order, as Code 1's sequential sweep.
 * B = 1 is red-black SOR; B >= max(rows, cols) is natural-order SOR.        */
static int64_t mc_colour(int64_t ca, int64_t cb, int64_t nc, int64_t i, int64_t j) {
  int64_t c = (ca * i + cb * j) % nc;
  return c < 0 ? c + nc : c;
}

#define DEFINE_VARIANTS(T, SUF, ABS)                                                   \
  static void cell_##SUF(T* u, int64_t ld, int64_t i, int64_t j, T w, int check, T* m) { \
    const T q = (T)0.25;                                                              \
    T* uc = u + i * ld + j;                                                           \
    T s = (uc[-ld] + uc[ld]) + (uc[-1] + uc[1]);                                      \
    T a = q * s;                                                                      \
    T r = a - uc[0];                                                                  \
    T un = uc[0] + w * r;                                                             \
    if (check) {                                                                      \
      T d = ABS(un - uc[0]);                                                          \
      if (d > *m || d != d) *m = d;                                                   \
    }                                                                                 \
    uc[0] = un;                                                                       \
  }                                                                                   \
  /* kind 0: multi-colour (p1, p2, p3) = (ca, cb, nc); kind 1: block, p1 = B */      \
  int orc_variant_run_##SUF(T* u, int64_t rows, int64_t cols, int kind, int64_t p1,   \
                            int64_t p2, int64_t p3, double omega, int mode,           \
                            int64_t n_iter, double tol, int64_t K, int measure_last,  \
                            orc_report* rep) {                                        \
    memset(rep, 0, sizeof(*rep));                                                     \
    int ok = check_args(rows, cols, omega, mode, n_iter, tol, K);                     \
    if (kind == 0) ok = ok && p3 >= 2 && p1 % p3 != 0 && p2 % p3 != 0;                \
    else if (kind == 1) ok = ok && p1 >= 1;                                           \
    else ok = 0;                                                                      \
    if (!ok) {                                                                        \
      rep->status = ORC_E_INVAL;                                                      \
      return ORC_E_INVAL;                                                             \
    }                                                                                 \
    const int64_t ld = cols + 2;                                                      \
    const T w = (T)omega;                                                             \
    rep->status = mode == 1 ? ORC_NOT_CONVERGED : ORC_DONE;                           \
    for (int64_t k = 1; k <= n_iter; ++k) {                    /* P:301 */            \
      int check = mode == 1 ? (k % K == 0) : (measure_last && k == n_iter);           \
      T m = (T)0;                                                                     \
      if (kind == 0) {                                                                \
        for (int64_t p = 0; p < p3; ++p) {                     /* colour phases */    \
          for (int64_t i = 1; i <= rows; ++i)                                         \
            for (int64_t j = 1; j <= cols; ++j)                                       \
              if (mc_colour(p1, p2, p3, i, j) == p) cell_##SUF(u, ld, i, j, w, check, &m); \
          rep->half_sweeps += 1;                                                      \
        }                                                                             \
      } else {                                                                        \
        const int64_t B = p1, nbi = (rows + B - 1) / B, nbj = (cols + B - 1) / B;      \
        for (int c = 0; c < 2; ++c) {                          /* red, then black */  \
          for (int64_t bi = 0; bi < nbi; ++bi)                                        \
            for (int64_t bj = 0; bj < nbj; ++bj) {                                    \
              if ((bi + bj) % 2 != c) continue;                                       \
              for (int64_t i = 1 + bi * B; i <= rows && i < 1 + (bi + 1) * B; ++i)    \
                for (int64_t j = 1 + bj * B; j <= cols && j < 1 + (bj + 1) * B; ++j)  \
                  cell_##SUF(u, ld, i, j, w, check, &m);                              \
            }                                                                         \
          rep->half_sweeps += 1;                                                      \
        }                                                                             \
      }                                                                               \
      rep->iters = k;                                                                 \
      if (check) {                                                                    \
        rep->checks += 1;                                                             \
        rep->max_change = (double)m;                                                  \
        if (mode == 1 && (double)m < tol) {                    /* P:327 */            \
          rep->status = ORC_DONE;                                                     \
          break;                                                                      \
        }                                                                             \
      }                                                                               \
    }                                                                                 \
    return rep->status;                                                               \
  }
DEFINE_VARIANTS(double, f64, fabs)
DEFINE_VARIANTS(float, f32, fabsf)
