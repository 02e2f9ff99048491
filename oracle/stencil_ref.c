/*
 * ORACLE — test / baseline infrastructure only; never linked by the product.
 *
 * Plain-C restatement of the reference interpreter executing the jacobi_2d
 * and heat_3d gradient programs (the C1/C2/C5 hot path), i.e. exactly the
 * programs tools/workloads_ref.py builds and the reference AD reverses:
 *
 *   forward  (interpreter.py:478-507 over the two maps of state `step`)
 *     for t in [1, T): B[x] = body(A) on the interior; A[x] = body(B)
 *     O = sum(A)                                   (reduce_sum, :447-451)
 *   reverse  (the emitted adjoint maps, autodiff.py:962-1081)
 *     A__grad[all] += O__grad                      (broadcast map, :940-960)
 *     for t = T-1 .. 1:
 *       per interior point x of the adjoint of map 2, in point order:
 *         g = A__grad[x]; B__grad[x + e] += c_e * g  (wcr sum); A__grad[x] = 0  (_z)
 *       per interior point x of the adjoint of map 1:
 *         g = B__grad[x]; A__grad[x + e] += c_e * g; B__grad[x] = 0
 *
 * Tasklet bodies are evaluated with the reference's expression order
 * (workloads_ref.py HEAT_BODY / jacobi body). Work is split over the outer
 * dimension with POSIX threads (this image has no OpenMP runtime); the
 * scatter-add maps run in two phases (even then odd chunks of >= 2 planes),
 * so no two threads touch the same element and the per-element accumulation
 * order differs from the strictly sequential reference only by
 * floating-point reassociation.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static int g_threads = 1;

typedef struct {
  void (*fn)(void *ctx, int64_t lo, int64_t hi);
  void *ctx;
  int64_t lo, hi;
} job_t;

static void *run_job(void *p) {
  job_t *j = (job_t *)p;
  j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}

/* static split of [lo, hi) over g_threads threads */
static void parallel_for(int64_t lo, int64_t hi, void (*fn)(void *, int64_t, int64_t), void *ctx) {
  int nt = g_threads;
  if (hi - lo < nt) nt = (int)(hi - lo);
  if (nt <= 1) {
    if (hi > lo) fn(ctx, lo, hi);
    return;
  }
  pthread_t th[256];
  job_t jobs[256];
  if (nt > 256) nt = 256;
  for (int t = 0; t < nt; ++t) {
    jobs[t].fn = fn;
    jobs[t].ctx = ctx;
    jobs[t].lo = lo + (hi - lo) * t / nt;
    jobs[t].hi = lo + (hi - lo) * (t + 1) / nt;
    pthread_create(&th[t], NULL, run_job, &jobs[t]);
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}

#define IDX3(i, j, k) (((int64_t)(i) * n + (j)) * n + (k))
#define IDX2(i, j) ((int64_t)(i) * n + (j))

static double heat_body(double cc, double ip, double im, double jp, double jm, double kp, double km) {
  /* (add (add (add cc (mul 0.125 (add (sub ip (mul 2.0 cc)) im)))
   *           (mul 0.125 (add (sub jp (mul 2.0 cc)) jm)))
   *      (mul 0.125 (add (sub kp (mul 2.0 cc)) km))) */
  double a = cc + 0.125 * ((ip - 2.0 * cc) + im);
  double b = a + 0.125 * ((jp - 2.0 * cc) + jm);
  return b + 0.125 * ((kp - 2.0 * cc) + km);
}

typedef struct {
  int n;
  const double *src;
  double *dst;
} sweep_ctx;

static void heat_sweep_rows(void *p, int64_t i0, int64_t i1) {
  sweep_ctx *c = (sweep_ctx *)p;
  const int n = c->n;
  const double *src = c->src;
  double *dst = c->dst;
  for (int64_t i = i0; i < i1; ++i)
    for (int j = 1; j < n - 1; ++j)
      for (int k = 1; k < n - 1; ++k)
        dst[IDX3(i, j, k)] = heat_body(src[IDX3(i, j, k)], src[IDX3(i + 1, j, k)], src[IDX3(i - 1, j, k)],
                                       src[IDX3(i, j + 1, k)], src[IDX3(i, j - 1, k)], src[IDX3(i, j, k + 1)],
                                       src[IDX3(i, j, k - 1)]);
}

static void heat_sweep(int n, const double *src, double *dst) {
  sweep_ctx c = {n, src, dst};
  parallel_for(1, n - 1, heat_sweep_rows, &c);
}

/* adjoint of dst = heat(src) on the interior: scatter g = dgd[x] into dsg,
 * then clear dgd[x]; outputs in tasklet order _dcc, _dip, _dim, _djp, _djm,
 * _dkp, _dkm, _z (reference adj_map output order). */
static void heat_adjoint_chunk(int n, int i0, int i1, double *dgd, double *dsg) {
  for (int i = i0; i < i1; ++i)
    for (int j = 1; j < n - 1; ++j)
      for (int k = 1; k < n - 1; ++k) {
        const double g = dgd[IDX3(i, j, k)];
        dsg[IDX3(i, j, k)] += 0.25 * g;
        dsg[IDX3(i + 1, j, k)] += 0.125 * g;
        dsg[IDX3(i - 1, j, k)] += 0.125 * g;
        dsg[IDX3(i, j + 1, k)] += 0.125 * g;
        dsg[IDX3(i, j - 1, k)] += 0.125 * g;
        dsg[IDX3(i, j, k + 1)] += 0.125 * g;
        dsg[IDX3(i, j, k - 1)] += 0.125 * g;
        dgd[IDX3(i, j, k)] = 0.0;
      }
}

typedef struct {
  int n, phase, nchunks, planes;
  void (*chunk)(int, int, int, double *, double *);
  double *dgd, *dsg;
} phase_ctx;

static void phase_chunks(void *p, int64_t c0, int64_t c1) {
  phase_ctx *c = (phase_ctx *)p;
  for (int64_t q = c0; q < c1; ++q) {
    int ch = 2 * (int)q + c->phase;
    if (ch >= c->nchunks) continue;
    int a = 1 + (int)((int64_t)c->planes * ch / c->nchunks);
    int b = 1 + (int)((int64_t)c->planes * (ch + 1) / c->nchunks);
    c->chunk(c->n, a, b, c->dgd, c->dsg);
  }
}

static void two_phase(int n, void (*chunk)(int, int, int, double *, double *), double *dgd, double *dsg) {
  int planes = n - 2;
  if (planes <= 0) return;
  int nchunks = 2 * g_threads;
  if (nchunks > planes / 2) nchunks = planes / 2;
  if (nchunks < 1) nchunks = 1;
  for (int phase = 0; phase < 2; ++phase) {
    phase_ctx c = {n, phase, nchunks, planes, chunk, dgd, dsg};
    parallel_for(0, (nchunks + 1) / 2, phase_chunks, &c);
  }
}

typedef struct {
  const double *x;
  double part[256];
  int64_t total;
  int nt;
} sum_ctx;

static void sum_part(void *p, int64_t t0, int64_t t1) {
  sum_ctx *c = (sum_ctx *)p;
  for (int64_t t = t0; t < t1; ++t) {
    int64_t lo = c->total * t / c->nt, hi = c->total * (t + 1) / c->nt;
    double s = 0.0;
    for (int64_t q = lo; q < hi; ++q) s += c->x[q];
    c->part[t] = s;
  }
}

static double sum_all(const double *x, int64_t total) {
  sum_ctx c;
  c.x = x;
  c.total = total;
  c.nt = g_threads > 256 ? 256 : g_threads;
  parallel_for(0, c.nt, sum_part, &c);
  double s = 0.0;
  for (int t = 0; t < c.nt; ++t) s += c.part[t];
  return s;
}

static void set_threads(int threads) {
  long hw = sysconf(_SC_NPROCESSORS_ONLN);
  g_threads = threads > 0 ? threads : (int)(hw > 0 ? hw : 1);
  if (g_threads > 256) g_threads = 256;
}

int heat3d_gradient(int n, int tsteps, const double *A0, const double *B0, double seed, double *value,
                    double *gradA, int threads) {
  set_threads(threads);
  const int64_t total = (int64_t)n * n * n;
  double *A = malloc(total * sizeof(double)), *B = malloc(total * sizeof(double));
  double *Bg = calloc(total, sizeof(double));
  if (!A || !B || !Bg) return 1;
  memcpy(A, A0, total * sizeof(double));
  memcpy(B, B0, total * sizeof(double));
  for (int t = 1; t < tsteps; ++t) {
    heat_sweep(n, A, B);
    heat_sweep(n, B, A);
  }
  *value = sum_all(A, total);
  for (int64_t q = 0; q < total; ++q) gradA[q] = seed;
  for (int t = tsteps - 1; t >= 1; --t) {
    two_phase(n, heat_adjoint_chunk, gradA, Bg); /* adjoint of A = heat(B) */
    two_phase(n, heat_adjoint_chunk, Bg, gradA); /* adjoint of B = heat(A) */
  }
  free(A);
  free(B);
  free(Bg);
  return 0;
}

static double jac_body(double cc, double ww, double ee, double ss, double nn) {
  /* (mul 0.2 (add (add (add (add cc ww) ee) ss) nn)) */
  return 0.2 * ((((cc + ww) + ee) + ss) + nn);
}

static void jac_sweep_rows(void *p, int64_t i0, int64_t i1) {
  sweep_ctx *c = (sweep_ctx *)p;
  const int n = c->n;
  const double *src = c->src;
  double *dst = c->dst;
  for (int64_t i = i0; i < i1; ++i)
    for (int j = 1; j < n - 1; ++j)
      dst[IDX2(i, j)] = jac_body(src[IDX2(i, j)], src[IDX2(i, j - 1)], src[IDX2(i, j + 1)], src[IDX2(i + 1, j)],
                                 src[IDX2(i - 1, j)]);
}

static void jac_sweep(int n, const double *src, double *dst) {
  sweep_ctx c = {n, src, dst};
  parallel_for(1, n - 1, jac_sweep_rows, &c);
}

static void jac_adjoint_chunk(int n, int i0, int i1, double *dgd, double *dsg) {
  for (int i = i0; i < i1; ++i)
    for (int j = 1; j < n - 1; ++j) {
      const double g = dgd[IDX2(i, j)];
      dsg[IDX2(i, j)] += 0.2 * g;
      dsg[IDX2(i, j - 1)] += 0.2 * g;
      dsg[IDX2(i, j + 1)] += 0.2 * g;
      dsg[IDX2(i + 1, j)] += 0.2 * g;
      dsg[IDX2(i - 1, j)] += 0.2 * g;
      dgd[IDX2(i, j)] = 0.0;
    }
}

int jacobi2d_gradient(int n, int tsteps, const double *A0, const double *B0, double seed, double *value,
                      double *gradA, int threads) {
  set_threads(threads);
  const int64_t total = (int64_t)n * n;
  double *A = malloc(total * sizeof(double)), *B = malloc(total * sizeof(double));
  double *Bg = calloc(total, sizeof(double));
  if (!A || !B || !Bg) return 1;
  memcpy(A, A0, total * sizeof(double));
  memcpy(B, B0, total * sizeof(double));
  for (int t = 1; t < tsteps; ++t) {
    jac_sweep(n, A, B);
    jac_sweep(n, B, A);
  }
  *value = sum_all(A, total);
  for (int64_t q = 0; q < total; ++q) gradA[q] = seed;
  for (int t = tsteps - 1; t >= 1; --t) {
    two_phase(n, jac_adjoint_chunk, gradA, Bg);
    two_phase(n, jac_adjoint_chunk, Bg, gradA);
  }
  free(A);
  free(B);
  free(Bg);
  return 0;
}

/*
 * corpus seidel_stencil (reference examples.py:159-182), forward only: the
 * in-place Gauss-Seidel nest for t, i, j in loop order, body
 * (mul 0.2 (add (add (add cc nn) (add ss ww)) ee)) in the reference's
 * evaluation order, then O = sum(A). Sequential by construction (single
 * thread); the program is linear, so parity of the engine's gradient is
 * checked through O(A + d) - O(A) = <grad, d>.
 */
double seidel2d_value(int n, int tsteps, const double *A0) {
  const int64_t total = (int64_t)n * n;
  double *A = malloc(total * sizeof(double));
  if (!A) return 0.0;
  memcpy(A, A0, total * sizeof(double));
  for (int t = 0; t < tsteps; ++t)
    for (int i = 1; i < n - 1; ++i)
      for (int j = 1; j < n - 1; ++j) {
        const double cc = A[IDX2(i, j)], nn = A[IDX2(i - 1, j)], ss = A[IDX2(i + 1, j)];
        const double ww = A[IDX2(i, j - 1)], ee = A[IDX2(i, j + 1)];
        A[IDX2(i, j)] = 0.2 * (((cc + nn) + (ss + ww)) + ee);
      }
  double v = 0.0;
  for (int64_t q = 0; q < total; ++q) v += A[q];
  free(A);
  return v;
}

int stencil_ref_max_threads(void) {
  set_threads(0);
  return g_threads;
}
