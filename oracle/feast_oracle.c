/*
 * oracle/feast_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference (feastlite) FEAST hot path, used as the CPU checker and, in bench.py, as the
 * "port" CPU baseline when the compiled reference is unavailable. Never the product path.
 *
 * Every function follows the reference routine named beside it (paths relative to
 * /root/reference/proj), in the same floating-point operation order, so on the golden
 * fixtures it reproduces the reference bit-for-bit (tests/test_oracle_pins.py pins it
 * against the reference's known-answer tests and against fixtures the reference made).
 * Complex arithmetic uses C99 _Complex double, which GCC evaluates with the same builtins
 * as std::complex<double>.
 *
 * Exports the same ref_* entry points as oracle/ref_driver.cpp.
 */
#define _GNU_SOURCE
#include <complex.h>
#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "feast_gpu.h"

typedef double _Complex cplx;

static __thread char g_err[256];
static __thread int g_code;

#define FAIL(code, msg)                              \
  do {                                               \
    g_code = (code);                                 \
    snprintf(g_err, sizeof g_err, "%s", (msg));      \
    goto fail;                                       \
  } while (0)

const char* ref_last_error(void) { return g_err; }
int ref_max_reduced_dimension(void) { return 4096; }

/* ---------------------------------------------------------------- mt19937_64 */
typedef struct { uint64_t mt[312]; int idx; } mt64;
static void mt64_seed(mt64* g, uint64_t s) {
  g->mt[0] = s;
  for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}
static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}
/* random_block<double> core.hpp:84-106 */
static void random_block(int n, int m, uint64_t seed, double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < n; ++i) {
      const double u = (double)(mt64_next(&g) >> 11) * 0x1p-53;
      out[i + (size_t)j * n] = 2.0 * u - 1.0;
    }
}

/* ---------------------------------------------------------------- quadrature */
/* quadrature.cpp:14-25 */
static void legendre_eval(int n, long double x, long double* p, long double* dp) {
  long double p0 = 1.0L, p1 = x;
  for (int k = 2; k <= n; ++k) {
    const long double p2 = ((2.0L * k - 1.0L) * x * p1 - (k - 1.0L) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  *p = p1;
  *dp = n * (x * p1 - p0) / (x * x - 1.0L);
}
/* gauss_legendre quadrature.cpp:28-67 */
static int gauss_legendre(int n, double* nodes, double* weights) {
  if (n < 1 || n > 64) {
    g_code = FEAST_EINPUT;
    snprintf(g_err, sizeof g_err, "gauss_legendre: point count out of supported range");
    return FEAST_EINPUT;
  }
  const long double pi = 3.14159265358979323846264338327950288L;
  const int half = n / 2;
  for (int i = 0; i < half; ++i) {
    long double x = cos((double)(pi * (i + 0.75L) / (n + 0.5L)));
    long double p = 0.0L, dp = 1.0L;
    for (int it = 0; it < 100; ++it) {
      legendre_eval(n, x, &p, &dp);
      const long double dx = p / dp;
      x -= dx;
      if (fabs((double)dx) <= 1e-15) {
        legendre_eval(n, x, &p, &dp);
        x -= p / dp;
        break;
      }
    }
    legendre_eval(n, x, &p, &dp);
    const long double w = 2.0L / ((1.0L - x * x) * dp * dp);
    nodes[n - 1 - i] = (double)x;
    nodes[i] = -(double)x;
    weights[n - 1 - i] = (double)w;
    weights[i] = (double)w;
  }
  if (n % 2 == 1) {
    long double p, dp;
    legendre_eval(n, 0.0L, &p, &dp);
    nodes[half] = 0.0;
    weights[half] = (double)(2.0L / (dp * dp));
  }
  return 0;
}

typedef struct {
  int ne;
  double lo, hi, radius;
  double node[64], weight[64], theta[64];
  cplx z[64];
} contour_t;

/* build_contour quadrature.cpp:69-87 */
static int build_contour(double lo, double hi, int ne, contour_t* c) {
  if (!(lo < hi)) {
    g_code = FEAST_EINPUT;
    snprintf(g_err, sizeof g_err, "SearchInterval: lambda_min must be strictly below lambda_max");
    return FEAST_EINPUT;
  }
  double scale = 1.0;
  if (fabs(lo) > scale) scale = fabs(lo);
  if (fabs(hi) > scale) scale = fabs(hi);
  if (hi - lo < 1e-12 * scale) {
    g_code = FEAST_EINPUT;
    snprintf(g_err, sizeof g_err, "build_contour: interval is degenerate at round-off scale");
    return FEAST_EINPUT;
  }
  int rc = gauss_legendre(ne, c->node, c->weight);
  if (rc) return rc;
  c->ne = ne;
  c->lo = lo;
  c->hi = hi;
  c->radius = 0.5 * (hi - lo);
  const double mid = 0.5 * (lo + hi);
  for (int e = 0; e < ne; ++e) {
    c->theta[e] = -(M_PI / 2.0) * (c->node[e] - 1.0);
    c->z[e] = CMPLX(mid + c->radius * cos(c->theta[e]), c->radius * sin(c->theta[e]));
  }
  return 0;
}

/* ---------------------------------------------------------------- operators */
typedef struct {
  int n, dense;
  double* d;      /* dense n*n */
  int *rp, *ci;   /* CSR */
  double* v;
} op_t;

static void op_free(op_t* o) {
  free(o->d);
  free(o->rp);
  free(o->ci);
  free(o->v);
  memset(o, 0, sizeof *o);
}

typedef struct { int r, c; double v; } trip_t;
static int trip_cmp(const void* a, const void* b) {
  const trip_t *x = a, *y = b;
  if (x->r != y->r) return x->r < y->r ? -1 : 1;
  if (x->c != y->c) return x->c < y->c ? -1 : 1;
  return 0;
}

/* SymmetricOperator::from_dense / from_triplets(Full) operator.hpp:45-104 */
static int op_from(const feast_operator_t* in, op_t* o) {
  memset(o, 0, sizeof *o);
  const int n = in->n;
  o->n = n;
  if (in->kind == FEAST_STORAGE_DENSE) {
    o->dense = 1;
    o->d = malloc(sizeof(double) * (size_t)n * n);
    memcpy(o->d, in->dense, sizeof(double) * (size_t)n * n);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i <= j; ++i)
        if (o->d[i + (size_t)j * n] != o->d[j + (size_t)i * n]) {
          g_code = FEAST_EINPUT;
          snprintf(g_err, sizeof g_err, "SymmetricOperator: matrix is not symmetric");
          return FEAST_EINPUT;
        }
    return 0;
  }
  size_t cap = 0, cnt = 0;
  trip_t* t = NULL;
#define PUSH(R, C, V)                                   \
  do {                                                  \
    if (cnt == cap) {                                   \
      cap = cap ? 2 * cap : 1024;                       \
      t = realloc(t, sizeof(trip_t) * cap);             \
    }                                                   \
    t[cnt].r = (R); t[cnt].c = (C); t[cnt].v = (V); ++cnt; \
  } while (0)
  if (in->kind == FEAST_STORAGE_CSR) {
    for (int i = 0; i < n; ++i)
      for (int k = in->row_ptr[i]; k < in->row_ptr[i + 1]; ++k) PUSH(i, in->col_idx[k], in->values[k]);
  } else {
    const int L = in->nblocks, b = in->bsize;
    for (int l = 0; l < L; ++l) {
      const double* d = in->diag + (size_t)l * b * b;
      for (int j = 0; j < b; ++j)
        for (int i = 0; i < b; ++i)
          if (d[i + (size_t)j * b] != 0.0) PUSH(l * b + i, l * b + j, d[i + (size_t)j * b]);
      if (l + 1 < L) {
        const double* c = in->lower + (size_t)l * b * b;
        for (int j = 0; j < b; ++j)
          for (int i = 0; i < b; ++i) {
            const double v = c[i + (size_t)j * b];
            if (v == 0.0) continue;
            PUSH((l + 1) * b + i, l * b + j, v);
            PUSH(l * b + j, (l + 1) * b + i, v);
          }
      }
    }
  }
#undef PUSH
  /* stable sort by (row, col): qsort is not stable, but duplicates are summed in input
     order only when coordinates repeat, which these inputs never do */
  qsort(t, cnt, sizeof(trip_t), trip_cmp);
  o->rp = calloc(n + 1, sizeof(int));
  o->ci = malloc(sizeof(int) * (cnt ? cnt : 1));
  o->v = malloc(sizeof(double) * (cnt ? cnt : 1));
  size_t k = 0, nz = 0;
  for (int i = 0; i < n; ++i) {
    o->rp[i] = (int)nz;
    while (k < cnt && t[k].r == i) {
      const int j = t[k].c;
      double v = 0.0;
      while (k < cnt && t[k].r == i && t[k].c == j) v += t[k++].v;
      o->ci[nz] = j;
      o->v[nz++] = v;
    }
  }
  o->rp[n] = (int)nz;
  free(t);
  return 0;
}

static int op_bandwidth(const op_t* o) {
  if (o->dense) return o->n > 0 ? o->n - 1 : 0;
  int bw = 0;
  for (int i = 0; i < o->n; ++i)
    for (int k = o->rp[i]; k < o->rp[i + 1]; ++k) {
      const int d = abs(i - o->ci[k]);
      if (d > bw) bw = d;
    }
  return bw;
}

/* SymmetricOperator::apply operator.hpp:132-158 (y zero-initialised) */
static void op_apply(const op_t* o, const double* x, int m, double* y) {
  const int n = o->n;
  memset(y, 0, sizeof(double) * (size_t)n * m);
  for (int c = 0; c < m; ++c) {
    const double* xc = x + (size_t)c * n;
    double* yc = y + (size_t)c * n;
    if (o->dense) {
      for (int j = 0; j < n; ++j) {
        const double xj = xc[j];
        if (xj == 0.0) continue;
        const double* aj = o->d + (size_t)j * n;
        for (int i = 0; i < n; ++i) yc[i] += aj[i] * xj;
      }
    } else {
      for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int k = o->rp[i]; k < o->rp[i + 1]; ++k) s += o->v[k] * xc[o->ci[k]];
        yc[i] = s;
      }
    }
  }
}

/* norm_one operator.hpp:195-212 */
static double op_norm_one(const op_t* o) {
  double best = 0.0;
  const int n = o->n;
  if (o->dense) {
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += fabs(o->d[i + (size_t)j * n]);
      if (s > best) best = s;
    }
  } else {
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int k = o->rp[i]; k < o->rp[i + 1]; ++k) s += fabs(o->v[k]);
      if (s > best) best = s;
    }
  }
  return best;
}

/* ---------------------------------------------------------------- shifted solves */
typedef struct {
  int banded, n, kl, ku, ldab;
  cplx* a;   /* dense LU (n*n) or band storage (ldab*n) */
  int* ipiv;
} shift_t;

static void shift_free(shift_t* s) {
  free(s->a);
  free(s->ipiv);
  memset(s, 0, sizeof *s);
}
#define BAND(s, i, j) ((s)->a[(size_t)((s)->kl + (s)->ku + (i) - (j)) + (size_t)(j) * (s)->ldab])

/* DirectSolver::prepare inner_solver.hpp:97-103 -> assemble (assemble.hpp) + factor (lu.hpp) */
static int shift_prepare(const op_t* A, const op_t* B, cplx z, int banded, shift_t* s) {
  const int n = A->n;
  memset(s, 0, sizeof *s);
  s->n = n;
  s->banded = banded;
  s->ipiv = malloc(sizeof(int) * n);
  if (!banded) {
    /* assemble_shifted_dense assemble.hpp:12-38 */
    cplx* m = calloc((size_t)n * n, sizeof(cplx));
    s->a = m;
    if (!A->dense) {
      for (int i = 0; i < n; ++i)
        for (int k = A->rp[i]; k < A->rp[i + 1]; ++k) m[i + (size_t)A->ci[k] * n] -= A->v[k];
    } else {
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) m[i + (size_t)j * n] -= A->d[i + (size_t)j * n];
    }
    if (!B->dense) {
      for (int i = 0; i < n; ++i)
        for (int k = B->rp[i]; k < B->rp[i + 1]; ++k) m[i + (size_t)B->ci[k] * n] += z * CMPLX(B->v[k], 0.0);
    } else {
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) m[i + (size_t)j * n] += z * CMPLX(B->d[i + (size_t)j * n], 0.0);
    }
    /* DenseLU lu.hpp:24-52 */
    for (int k = 0; k < n; ++k) {
      int p = k;
      double best = cabs(m[k + (size_t)k * n]);
      for (int i = k + 1; i < n; ++i) {
        const double v = cabs(m[i + (size_t)k * n]);
        if (v > best) { best = v; p = i; }
      }
      if (best == 0.0) {
        g_code = FEAST_ENUMERICAL;
        snprintf(g_err, sizeof g_err, "DenseLU: matrix is numerically singular");
        return FEAST_ENUMERICAL;
      }
      s->ipiv[k] = p;
      if (p != k)
        for (int j = 0; j < n; ++j) {
          const cplx t = m[k + (size_t)j * n];
          m[k + (size_t)j * n] = m[p + (size_t)j * n];
          m[p + (size_t)j * n] = t;
        }
      const cplx pivot = m[k + (size_t)k * n];
      for (int i = k + 1; i < n; ++i) m[i + (size_t)k * n] /= pivot;
      for (int j = k + 1; j < n; ++j) {
        const cplx ukj = m[k + (size_t)j * n];
        if (ukj == 0.0) continue;
        cplx* colj = m + (size_t)j * n;
        const cplx* colk = m + (size_t)k * n;
        for (int i = k + 1; i < n; ++i) colj[i] -= colk[i] * ukj;
      }
    }
    return 0;
  }
  /* assemble_shifted_banded assemble.hpp:41-57 */
  int bw = op_bandwidth(A), bwb = op_bandwidth(B);
  if (bwb > bw) bw = bwb;
  s->kl = s->ku = bw;
  s->ldab = 2 * bw + bw + 1;
  s->a = calloc((size_t)s->ldab * n, sizeof(cplx));
  for (int i = 0; i < n; ++i)
    for (int k = A->rp[i]; k < A->rp[i + 1]; ++k) BAND(s, i, A->ci[k]) -= A->v[k];
  for (int i = 0; i < n; ++i)
    for (int k = B->rp[i]; k < B->rp[i + 1]; ++k) BAND(s, i, B->ci[k]) += z * CMPLX(B->v[k], 0.0);
  /* BandedLU lu.hpp:127-158 */
  const int kl = s->kl, kw = s->kl + s->ku;
  for (int k = 0; k < n; ++k) {
    const int last_row = n - 1 < k + kl ? n - 1 : k + kl;
    int p = k;
    double best = cabs(BAND(s, k, k));
    for (int i = k + 1; i <= last_row; ++i) {
      const double v = cabs(BAND(s, i, k));
      if (v > best) { best = v; p = i; }
    }
    if (best == 0.0) {
      g_code = FEAST_ENUMERICAL;
      snprintf(g_err, sizeof g_err, "BandedLU: matrix is numerically singular");
      return FEAST_ENUMERICAL;
    }
    s->ipiv[k] = p;
    const int last_col = n - 1 < k + kw ? n - 1 : k + kw;
    if (p != k)
      for (int j = k; j <= last_col; ++j) {
        const cplx t = BAND(s, k, j);
        BAND(s, k, j) = BAND(s, p, j);
        BAND(s, p, j) = t;
      }
    const cplx pivot = BAND(s, k, k);
    for (int i = k + 1; i <= last_row; ++i) {
      const cplx l = BAND(s, i, k) / pivot;
      BAND(s, i, k) = l;
      if (l == 0.0) continue;
      for (int j = k + 1; j <= last_col; ++j) BAND(s, i, j) -= l * BAND(s, k, j);
    }
  }
  return 0;
}

/* DenseLU::solve_in_place lu.hpp:56-95 / BandedLU::solve_in_place lu.hpp:162-201 */
static void shift_solve(const shift_t* s, cplx* rhs, int m, int mode) {
  const int n = s->n;
  for (int c = 0; c < m; ++c) {
    cplx* b = rhs + (size_t)c * n;
    if (!s->banded) {
      const cplx* lu = s->a;
      if (mode == 0) {
        for (int k = 0; k < n; ++k)
          if (s->ipiv[k] != k) { const cplx t = b[k]; b[k] = b[s->ipiv[k]]; b[s->ipiv[k]] = t; }
        for (int k = 0; k < n; ++k) {
          const cplx bk = b[k];
          if (bk == 0.0) continue;
          const cplx* colk = lu + (size_t)k * n;
          for (int i = k + 1; i < n; ++i) b[i] -= colk[i] * bk;
        }
        for (int k = n - 1; k >= 0; --k) {
          b[k] /= lu[k + (size_t)k * n];
          const cplx bk = b[k];
          if (bk == 0.0) continue;
          const cplx* colk = lu + (size_t)k * n;
          for (int i = 0; i < k; ++i) b[i] -= colk[i] * bk;
        }
      } else {
        for (int k = 0; k < n; ++k) {
          cplx sum = b[k];
          const cplx* colk = lu + (size_t)k * n;
          for (int i = 0; i < k; ++i) sum -= conj(colk[i]) * b[i];
          b[k] = sum / conj(colk[k]);
        }
        for (int k = n - 1; k >= 0; --k) {
          cplx sum = b[k];
          const cplx* colk = lu + (size_t)k * n;
          for (int i = k + 1; i < n; ++i) sum -= conj(colk[i]) * b[i];
          b[k] = sum;
        }
        for (int k = n - 1; k >= 0; --k)
          if (s->ipiv[k] != k) { const cplx t = b[k]; b[k] = b[s->ipiv[k]]; b[s->ipiv[k]] = t; }
      }
    } else {
      const int kl = s->kl, kw = s->kl + s->ku;
      if (mode == 0) {
        for (int k = 0; k < n; ++k) {
          if (s->ipiv[k] != k) { const cplx t = b[k]; b[k] = b[s->ipiv[k]]; b[s->ipiv[k]] = t; }
          const cplx bk = b[k];
          if (bk == 0.0) continue;
          const int last_row = n - 1 < k + kl ? n - 1 : k + kl;
          for (int i = k + 1; i <= last_row; ++i) b[i] -= BAND(s, i, k) * bk;
        }
        for (int k = n - 1; k >= 0; --k) {
          cplx sum = b[k];
          const int last_col = n - 1 < k + kw ? n - 1 : k + kw;
          for (int j = k + 1; j <= last_col; ++j) sum -= BAND(s, k, j) * b[j];
          b[k] = sum / BAND(s, k, k);
        }
      } else {
        for (int k = 0; k < n; ++k) {
          cplx sum = b[k];
          const int first = k - kw > 0 ? k - kw : 0;
          for (int j = first; j < k; ++j) sum -= conj(BAND(s, j, k)) * b[j];
          b[k] = sum / conj(BAND(s, k, k));
        }
        for (int k = n - 1; k >= 0; --k) {
          cplx sum = b[k];
          const int last_row = n - 1 < k + kl ? n - 1 : k + kl;
          for (int i = k + 1; i <= last_row; ++i) sum -= conj(BAND(s, i, k)) * b[i];
          b[k] = sum;
          if (s->ipiv[k] != k) { const cplx t = b[k]; b[k] = b[s->ipiv[k]]; b[s->ipiv[k]] = t; }
        }
      }
    }
  }
}

/* DirectSolver Auto policy inner_solver.hpp:84-92 */
static int use_banded(const op_t* A, const op_t* B) {
  if (A->dense || B->dense) return 0;
  int bw = op_bandwidth(A), bwb = op_bandwidth(B);
  if (bwb > bw) bw = bwb;
  return (3 * bw + 1) * 2 <= A->n;
}

/* ---------------------------------------------------------------- contour accumulation */
typedef struct {
  const contour_t* c;
  const op_t *A, *B;
  shift_t* sys;
  const double* y;
  int n, m, threads, wid, banded, rc;
  double* terms;  /* ne * n*m */
  int prepare;
  const double* yc; /* hermitian: complex block (interleaved n*m) */
  double* tc;       /* hermitian: complex terms ne * 2n*m */
  int herm;
} work_t;

static void* point_worker(void* arg) {
  work_t* w = arg;
  const int n = w->n, m = w->m;
  for (int e = w->wid; e < w->c->ne; e += w->threads) {
    if (w->prepare) {
      int rc = shift_prepare(w->A, w->B, w->c->z[e], w->banded, &w->sys[e]);
      if (rc && !w->rc) w->rc = rc;
      continue;
    }
    if (w->herm) {
      /* accumulate_subspace_hermitian core.hpp:198-210: the Normal and the ConjTranspose solve
         on the same factorisation, term = c1 s1 + c2 s2 with c1,2 = (w r / 4) e^{+-i theta} */
      const size_t nm = (size_t)n * m;
      cplx* s1 = malloc(sizeof(cplx) * nm);
      cplx* s2 = malloc(sizeof(cplx) * nm);
      for (size_t k = 0; k < nm; ++k) s1[k] = s2[k] = CMPLX(w->yc[2 * k], w->yc[2 * k + 1]);
      shift_solve(&w->sys[e], s1, m, 0);
      shift_solve(&w->sys[e], s2, m, 1);
      const double pref = 0.25 * w->c->weight[e] * w->c->radius;
      const cplx c1 = CMPLX(pref * cos(w->c->theta[e]), pref * sin(w->c->theta[e]));
      const cplx c2 = CMPLX(pref * cos(w->c->theta[e]), -pref * sin(w->c->theta[e]));
      double* term = w->tc + (size_t)e * 2 * nm;
      for (size_t k = 0; k < nm; ++k) {
        const cplx t = c1 * s1[k] + c2 * s2[k];
        term[2 * k] = creal(t);
        term[2 * k + 1] = cimag(t);
      }
      free(s1);
      free(s2);
      continue;
    }
    /* accumulate_subspace_real core.hpp:170-180 */
    cplx* rhs = malloc(sizeof(cplx) * (size_t)n * m);
    for (size_t k = 0; k < (size_t)n * m; ++k) rhs[k] = CMPLX(w->y[k], 0.0);
    shift_solve(&w->sys[e], rhs, m, 0);
    const double f = 0.5 * w->c->weight[e] * w->c->radius;
    const cplx coeff = CMPLX(f * cos(w->c->theta[e]), f * sin(w->c->theta[e]));
    double* term = w->terms + (size_t)e * n * m;
    for (size_t k = 0; k < (size_t)n * m; ++k) term[k] = creal(coeff * rhs[k]);
    free(rhs);
  }
  return NULL;
}

/* parallel_points core.hpp:131-155 (static striping) */
static int run_points(work_t* proto, int threads) {
  const int workers = threads < proto->c->ne ? (threads > 0 ? threads : 1) : proto->c->ne;
  work_t w[64];
  pthread_t th[64];
  for (int i = 0; i < workers; ++i) {
    w[i] = *proto;
    w[i].threads = workers;
    w[i].wid = i;
    w[i].rc = 0;
  }
  if (workers == 1) {
    point_worker(&w[0]);
  } else {
    for (int i = 0; i < workers; ++i) pthread_create(&th[i], NULL, point_worker, &w[i]);
    for (int i = 0; i < workers; ++i) pthread_join(th[i], NULL);
  }
  for (int i = 0; i < workers; ++i)
    if (w[i].rc) return w[i].rc;
  return 0;
}

static int prepare_all(const op_t* A, const op_t* B, const contour_t* c, int threads, shift_t* sys) {
  work_t p = {0};
  p.c = c; p.A = A; p.B = B; p.sys = sys; p.n = A->n; p.prepare = 1; p.banded = use_banded(A, B);
  return run_points(&p, threads);
}

static void accumulate(const op_t* A, const contour_t* c, shift_t* sys, const double* y, int m, int threads,
                       double* q) {
  const int n = A->n;
  work_t p = {0};
  p.c = c; p.A = A; p.sys = sys; p.y = y; p.n = n; p.m = m;
  p.terms = malloc(sizeof(double) * (size_t)c->ne * n * m);
  run_points(&p, threads);
  memset(q, 0, sizeof(double) * (size_t)n * m);
  for (int e = 0; e < c->ne; ++e)
    for (size_t k = 0; k < (size_t)n * m; ++k) q[k] -= p.terms[(size_t)e * n * m + k];
  free(p.terms);
}

/* accumulate_subspace_hermitian core.hpp:190-215 (ascending e reduction of the terms) */
static void accumulate_herm(const op_t* A, const contour_t* c, shift_t* sys, const double* yc, int m, int threads,
                            double* qc) {
  const int n = A->n;
  const size_t nm2 = 2 * (size_t)n * m;
  work_t p = {0};
  p.c = c; p.A = A; p.sys = sys; p.yc = yc; p.n = n; p.m = m; p.herm = 1;
  p.tc = malloc(sizeof(double) * (size_t)c->ne * nm2);
  run_points(&p, threads);
  memset(qc, 0, sizeof(double) * nm2);
  for (int e = 0; e < c->ne; ++e)
    for (size_t k = 0; k < nm2; k += 2) {  /* complex subtraction, component-wise */
      qc[k] -= p.tc[(size_t)e * nm2 + k];
      qc[k + 1] -= p.tc[(size_t)e * nm2 + k + 1];
    }
  free(p.tc);
}

/* ---------------------------------------------------------------- reduced problem */
/* hermitian_part dense.hpp:127-134 */
static void herm(const double* mi, int n, double* h) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) h[i + (size_t)j * n] = (mi[i + (size_t)j * n] + mi[j + (size_t)i * n]) * 0.5;
}
/* adjoint_matmul dense.hpp:76-90: C = A^T B (A rows x ac, B rows x bc) */
static void adj_matmul(const double* a, int rows, int ac, const double* b, int bc, double* c) {
  for (int j = 0; j < bc; ++j)
    for (int i = 0; i < ac; ++i) {
      double s = 0.0;
      for (int k = 0; k < rows; ++k) s += a[k + (size_t)i * rows] * b[k + (size_t)j * rows];
      c[i + (size_t)j * ac] = s;
    }
}
/* matmul dense.hpp:59-73: C = A B (A rows x inner, B inner x bc) */
static void matmul(const double* a, int rows, int inner, const double* b, int bc, double* c) {
  memset(c, 0, sizeof(double) * (size_t)rows * bc);
  for (int j = 0; j < bc; ++j) {
    double* cj = c + (size_t)j * rows;
    for (int k = 0; k < inner; ++k) {
      const double bkj = b[k + (size_t)j * inner];
      if (bkj == 0.0) continue;
      const double* ak = a + (size_t)k * rows;
      for (int i = 0; i < rows; ++i) cj[i] += ak[i] * bkj;
    }
  }
}
static void transpose(const double* a, int r, int c, double* t) {
  for (int j = 0; j < c; ++j)
    for (int i = 0; i < r; ++i) t[j + (size_t)i * c] = a[i + (size_t)j * r];
}

/* cholesky eigh.hpp:20-43; returns 1 on NotPositiveDefinite */
static int cholesky(const double* m, int n, double rel, double* l) {
  double md = 0.0;
  for (int i = 0; i < n; ++i) if (m[i + (size_t)i * n] > md) md = m[i + (size_t)i * n];
  const double floor_ = rel * md;
  memset(l, 0, sizeof(double) * (size_t)n * n);
  for (int j = 0; j < n; ++j) {
    double d = m[j + (size_t)j * n];
    for (int k = 0; k < j; ++k) { const double v = l[j + (size_t)k * n]; d -= v * v; }
    if (d <= 0.0 || d <= floor_) return 1;
    const double ljj = sqrt(d);
    l[j + (size_t)j * n] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = m[i + (size_t)j * n];
      for (int k = 0; k < j; ++k) s -= l[i + (size_t)k * n] * l[j + (size_t)k * n];
      l[i + (size_t)j * n] = s / ljj;
    }
  }
  return 0;
}
/* solve_lower_in_place eigh.hpp:46-58 */
static void solve_lower(const double* l, int n, double* x, int m) {
  for (int c = 0; c < m; ++c) {
    double* b = x + (size_t)c * n;
    for (int k = 0; k < n; ++k) {
      b[k] /= l[k + (size_t)k * n];
      const double bk = b[k];
      for (int i = k + 1; i < n; ++i) b[i] -= l[i + (size_t)k * n] * bk;
    }
  }
}
/* solve_lower_adjoint_in_place eigh.hpp:61-73 */
static void solve_lower_adj(const double* l, int n, double* x, int m) {
  for (int c = 0; c < m; ++c) {
    double* b = x + (size_t)c * n;
    for (int k = n - 1; k >= 0; --k) {
      double s = b[k];
      for (int i = k + 1; i < n; ++i) s -= l[i + (size_t)k * n] * b[i];
      b[k] = s / l[k + (size_t)k * n];
    }
  }
}

typedef struct { double v; int i; } kv_t;
static int kv_cmp(const void* a, const void* b) {  /* stable via index tiebreak */
  const kv_t *x = a, *y = b;
  if (x->v < y->v) return -1;
  if (y->v < x->v) return 1;
  return x->i < y->i ? -1 : (x->i > y->i);
}

/* jacobi_eigh eigh.hpp:84-163 (real case): evals ascending, vecs n*n */
static void jacobi_eigh(const double* m_in, int n, double* evals, double* vecs) {
  double* w = malloc(sizeof(double) * (size_t)n * n);
  double* v = calloc((size_t)n * n, sizeof(double));
  herm(m_in, n, w);
  for (int i = 0; i < n; ++i) v[i + (size_t)i * n] = 1.0;
  double fro = 0.0;
  for (size_t k = 0; k < (size_t)n * n; ++k) fro += w[k] * w[k];
  fro = sqrt(fro);
  const double eps = DBL_EPSILON;
  const double scale = fro > DBL_MIN ? fro : DBL_MIN;
#define W(i, j) w[(i) + (size_t)(j) * n]
#define V(i, j) v[(i) + (size_t)(j) * n]
  for (int sweep = 0; sweep < 50; ++sweep) {
    double off = 0.0;
    for (int q = 1; q < n; ++q)
      for (int p = 0; p < q; ++p) off += W(p, q) * W(p, q);
    off = sqrt(off);
    if (off <= n * eps * scale) break;
    const double thresh = sweep < 3 ? 0.2 * off / ((double)n * n) : 0.0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = W(p, q);
        const double a = fabs(apq);
        const double app = W(p, p), aqq = W(q, q);
        if (a <= thresh) continue;
        if (sweep > 3 && a <= eps * 0.5 * (fabs(app) + fabs(aqq))) {
          W(p, q) = 0.0;
          W(q, p) = 0.0;
          continue;
        }
        if (a == 0.0) continue;
        const double ph = apq * (1.0 / a);
        const double phc = ph;
        const double tau = (aqq - app) / (2.0 * a);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + hypot(1.0, tau));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = t * c;
        for (int i = 0; i < n; ++i) {
          const double wip = W(i, p), wiq = W(i, q);
          W(i, p) = wip * c - wiq * (phc * s);
          W(i, q) = wip * s + wiq * (phc * c);
        }
        for (int j = 0; j < n; ++j) {
          const double wpj = W(p, j), wqj = W(q, j);
          W(p, j) = wpj * c - wqj * (ph * s);
          W(q, j) = wpj * s + wqj * (ph * c);
        }
        W(p, q) = 0.0;
        W(q, p) = 0.0;
        for (int i = 0; i < n; ++i) {
          const double vip = V(i, p), viq = V(i, q);
          V(i, p) = vip * c - viq * (phc * s);
          V(i, q) = vip * s + viq * (phc * c);
        }
      }
  }
  kv_t* kv = malloc(sizeof(kv_t) * n);
  for (int i = 0; i < n; ++i) { kv[i].v = W(i, i); kv[i].i = i; }
  qsort(kv, n, sizeof(kv_t), kv_cmp);
  for (int i = 0; i < n; ++i) {
    evals[i] = kv[i].v;
    memcpy(vecs + (size_t)i * n, v + (size_t)kv[i].i * n, sizeof(double) * n);
  }
#undef W
#undef V
  free(kv);
  free(w);
  free(v);
}

/* reduced_gevp eigh.hpp:178-225; phi is m*m (first *mo columns valid) */
static int reduced_gevp(const double* aq, const double* bq, int m, double* evals, double* phi, int* mo,
                        int* truncated) {
  if (m == 0) { *mo = 0; *truncated = 0; return 0; }
  const size_t mm = (size_t)m * m;
  double* l = malloc(sizeof(double) * mm);
  double* t1 = malloc(sizeof(double) * mm);
  double* t2 = malloc(sizeof(double) * mm);
  int rc = 0;
  if (!cholesky(bq, m, 1e-13, l)) {
    memcpy(t1, aq, sizeof(double) * mm);
    solve_lower(l, m, t1, m);
    transpose(t1, m, m, t2);
    solve_lower(l, m, t2, m);
    transpose(t2, m, m, t1);
    jacobi_eigh(t1, m, evals, phi);
    solve_lower_adj(l, m, phi, m);
    *mo = m;
    *truncated = 0;
    goto done;
  }
  {
    double* bev = malloc(sizeof(double) * m);
    double* bv = malloc(sizeof(double) * mm);
    jacobi_eigh(bq, m, bev, bv);
    const double dmax = bev[m - 1];
    if (!(dmax > 0.0)) {
      free(bev); free(bv);
      g_code = FEAST_EBREAKDOWN;
      snprintf(g_err, sizeof g_err, "reduced_gevp: projected mass matrix has no positive modes");
      rc = FEAST_EBREAKDOWN;
      goto done;
    }
    int k = 0;
    int* keep = malloc(sizeof(int) * m);
    for (int i = 0; i < m; ++i) if (bev[i] > 1e-14 * dmax) keep[k++] = i;
    if (!k) {
      free(bev); free(bv); free(keep);
      g_code = FEAST_EBREAKDOWN;
      snprintf(g_err, sizeof g_err, "reduced_gevp: projected mass matrix has no usable modes");
      rc = FEAST_EBREAKDOWN;
      goto done;
    }
    double* s = malloc(sizeof(double) * (size_t)m * k);
    for (int j = 0; j < k; ++j) {
      const double inv = 1.0 / sqrt(bev[keep[j]]);
      for (int i = 0; i < m; ++i) s[i + (size_t)j * m] = bv[i + (size_t)keep[j] * m] * inv;
    }
    double* as = malloc(sizeof(double) * (size_t)m * k);
    double* ared = malloc(sizeof(double) * (size_t)k * k);
    double* ah = malloc(sizeof(double) * (size_t)k * k);
    double* wv = malloc(sizeof(double) * (size_t)k * k);
    matmul(aq, m, m, s, k, as);
    adj_matmul(s, m, k, as, k, ared);
    herm(ared, k, ah);
    jacobi_eigh(ah, k, evals, wv);
    matmul(s, m, k, wv, k, phi);
    *mo = k;
    *truncated = 1;
    free(bev); free(bv); free(keep); free(s); free(as); free(ared); free(ah); free(wv);
  }
done:
  free(l); free(t1); free(t2);
  return rc;
}

/* rayleigh_ritz core.hpp:228-240 */
static int rayleigh_ritz(const op_t* A, const op_t* B, const double* q, int m, double* evals, double* x,
                         int* mo, int* truncated) {
  const int n = A->n;
  const size_t mm = (size_t)m * m;
  double* w = malloc(sizeof(double) * (size_t)n * m);
  double* t = malloc(sizeof(double) * mm);
  double* aq = malloc(sizeof(double) * mm);
  double* bq = malloc(sizeof(double) * mm);
  double* phi = malloc(sizeof(double) * mm);
  op_apply(A, q, m, w);
  adj_matmul(q, n, m, w, m, t);
  herm(t, m, aq);
  op_apply(B, q, m, w);
  adj_matmul(q, n, m, w, m, t);
  herm(t, m, bq);
  int rc = reduced_gevp(aq, bq, m, evals, phi, mo, truncated);
  if (!rc) matmul(q, n, m, phi, *mo, x);
  free(w); free(t); free(aq); free(bq); free(phi);
  return rc;
}

/* residual_norms residual.hpp:29-68 */
static void residual_norms(const op_t* A, const op_t* B, const double* lam, int m, const double* x,
                           double* res, int32_t* absonly, double* maxres) {
  const int n = A->n;
  *maxres = 0.0;
  if (!m) return;
  const double an = op_norm_one(A);
  double* ax = malloc(sizeof(double) * (size_t)n * m);
  double* bx = malloc(sizeof(double) * (size_t)n * m);
  op_apply(A, x, m, ax);
  op_apply(B, x, m, bx);
  for (int j = 0; j < m; ++j) {
    double num = 0.0, den = 0.0, xn = 0.0;
    for (int i = 0; i < n; ++i) {
      num += fabs(ax[i + (size_t)j * n] - lam[j] * bx[i + (size_t)j * n]);
      den += fabs(ax[i + (size_t)j * n]);
      xn += fabs(x[i + (size_t)j * n]);
    }
    const double floor_ = 4.0 * n * DBL_EPSILON * an * xn;
    if (den <= (1e-300 > floor_ ? 1e-300 : floor_)) {
      res[j] = num;
      absonly[j] = 1;
    } else {
      res[j] = num / den;
      absonly[j] = 0;
    }
    if (res[j] > *maxres) *maxres = res[j];
  }
  free(ax);
  free(bx);
}

/* ================================================================ exports */
int ref_gauss_legendre(int n, double* nodes, double* weights) { return gauss_legendre(n, nodes, weights); }

int ref_build_contour(double emin, double emax, int ne, double* node, double* weight, double* theta, double* z,
                      double* radius) {
  contour_t c;
  int rc = build_contour(emin, emax, ne, &c);
  if (rc) return rc;
  for (int e = 0; e < ne; ++e) {
    node[e] = c.node[e];
    weight[e] = c.weight[e];
    theta[e] = c.theta[e];
    z[2 * e] = creal(c.z[e]);
    z[2 * e + 1] = cimag(c.z[e]);
  }
  *radius = c.radius;
  return 0;
}

int ref_random_block(int n, int m, uint64_t seed, double* out) {
  random_block(n, m, seed, out);
  return 0;
}

/* oracle::scalar_filter oracle.cpp:200-208 */
double ref_scalar_filter(double lambda, double emin, double emax, int ne) {
  contour_t c;
  if (build_contour(emin, emax, ne, &c)) return NAN;
  double f = 0.0;
  for (int e = 0; e < ne; ++e) {
    const cplx reith = CMPLX(cos(c.theta[e]), sin(c.theta[e]));
    f -= 0.5 * c.weight[e] * creal(c.radius * reith / (c.z[e] - lambda));
  }
  return f;
}

int ref_reduced_gevp(int m, const double* aq, const double* bq, double* evals, double* phi, int* m_out,
                     int* truncated) {
  return reduced_gevp(aq, bq, m, evals, phi, m_out, truncated);
}

int ref_accumulate_real(const feast_operator_t* a, const feast_operator_t* b, double emin, double emax, int ne,
                        const double* y, int m, double* q, int threads) {
  op_t A, B;
  contour_t c;
  shift_t* sys = NULL;
  int rc;
  memset(&A, 0, sizeof A);
  memset(&B, 0, sizeof B);
  if ((rc = op_from(a, &A)) || (rc = op_from(b, &B)) || (rc = build_contour(emin, emax, ne, &c))) goto out;
  sys = calloc(ne, sizeof(shift_t));
  if ((rc = prepare_all(&A, &B, &c, threads, sys))) goto out;
  accumulate(&A, &c, sys, y, m, threads, q);
out:
  if (sys) { for (int e = 0; e < ne; ++e) shift_free(&sys[e]); free(sys); }
  op_free(&A);
  op_free(&B);
  return rc;
}

int ref_accumulate_hermitian(const feast_operator_t* a, const feast_operator_t* b, double emin, double emax,
                             int ne, const double* y, int m, double* q, int threads) {
  op_t A, B;
  contour_t c;
  shift_t* sys = NULL;
  int rc;
  memset(&A, 0, sizeof A);
  memset(&B, 0, sizeof B);
  if ((rc = op_from(a, &A)) || (rc = op_from(b, &B)) || (rc = build_contour(emin, emax, ne, &c))) goto out;
  sys = calloc(ne, sizeof(shift_t));
  if ((rc = prepare_all(&A, &B, &c, threads, sys))) goto out;
  accumulate_herm(&A, &c, sys, y, m, threads, q);
out:
  if (sys) { for (int e = 0; e < ne; ++e) shift_free(&sys[e]); free(sys); }
  op_free(&A);
  op_free(&B);
  return rc;
}

int ref_shift_solve(const feast_operator_t* a, const feast_operator_t* b, double zr, double zi, double* rhs,
                    int m, int mode) {
  op_t A, B;
  shift_t s;
  int rc;
  memset(&A, 0, sizeof A);
  memset(&B, 0, sizeof B);
  memset(&s, 0, sizeof s);
  if ((rc = op_from(a, &A)) || (rc = op_from(b, &B))) goto out;
  if ((rc = shift_prepare(&A, &B, CMPLX(zr, zi), use_banded(&A, &B), &s))) goto out;
  shift_solve(&s, (cplx*)rhs, m, mode);
out:
  shift_free(&s);
  op_free(&A);
  op_free(&B);
  return rc;
}

int ref_rayleigh_ritz(const feast_operator_t* a, const feast_operator_t* b, const double* q, int m,
                      double* evals, double* x, int* m_out, int* truncated) {
  op_t A, B;
  int rc;
  memset(&A, 0, sizeof A);
  memset(&B, 0, sizeof B);
  if (!(rc = op_from(a, &A)) && !(rc = op_from(b, &B))) rc = rayleigh_ritz(&A, &B, q, m, evals, x, m_out, truncated);
  op_free(&A);
  op_free(&B);
  return rc;
}

int ref_residual_norms(const feast_operator_t* a, const feast_operator_t* b, int m, const double* lambdas,
                       const double* x, double* res, int32_t* absonly, double* maxres) {
  op_t A, B;
  int rc;
  memset(&A, 0, sizeof A);
  memset(&B, 0, sizeof B);
  if (!(rc = op_from(a, &A)) && !(rc = op_from(b, &B))) residual_norms(&A, &B, lambdas, m, x, res, absonly, maxres);
  op_free(&A);
  op_free(&B);
  return rc;
}

/* independent dense GEVP for small n (oracle.cpp:162-193 role): Cholesky + Jacobi */
int ref_reference_gevp(const feast_operator_t* a, const feast_operator_t* b, double* evals, double* evecs) {
  op_t A, B;
  int rc, mo, tr;
  memset(&A, 0, sizeof A);
  memset(&B, 0, sizeof B);
  if ((rc = op_from(a, &A)) || (rc = op_from(b, &B))) goto out;
  {
    const int n = A.n;
    double* ad = calloc((size_t)n * n, sizeof(double));
    double* bd = calloc((size_t)n * n, sizeof(double));
    double* e = evecs ? evecs : malloc(sizeof(double) * (size_t)n * n);
    double* x = malloc(sizeof(double) * (size_t)n * n);
    for (int j = 0; j < n; ++j) x[j] = 0;
    for (int c = 0; c < n; ++c) {
      for (int i = 0; i < n; ++i) x[i] = (i == c);
      op_apply(&A, x, 1, ad + (size_t)c * n);
      op_apply(&B, x, 1, bd + (size_t)c * n);
    }
    rc = reduced_gevp(ad, bd, n, evals, e, &mo, &tr);
    if (!evecs) free(e);
    free(ad); free(bd); free(x);
  }
out:
  op_free(&A);
  op_free(&B);
  return rc;
}

static double now_s(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + 1e-9 * t.tv_nsec;
}

int ref_bench_passes(const feast_operator_t* a, const feast_operator_t* b, double emin, double emax, int m0,
                     int ne, uint64_t seed, int threads, int passes, double* out) {
  op_t A, B;
  contour_t c;
  shift_t* sys = NULL;
  int rc;
  memset(&A, 0, sizeof A);
  memset(&B, 0, sizeof B);
  if ((rc = op_from(a, &A)) || (rc = op_from(b, &B)) || (rc = build_contour(emin, emax, ne, &c))) goto out;
  {
    const int n = A.n;
    sys = calloc(ne, sizeof(shift_t));
    double t0 = now_s();
    if ((rc = prepare_all(&A, &B, &c, threads, sys))) goto out;
    out[0] = now_s() - t0;
    out[1] = out[2] = out[3] = 0.0;
    int m = m0;
    double* y = malloc(sizeof(double) * (size_t)n * m0);
    double* q = malloc(sizeof(double) * (size_t)n * m0);
    double* x = malloc(sizeof(double) * (size_t)n * m0);
    double* ev = malloc(sizeof(double) * m0);
    random_block(n, m0, seed, y);
    for (int p = 0; p < passes && !rc; ++p) {
      t0 = now_s();
      accumulate(&A, &c, sys, y, m, threads, q);
      out[1] += now_s() - t0;
      t0 = now_s();
      int mo, tr;
      rc = rayleigh_ritz(&A, &B, q, m, ev, x, &mo, &tr);
      out[2] += now_s() - t0;
      if (rc) break;
      int cnt = 0;
      for (int i = 0; i < mo; ++i) cnt += (emin <= ev[i] && ev[i] <= emax);
      out[3] = cnt;
      m = mo;
      op_apply(&B, x, m, y);
    }
    free(y); free(q); free(x); free(ev);
  }
out:
  if (sys) { for (int e = 0; e < ne; ++e) shift_free(&sys[e]); free(sys); }
  op_free(&A);
  op_free(&B);
  return rc;
}

/* feast_solve core.hpp:264-391 */
int ref_feast_solve(const feast_operator_t* a, const feast_operator_t* b, double emin, double emax,
                    const feast_config_t* cfg, const double* initial_y, int y_cols, feast_result_t* out) {
  op_t A, B;
  contour_t c;
  shift_t* sys = NULL;
  double *y = NULL, *q = NULL, *x = NULL, *ev = NULL, *hist = NULL;
  int* cnts = NULL;
  int rc = 0;
  const double t_start = now_s();
  memset(&A, 0, sizeof A);
  memset(&B, 0, sizeof B);
  if ((rc = op_from(a, &A)) || (rc = op_from(b, &B))) goto out;
  const int n = A.n, m0 = cfg->m0;
  if (a->n != b->n) { g_code = 4; snprintf(g_err, sizeof g_err, "feast_solve: operator dimensions differ"); rc = 4; goto out; }
  if (m0 < 1 || m0 > n) { snprintf(g_err, sizeof g_err, "feast_solve: m0 must be in [1, n]"); rc = 4; goto out; }
  if (cfg->max_loops < 1) { snprintf(g_err, sizeof g_err, "feast_solve: max_loops must be positive"); rc = 4; goto out; }
  if (!(cfg->trace_tol > 0.0)) { snprintf(g_err, sizeof g_err, "feast_solve: trace_tol must be positive"); rc = 4; goto out; }
  if (cfg->threads < 1) { snprintf(g_err, sizeof g_err, "feast_solve: threads must be positive"); rc = 4; goto out; }
  if (initial_y && (y_cols < 1 || y_cols > m0)) { snprintf(g_err, sizeof g_err, "feast_solve: initial block shape mismatch"); rc = 4; goto out; }
  if ((rc = build_contour(emin, emax, cfg->n_e, &c))) goto out;
  {
    const int ne = cfg->n_e;
    const double effective_tol = cfg->trace_tol;
    y = malloc(sizeof(double) * (size_t)n * m0);
    q = malloc(sizeof(double) * (size_t)n * m0);
    x = malloc(sizeof(double) * (size_t)n * m0);
    ev = malloc(sizeof(double) * m0);
    hist = malloc(sizeof(double) * (cfg->max_loops + 1));
    cnts = malloc(sizeof(int) * (cfg->max_loops + 1));
    int m = initial_y ? y_cols : m0;
    if (initial_y) memcpy(y, initial_y, sizeof(double) * (size_t)n * m);
    else random_block(n, m0, cfg->seed, y);
    sys = calloc(ne, sizeof(shift_t));
    int have = 0;
    double prev_trace = 0.0;
    int prev_count = -1;
    memset(&out->m, 0, sizeof(feast_result_t) - offsetof(feast_result_t, m));
    for (int pass = 0; pass <= cfg->max_loops; ++pass) {
      if (cfg->low_memory && have) { for (int e = 0; e < ne; ++e) shift_free(&sys[e]); have = 0; }
      if (!have) {
        const double t0 = now_s();
        if ((rc = prepare_all(&A, &B, &c, cfg->threads, sys))) goto out;
        have = 1;
        out->factorize_s += now_s() - t0;
      }
      double t0 = now_s();
      accumulate(&A, &c, sys, y, m, cfg->threads, q);
      out->solve_s += now_s() - t0;
      t0 = now_s();
      int mo = 0, tr = 0;
      rc = rayleigh_ritz(&A, &B, q, m, ev, x, &mo, &tr);
      out->reduce_s += now_s() - t0;
      if (rc == FEAST_EBREAKDOWN) {
        rc = 0;
        out->status = FEAST_STATUS_BREAKDOWN;
        out->loops_used = pass;
        if (out->trace_history) memcpy(out->trace_history, hist, sizeof(double) * pass);
        if (out->in_interval_counts) memcpy(out->in_interval_counts, cnts, sizeof(int) * pass);
        out->total_s = now_s() - t_start;
        goto out;
      }
      if (rc) goto out;
      double trc = 0.0;
      int cnt = 0;
      for (int i = 0; i < mo; ++i)
        if (emin <= ev[i] && ev[i] <= emax) { trc += ev[i]; ++cnt; }
      hist[pass] = trc;
      cnts[pass] = cnt;
      int status = -1;
      if (cnt == m0) status = FEAST_STATUS_SATURATED;
      else if (pass >= 1) {
        if (cnt == 0 && prev_count == 0) status = FEAST_STATUS_NO_EIGENVALUES;
        else {
          const double w = emax - emin;
          const double denom = fabs(trc) > w ? fabs(trc) : w;
          if (cnt == prev_count && fabs(trc - prev_trace) <= effective_tol * denom) status = FEAST_STATUS_CONVERGED;
        }
      }
      if (status < 0 && pass == cfg->max_loops) status = FEAST_STATUS_MAX_LOOPS;
      if (status >= 0) {
        /* finalize core.hpp:316-332 */
        out->status = status;
        out->loops_used = pass;
        int k = 0;
        double* lam = malloc(sizeof(double) * mo);
        double* vecs = malloc(sizeof(double) * (size_t)n * (mo ? mo : 1));
        for (int i = 0; i < mo; ++i)
          if (emin <= ev[i] && ev[i] <= emax) {
            lam[k] = ev[i];
            memcpy(vecs + (size_t)k * n, x + (size_t)i * n, sizeof(double) * n);
            ++k;
          }
        out->m = k;
        out->subspace_cols = mo;
        if (out->eigenvalues) memcpy(out->eigenvalues, lam, sizeof(double) * k);
        if (out->eigenvectors) memcpy(out->eigenvectors, vecs, sizeof(double) * (size_t)n * k);
        if (out->subspace) memcpy(out->subspace, x, sizeof(double) * (size_t)n * mo);
        double* res = malloc(sizeof(double) * (k ? k : 1));
        int32_t* ab = malloc(sizeof(int32_t) * (k ? k : 1));
        residual_norms(&A, &B, lam, k, vecs, res, ab, &out->max_residual);
        if (out->residuals) memcpy(out->residuals, res, sizeof(double) * k);
        if (out->residual_absolute_only) memcpy(out->residual_absolute_only, ab, sizeof(int32_t) * k);
        if (out->trace_history) memcpy(out->trace_history, hist, sizeof(double) * (pass + 1));
        if (out->in_interval_counts) memcpy(out->in_interval_counts, cnts, sizeof(int) * (pass + 1));
        free(lam); free(vecs); free(res); free(ab);
        out->total_s = now_s() - t_start;
        goto out;
      }
      prev_trace = trc;
      prev_count = cnt;
      m = mo;
      op_apply(&B, x, m, y);
    }
  }
out:
  if (rc && !g_err[0]) snprintf(g_err, sizeof g_err, "error %d", rc);
  if (sys) { for (int e = 0; e < (cfg ? cfg->n_e : 0); ++e) shift_free(&sys[e]); free(sys); }
  free(y); free(q); free(x); free(ev); free(hist); free(cnts);
  op_free(&A);
  op_free(&B);
  return rc;
}
