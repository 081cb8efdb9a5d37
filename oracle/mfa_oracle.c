/* oracle/mfa_oracle.c — plain-C restatement of the reference MFA encode path.
 *
 * TEST INFRASTRUCTURE ONLY (see mfa_oracle.h).  Each function cites the
 * reference file:line it restates (paths under /root/reference/proj).  The
 * restatement is validated against the reference itself (oracle/_ref) by
 * tests/test_oracle_vs_ref.py and against tests/golden/ fixtures.
 *
 * Numerical notes: Gram and R^T accumulations run in the same row order as
 * the reference; the Cholesky is a dense Cholesky-Crout (the reference calls
 * Eigen's LLT, whose last bits depend on the Eigen build), so control points
 * agree with the reference at rounding level, not bitwise.  Spans,
 * first_col/count and every layout integer are bit-exact.
 */
#include "mfa_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];
static int g_err_dim = -1;
static int64_t g_err_span = -1;

const char* orc_last_error(void) { return g_err; }
int orc_last_error_dim(void) { return g_err_dim; }
int64_t orc_last_error_span(void) { return g_err_span; }

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

#define TRY(x)             \
  do {                     \
    int rc_ = (x);         \
    if (rc_) return rc_;   \
  } while (0)

static int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
static int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

/* ------------------------------------------------------------------ knots */

/* knots.cpp:48-81 */
int orc_make_knot_vector(int degree, int basis_count, double a, double b, int clamp_left, int clamp_right,
                         double* out) {
  if (degree < 1) return fail(1, "make_knot_vector: degree must be >= 1");
  if (basis_count < degree + 1) return fail(1, "make_knot_vector: basis count must be at least p+1");
  if (!(a < b)) return fail(1, "make_knot_vector: range must satisfy a < b");
  const int p = degree, n = basis_count, spans = n - p;
  const double h = (b - a) / spans;
  int o = 0;
  if (clamp_left) {
    for (int i = 0; i <= p; ++i) out[o++] = a;
  } else {
    for (int i = p; i >= 1; --i) out[o++] = a - i * h;
    out[o++] = a;
  }
  for (int k = 1; k < spans; ++k) out[o++] = a + k * h;
  if (clamp_right) {
    for (int i = 0; i <= p; ++i) out[o++] = b;
  } else {
    out[o++] = b;
    for (int i = 1; i <= p; ++i) out[o++] = b + i * h;
  }
  return 0;
}

/* knots.cpp:83-106: knots[s] <= u < knots[s+1]; u == max -> last nonempty */
int orc_find_span(const double* knots, int nknots, int degree, double u, int* out_span) {
  const int p = degree, n = nknots - p - 1;
  const double lo = knots[p], hi = knots[n];
  if (u < lo || u > hi) return fail(2, "find_span: parameter %g outside evaluable range [%g, %g]", u, lo, hi);
  if (u >= hi) {
    int s = n - 1;
    while (s > p && knots[s] == knots[s + 1]) --s;
    *out_span = s;
    return 0;
  }
  int low = p, high = n, mid = (low + high) / 2;
  while (u < knots[mid] || u >= knots[mid + 1]) {
    if (u < knots[mid])
      high = mid;
    else
      low = mid;
    mid = (low + high) / 2;
  }
  *out_span = mid;
  return 0;
}

/* knots.cpp:108-129: Cox-de Boor triangle */
void orc_basis_funs(const double* knots, int degree, int span, double u, double* N) {
  const int p = degree;
  double left[32], right[32];
  N[0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    left[j] = u - knots[span + 1 - j];
    right[j] = knots[span + j] - u;
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      const double denom = right[r + 1] + left[j - r];
      const double temp = N[r] / denom;
      N[r] = saved + right[r + 1] * temp;
      saved = left[j - r] * temp;
    }
    N[j] = saved;
  }
}

/* ------------------------------------------------------------ collocation */

typedef struct {
  int64_t rows, cols;
  int band;
  int64_t* first_col;
  int* count;
  double* values; /* rows x band */
} banded_t;

static void banded_free(banded_t* m) {
  free(m->first_col);
  free(m->count);
  free(m->values);
  memset(m, 0, sizeof *m);
}

/* collocation.cpp:83-111 (window clipping at :98-108) */
static int collocation_window(const double* knots, int nknots, int p, const double* params, int64_t m, int64_t col_lo,
                              int64_t col_hi, banded_t* out) {
  const int nbasis = nknots - p - 1;
  if (m <= 0) return fail(1, "collocation_matrix: empty parameter list");
  if (col_lo < 0 || col_hi > nbasis || col_lo >= col_hi) return fail(1, "collocation_matrix: bad column window");
  for (int64_t j = 1; j < m; ++j)
    if (params[j] < params[j - 1]) return fail(1, "collocation_matrix: params must be ascending");
  out->rows = m;
  out->cols = col_hi - col_lo;
  out->band = p + 1;
  out->first_col = calloc((size_t)m, sizeof(int64_t));
  out->count = calloc((size_t)m, sizeof(int));
  out->values = calloc((size_t)(m * (p + 1)), sizeof(double));
  double nb[32];
  for (int64_t j = 0; j < m; ++j) {
    int span;
    int rc = orc_find_span(knots, nknots, p, params[j], &span);
    if (rc) {
      banded_free(out);
      return rc;
    }
    orc_basis_funs(knots, p, span, params[j], nb);
    const int64_t g0 = span - p;
    const int64_t lo = imax64(g0, col_lo), hi = imin64(g0 + p + 1, col_hi);
    if (lo >= hi) {
      banded_free(out);
      return fail(1, "collocation_matrix: param %g has no active basis inside the column window", params[j]);
    }
    int c = 0;
    for (int64_t g = lo; g < hi; ++g) out->values[j * (p + 1) + c++] = nb[g - g0];
    out->first_col[j] = lo - col_lo;
    out->count[j] = c;
  }
  return 0;
}

int orc_collocation(const double* knots, int nknots, int degree, const double* params, int64_t m, int64_t col_lo,
                    int64_t col_hi, int64_t* out_first_col, int* out_count, double* out_values) {
  banded_t bc;
  TRY(collocation_window(knots, nknots, degree, params, m, col_lo, col_hi, &bc));
  memcpy(out_first_col, bc.first_col, (size_t)m * sizeof(int64_t));
  memcpy(out_count, bc.count, (size_t)m * sizeof(int));
  memcpy(out_values, bc.values, (size_t)(m * (degree + 1)) * sizeof(double));
  banded_free(&bc);
  return 0;
}

/* collocation.cpp:36-44: y[j] = sum_k v[k] x[(c0+k)*stride] */
static void apply_line(const banded_t* m, const double* x, int64_t xs, double* y) {
  for (int64_t j = 0; j < m->rows; ++j) {
    const double* v = m->values + j * m->band;
    const int64_t c0 = m->first_col[j];
    double acc = 0.0;
    for (int k = 0; k < m->count[j]; ++k) acc += v[k] * x[(c0 + k) * xs];
    y[j] = acc;
  }
}

/* collocation.cpp:46-54: x[c0+k] += v[k] y[j], row order */
static void apply_transpose_line(const banded_t* m, const double* y, int64_t ys, double* x) {
  for (int64_t c = 0; c < m->cols; ++c) x[c] = 0.0;
  for (int64_t j = 0; j < m->rows; ++j) {
    const double* v = m->values + j * m->band;
    const int64_t c0 = m->first_col[j];
    const double yj = y[j * ys];
    for (int k = 0; k < m->count[j]; ++k) x[c0 + k] += v[k] * yj;
  }
}

/* collocation.cpp:56-67: dense A^T A, accumulated row by row */
static double* gram(const banded_t* m) {
  const int64_t n = m->cols;
  double* g = calloc((size_t)(n * n), sizeof(double));
  for (int64_t j = 0; j < m->rows; ++j) {
    const double* v = m->values + j * m->band;
    const int64_t c0 = m->first_col[j];
    const int c = m->count[j];
    for (int a = 0; a < c; ++a)
      for (int b = 0; b < c; ++b) g[(c0 + a) * n + (c0 + b)] += v[a] * v[b];
  }
  return g;
}

/* --------------------------------------------------------------- tensors */

typedef struct {
  int rank;
  int64_t ext[3];
  double* data;
} tensor_t;

static int64_t tsize(const tensor_t* t) {
  int64_t s = 1;
  for (int d = 0; d < t->rank; ++d) s *= t->ext[d];
  return s;
}

static void tstrides(int rank, const int64_t* ext, int64_t* st) {
  int64_t s = 1;
  for (int d = rank - 1; d >= 0; --d) {
    st[d] = s;
    s *= ext[d];
  }
}

typedef void (*line_fn)(const void* ctx, const double* src, int64_t stride, double* dst);

/* tensor.hpp:78-106 apply_along_axis: lines enumerate in row-major order of
 * the non-axis indices; fn writes out_extent dense values. */
static tensor_t apply_along_axis(const tensor_t* in, int axis, int64_t out_extent, line_fn fn, const void* ctx) {
  tensor_t out;
  out.rank = in->rank;
  for (int d = 0; d < in->rank; ++d) out.ext[d] = in->ext[d];
  out.ext[axis] = out_extent;
  out.data = calloc((size_t)tsize(&out), sizeof(double));
  int64_t ist[3], ost[3];
  tstrides(in->rank, in->ext, ist);
  tstrides(out.rank, out.ext, ost);
  double* line = malloc((size_t)out_extent * sizeof(double));
  int64_t idx[3] = {0, 0, 0};
  for (;;) {
    int64_t ib = 0, ob = 0;
    for (int d = 0; d < in->rank; ++d)
      if (d != axis) {
        ib += idx[d] * ist[d];
        ob += idx[d] * ost[d];
      }
    fn(ctx, in->data + ib, ist[axis], line);
    for (int64_t k = 0; k < out_extent; ++k) out.data[ob + k * ost[axis]] = line[k];
    int d = in->rank - 1;
    for (; d >= 0; --d) {
      if (d == axis) continue;
      if (++idx[d] < in->ext[d]) break;
      idx[d] = 0;
    }
    if (d < 0) break;
  }
  free(line);
  return out;
}

/* ------------------------------------------------------------------ LSQ */

typedef struct {
  const banded_t* m;
  const double* L; /* n x n lower, row-major */
  int64_t n;
} fit_ctx;

/* lsq.cpp:57-61: line -> L^-T L^-1 (R^T line) */
static void fit_line(const void* vctx, const double* src, int64_t stride, double* dst) {
  const fit_ctx* c = vctx;
  apply_transpose_line(c->m, src, stride, dst);
  const int64_t n = c->n;
  for (int64_t i = 0; i < n; ++i) {
    double s = dst[i];
    for (int64_t k = 0; k < i; ++k) s -= c->L[i * n + k] * dst[k];
    dst[i] = s / c->L[i * n + i];
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = dst[i];
    for (int64_t k = i + 1; k < n; ++k) s -= c->L[k * n + i] * dst[k];
    dst[i] = s / c->L[i * n + i];
  }
}

static void decode_line(const void* vctx, const double* src, int64_t stride, double* dst) {
  apply_line(((const fit_ctx*)vctx)->m, src, stride, dst);
}

/* lsq.cpp:25-35 */
static int64_t uncovered_column(const banded_t* m) {
  char* cov = calloc((size_t)m->cols, 1);
  for (int64_t j = 0; j < m->rows; ++j)
    for (int k = 0; k < m->count[j]; ++k)
      if (m->values[j * m->band + k] != 0.0) cov[m->first_col[j] + k] = 1;
  int64_t r = -1;
  for (int64_t c = 0; c < m->cols; ++c)
    if (!cov[c]) {
      r = c;
      break;
    }
  free(cov);
  return r;
}

/* lsq.cpp:9-20 LocalProblem::validate + lsq.cpp:39-64 fit_unconstrained.
 * The Cholesky (Eigen LLT at lsq.cpp:48) is restated as dense Crout. */
static int fit(const banded_t* r, const tensor_t* q, tensor_t* out) {
  for (int d = 0; d < q->rank; ++d) {
    if (r[d].rows != q->ext[d]) return fail(1, "LocalProblem: row count mismatch in dimension %d", d);
    if (r[d].rows < r[d].cols)
      return fail(1, "LocalProblem: underdetermined in dimension %d (%lld rows < %lld cols)", d,
                  (long long)r[d].rows, (long long)r[d].cols);
  }
  tensor_t cur = *q;
  cur.data = malloc((size_t)tsize(q) * sizeof(double));
  memcpy(cur.data, q->data, (size_t)tsize(q) * sizeof(double));
  for (int d = 0; d < q->rank; ++d) {
    const int64_t n = r[d].cols;
    double* g = gram(&r[d]);
    double* L = calloc((size_t)(n * n), sizeof(double));
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j <= i; ++j) {
        double s = g[i * n + j];
        for (int64_t k = 0; k < j; ++k) s -= L[i * n + k] * L[j * n + k];
        if (i == j) {
          if (!(s > 0.0)) {
            const int64_t col = uncovered_column(&r[d]);
            free(g);
            free(L);
            free(cur.data);
            g_err_dim = d;
            g_err_span = col;
            return fail(3, "fit_unconstrained: singular normal matrix in dimension %d", d);
          }
          L[i * n + i] = sqrt(s);
        } else {
          L[i * n + j] = s / L[j * n + j];
        }
      }
    fit_ctx c = {&r[d], L, n};
    tensor_t nxt = apply_along_axis(&cur, d, n, fit_line, &c);
    free(cur.data);
    cur = nxt;
    free(g);
    free(L);
  }
  *out = cur;
  return 0;
}

/* decode.cpp:83-97 with pre-built windowed rows */
static tensor_t decode_rows(const tensor_t* controls, const banded_t* r) {
  tensor_t cur = *controls;
  cur.data = malloc((size_t)tsize(controls) * sizeof(double));
  memcpy(cur.data, controls->data, (size_t)tsize(controls) * sizeof(double));
  for (int d = 0; d < controls->rank; ++d) {
    fit_ctx c = {&r[d], NULL, 0};
    tensor_t nxt = apply_along_axis(&cur, d, r[d].rows, decode_line, &c);
    free(cur.data);
    cur = nxt;
  }
  return cur;
}

int orc_fit_unconstrained(int rank, int degree, const double* knots, const int64_t* kn_off, const double* params,
                          const int64_t* pm_off, const int64_t* col_lo, const int64_t* col_hi, const double* q,
                          double* out_p) {
  banded_t r[3];
  memset(r, 0, sizeof r);
  tensor_t qt = {rank, {1, 1, 1}, (double*)q};
  int rc = 0;
  for (int d = 0; d < rank && !rc; ++d) {
    qt.ext[d] = pm_off[d + 1] - pm_off[d];
    rc = collocation_window(knots + kn_off[d], (int)(kn_off[d + 1] - kn_off[d]), degree, params + pm_off[d],
                            qt.ext[d], col_lo[d], col_hi[d], &r[d]);
  }
  if (!rc) {
    tensor_t p;
    rc = fit(r, &qt, &p);
    if (!rc) {
      memcpy(out_p, p.data, (size_t)tsize(&p) * sizeof(double));
      free(p.data);
    }
  }
  for (int d = 0; d < rank; ++d) banded_free(&r[d]);
  return rc;
}

int orc_decode(int rank, int degree, const double* knots, const int64_t* kn_off, const double* params,
               const int64_t* pm_off, const int64_t* ctrl_ext, const int64_t* col_offset, const double* controls,
               double* out) {
  banded_t r[3];
  memset(r, 0, sizeof r);
  tensor_t ct = {rank, {1, 1, 1}, (double*)controls};
  int rc = 0;
  for (int d = 0; d < rank && !rc; ++d) {
    ct.ext[d] = ctrl_ext[d];
    const int64_t off = col_offset ? col_offset[d] : 0;
    rc = collocation_window(knots + kn_off[d], (int)(kn_off[d + 1] - kn_off[d]), degree, params + pm_off[d],
                            pm_off[d + 1] - pm_off[d], off, off + ctrl_ext[d], &r[d]);
  }
  if (!rc) {
    tensor_t o = decode_rows(&ct, r);
    memcpy(out, o.data, (size_t)tsize(&o) * sizeof(double));
    free(o.data);
  }
  for (int d = 0; d < rank; ++d) banded_free(&r[d]);
  return rc;
}

/* ---------------------------------------------------------------- layout */

enum { BD_SPAN_LO, BD_SPAN_HI, BD_DELTA_LO, BD_DELTA_HI, BD_OVL_LO, BD_OVL_HI, BD_LSPAN_LO, BD_LSPAN_HI,
       BD_DOF_LO, BD_DOF_HI, BD_OWN_LO, BD_OWN_HI, BD_IN_LO, BD_IN_HI, BD_OWNIN_LO, BD_OWNIN_HI, BD_N };

struct orc_dec {
  int rank, degree, clamp, nblocks;
  int64_t overlap;
  int64_t grid[3], n_ctrl[3], T[3];
  int blocks[3];
  int nknots[3];
  double* knots[3];
  int* span_knot[3];
  int* coords;  /* nblocks*rank */
  int64_t* bd;  /* nblocks*rank*BD_N */
  int* hr[3];   /* 2*n_ctrl */
  int* nbr_off; /* nblocks+1 */
  int* nbrs;
};

static int64_t* BD(const orc_dec* d, int b, int k) { return d->bd + ((int64_t)b * d->rank + k) * BD_N; }

/* layout.cpp:63-65 */
static int64_t face_span(int64_t a, int64_t T, int64_t B) { return (2 * a * T + B - 1) / (2 * B); }
/* layout.cpp:68-70 */
static int64_t input_floor(int64_t t, int64_t T, int64_t m) { return (t * (m - 1) + T - 1) / T; }

void orc_dec_free(orc_dec* d) {
  if (!d) return;
  for (int k = 0; k < 3; ++k) {
    free(d->knots[k]);
    free(d->span_knot[k]);
    free(d->hr[k]);
  }
  free(d->coords);
  free(d->bd);
  free(d->nbr_off);
  free(d->nbrs);
  free(d);
}

/* layout.cpp:205-215 shared_dof_box emptiness */
static int shared_box(const orc_dec* d, int a, int b, int64_t box[3][2]) {
  for (int k = 0; k < d->rank; ++k) {
    const int64_t* da = BD(d, a, k);
    const int64_t* db = BD(d, b, k);
    box[k][0] = imax64(da[BD_DOF_LO], db[BD_DOF_LO]);
    box[k][1] = imin64(da[BD_DOF_HI], db[BD_DOF_HI]);
    if (box[k][0] >= box[k][1]) return 0;
  }
  return 1;
}

/* layout.cpp:217-342 partition (+ plan_dim :81-121, SharedDofMap :125-146) */
int orc_partition(int rank, const int64_t* grid, const int* blocks, int degree, const int64_t* nctrl_blk,
                  int64_t overlap, int clamp, orc_dec** out) {
  if (rank < 1 || rank > 3) return fail(1, "partition: 1, 2 or 3 dimensions supported");
  if (degree < 1) return fail(1, "partition: degree must be >= 1");
  if (overlap < 0) return fail(1, "partition: overlap must be >= 0");
  const int p = degree;
  const int64_t w = p / 2;
  orc_dec* d = calloc(1, sizeof *d);
  d->rank = rank;
  d->degree = p;
  d->clamp = clamp;
  d->overlap = clamp ? 0 : overlap;
  int64_t* face[3] = {0, 0, 0};
  int rc = 0;
  for (int k = 0; k < rank && !rc; ++k) {
    d->grid[k] = grid[k];
    d->blocks[k] = blocks[k];
    if (blocks[k] < 1) {
      rc = fail(1, "partition: blocks per dimension must be >= 1");
      break;
    }
    if (nctrl_blk[k] < p + 1) {
      rc = fail(1, "partition: nctrl per block must be at least p+1 in dimension %d", k);
      break;
    }
    const int B = blocks[k];
    const int64_t nb = nctrl_blk[k];
    if (!clamp || B == 1) {
      d->n_ctrl[k] = (int64_t)B * nb;
      d->nknots[k] = (int)(d->n_ctrl[k] + p + 1);
      d->knots[k] = malloc((size_t)d->nknots[k] * sizeof(double));
      rc = orc_make_knot_vector(p, (int)d->n_ctrl[k], 0.0, 1.0, 1, 1, d->knots[k]);
      if (rc) break;
    } else {
      d->n_ctrl[k] = (int64_t)B * (nb - 1) + 1;
      const int64_t seg = nb - p;
      if (seg < 1) {
        rc = fail(1, "partition: clamp_interfaces requires nctrl per block > degree");
        break;
      }
      const int64_t spans = (int64_t)B * seg;
      const double h = 1.0 / (double)spans;
      d->nknots[k] = (int)(d->n_ctrl[k] + p + 1);
      d->knots[k] = malloc((size_t)d->nknots[k] * sizeof(double));
      int o = 0;
      for (int i = 0; i <= p; ++i) d->knots[k][o++] = 0.0;
      for (int64_t t = 1; t < spans; ++t) {
        const double v = (double)t * h;
        d->knots[k][o++] = v;
        if (t % seg == 0)
          for (int r = 1; r < p; ++r) d->knots[k][o++] = v;
      }
      for (int i = 0; i <= p; ++i) d->knots[k][o++] = 1.0;
    }
    const int n = d->nknots[k] - p - 1;
    d->span_knot[k] = malloc((size_t)n * sizeof(int));
    int T = 0;
    for (int s = p; s < n; ++s)
      if (d->knots[k][s] < d->knots[k][s + 1]) d->span_knot[k][T++] = s;
    d->T[k] = T;
    face[k] = malloc((size_t)(B + 1) * sizeof(int64_t));
    for (int b = 0; b <= B; ++b) face[k][b] = (!clamp || B == 1) ? face_span(b, T, B) : (int64_t)b * (nb - p);
    face[k][0] = 0;
    face[k][B] = T;
    if (grid[k] < d->n_ctrl[k]) {
      rc = fail(1, "partition: input count must be >= control count in dimension %d", k);
      break;
    }
    if (!clamp && B > 1) {
      int64_t mn = INT64_MAX;
      for (int b = 0; b < B; ++b) mn = imin64(mn, face[k][b + 1] - face[k][b]);
      if (w + d->overlap > mn) {
        rc = fail(1,
                  "partition: overlap too large in dimension %d: delta+overlap spans (%lld) exceed the smallest "
                  "block (%lld spans); exchanges would cross non-neighbor blocks",
                  k, (long long)(w + d->overlap), (long long)mn);
        break;
      }
    }
  }
  if (rc) {
    for (int k = 0; k < 3; ++k) free(face[k]);
    orc_dec_free(d);
    return rc;
  }
  int nblocks = 1;
  for (int k = 0; k < rank; ++k) nblocks *= blocks[k];
  d->nblocks = nblocks;
  d->coords = calloc((size_t)nblocks * rank, sizeof(int));
  d->bd = calloc((size_t)nblocks * rank * BD_N, sizeof(int64_t));
  const int64_t c_hi = p - w;
  int coords[3] = {0, 0, 0};
  for (int id = 0; id < nblocks; ++id) {
    for (int k = 0; k < rank; ++k) {
      d->coords[id * rank + k] = coords[k];
      const int b = coords[k], B = blocks[k];
      const int64_t T = d->T[k], m = grid[k];
      int64_t* bd = BD(d, id, k);
      bd[BD_SPAN_LO] = face[k][b];
      bd[BD_SPAN_HI] = face[k][b + 1];
      if (!clamp) {
        bd[BD_DELTA_LO] = b > 0 ? w : 0;
        bd[BD_DELTA_HI] = b < B - 1 ? w : 0;
        bd[BD_OVL_LO] = b > 0 ? d->overlap : 0;
        bd[BD_OVL_HI] = b < B - 1 ? d->overlap : 0;
      }
      bd[BD_LSPAN_LO] = bd[BD_SPAN_LO] - bd[BD_DELTA_LO] - bd[BD_OVL_LO];
      bd[BD_LSPAN_HI] = bd[BD_SPAN_HI] + bd[BD_DELTA_HI] + bd[BD_OVL_HI];
      if (!clamp) {
        /* layout.cpp:298-305 */
        bd[BD_DOF_LO] = bd[BD_LSPAN_LO] == 0 ? 0 : bd[BD_LSPAN_LO] + c_hi;
        bd[BD_DOF_HI] = bd[BD_LSPAN_HI] == T ? d->n_ctrl[k] : bd[BD_LSPAN_HI] + c_hi;
        bd[BD_OWN_LO] = bd[BD_SPAN_LO] == 0 ? 0 : bd[BD_SPAN_LO] + c_hi;
        bd[BD_OWN_HI] = bd[BD_SPAN_HI] == T ? d->n_ctrl[k] : bd[BD_SPAN_HI] + c_hi;
      } else {
        /* layout.cpp:306-313 */
        bd[BD_DOF_LO] = d->span_knot[k][bd[BD_LSPAN_LO]] - p;
        bd[BD_DOF_HI] = d->span_knot[k][bd[BD_LSPAN_HI] - 1] + 1;
        bd[BD_OWN_LO] = bd[BD_DOF_LO] + (b > 0 ? 1 : 0);
        bd[BD_OWN_HI] = bd[BD_DOF_HI];
      }
      /* layout.cpp:315-318 */
      bd[BD_IN_LO] = input_floor(bd[BD_LSPAN_LO], T, m);
      bd[BD_IN_HI] = bd[BD_LSPAN_HI] == T ? m : input_floor(bd[BD_LSPAN_HI], T, m);
      bd[BD_OWNIN_LO] = input_floor(bd[BD_SPAN_LO], T, m);
      bd[BD_OWNIN_HI] = bd[BD_SPAN_HI] == T ? m : input_floor(bd[BD_SPAN_HI], T, m);
    }
    for (int k = rank - 1; k >= 0; --k) {
      if (++coords[k] < blocks[k]) break;
      coords[k] = 0;
    }
  }
  for (int k = 0; k < 3; ++k) free(face[k]);
  /* layout.cpp:125-146 SharedDofMap holder ranges */
  for (int k = 0; k < rank; ++k) {
    d->hr[k] = malloc((size_t)(2 * d->n_ctrl[k]) * sizeof(int));
    for (int64_t i = 0; i < d->n_ctrl[k]; ++i) {
      d->hr[k][2 * i] = 0;
      d->hr[k][2 * i + 1] = -1;
    }
    for (int id = 0; id < nblocks; ++id) {
      const int c = d->coords[id * rank + k];
      const int64_t* bd = BD(d, id, k);
      for (int64_t i = bd[BD_DOF_LO]; i < bd[BD_DOF_HI]; ++i) {
        int* r = d->hr[k] + 2 * i;
        if (r[1] < r[0]) {
          r[0] = c;
          r[1] = c;
        } else {
          if (c < r[0]) r[0] = c;
          if (c > r[1]) r[1] = c;
        }
      }
    }
  }
  /* layout.cpp:328-340 neighbors */
  d->nbr_off = calloc((size_t)nblocks + 1, sizeof(int));
  d->nbrs = malloc((size_t)nblocks * 27 * sizeof(int));
  int cnt = 0;
  for (int id = 0; id < nblocks; ++id) {
    d->nbr_off[id] = cnt;
    for (int o = 0; o < nblocks; ++o) {
      if (o == id) continue;
      int adj = 1;
      for (int k = 0; k < rank; ++k) {
        const int diff = abs(d->coords[o * rank + k] - d->coords[id * rank + k]);
        if (diff > 1) adj = 0;
      }
      int64_t box[3][2];
      if (adj && shared_box(d, id, o, box)) d->nbrs[cnt++] = o;
    }
  }
  d->nbr_off[nblocks] = cnt;
  *out = d;
  return 0;
}

int orc_dec_nblocks(const orc_dec* d) { return d->nblocks; }
void orc_dec_blockdims(const orc_dec* d, int64_t* out) {
  memcpy(out, d->bd, (size_t)d->nblocks * d->rank * BD_N * sizeof(int64_t));
}
void orc_dec_coords(const orc_dec* d, int* out) { memcpy(out, d->coords, (size_t)d->nblocks * d->rank * sizeof(int)); }
void orc_dec_nctrl(const orc_dec* d, int64_t* out) {
  for (int k = 0; k < d->rank; ++k) out[k] = d->n_ctrl[k];
}
int orc_dec_knots(const orc_dec* d, int dim, double* out) {
  if (out) memcpy(out, d->knots[dim], (size_t)d->nknots[dim] * sizeof(double));
  return d->nknots[dim];
}
void orc_dec_holder_ranges(const orc_dec* d, int dim, int* out) {
  memcpy(out, d->hr[dim], (size_t)(2 * d->n_ctrl[dim]) * sizeof(int));
}
int orc_dec_neighbors(const orc_dec* d, int block, int* out, int cap) {
  const int n = d->nbr_off[block + 1] - d->nbr_off[block];
  for (int i = 0; i < n && i < cap; ++i) out[i] = d->nbrs[d->nbr_off[block] + i];
  return n;
}

/* ---------------------------------------------------------------- solver */

typedef struct {
  int iteration;
  double dp, jss, jms;
  double* block_err; /* nblocks*2 or NULL */
} epoch_t;

struct orc_result {
  int converged, ci, nepochs, njumps, nblocks, rank;
  double final_dp, l2, linf;
  epoch_t* epochs;
  double* jumps; /* 4 per pair */
  tensor_t controls, error;
  tensor_t* bp;
};

void orc_result_free(orc_result* r) {
  if (!r) return;
  for (int e = 0; e < r->nepochs; ++e) free(r->epochs[e].block_err);
  free(r->epochs);
  free(r->jumps);
  free(r->controls.data);
  free(r->error.data);
  if (r->bp)
    for (int b = 0; b < r->nblocks; ++b) free(r->bp[b].data);
  free(r->bp);
  free(r);
}

static int n_s_of(const orc_dec* d, const int64_t* dof) {
  int c = 1;
  for (int k = 0; k < d->rank; ++k) c *= d->hr[k][2 * dof[k] + 1] - d->hr[k][2 * dof[k]] + 1;
  return c;
}

/* layout.cpp:177-195 holders(): ascending block ids */
static int holders_of(const orc_dec* d, const int64_t* dof, int* ids) {
  int n = 0, c[3] = {0, 0, 0};
  for (int k = 0; k < d->rank; ++k) c[k] = d->hr[k][2 * dof[k]];
  for (;;) {
    int id = 0;
    for (int k = 0; k < d->rank; ++k) id = id * d->blocks[k] + c[k];
    ids[n++] = id;
    int k = d->rank - 1;
    for (; k >= 0; --k) {
      if (++c[k] <= d->hr[k][2 * dof[k] + 1]) break;
      c[k] = d->hr[k][2 * dof[k]];
    }
    if (k < 0) break;
  }
  /* ids are generated in lexicographic coordinate order == ascending id */
  return n;
}

static double* bp_at(const orc_dec* d, tensor_t* bp, int b, const int64_t* dof) {
  int64_t off = 0;
  for (int k = 0; k < d->rank; ++k) off = off * bp[b].ext[k] + (dof[k] - BD(d, b, k)[BD_DOF_LO]);
  return bp[b].data + off;
}

/* box iteration helper: advances idx in row-major order within box */
static int box_next(int rank, int64_t box[3][2], int64_t* idx) {
  int k = rank - 1;
  for (; k >= 0; --k) {
    if (++idx[k] < box[k][1]) return 1;
    idx[k] = box[k][0];
  }
  return 0;
}

/* solver.cpp:166-193 jump_residuals, reduced per class; fills per-pair list
 * when `pairs` is non-NULL. */
static void jumps(const orc_dec* d, tensor_t* bp, double* jss, double* jms, double* pairs, int* npairs) {
  *jss = 0.0;
  *jms = 0.0;
  int np = 0;
  for (int a = 0; a < d->nblocks; ++a)
    for (int t = d->nbr_off[a]; t < d->nbr_off[a + 1]; ++t) {
      const int b = d->nbrs[t];
      if (b < a) continue;
      int64_t box[3][2], idx[3];
      double ss = 0.0, ms = 0.0;
      if (shared_box(d, a, b, box)) {
        for (int k = 0; k < d->rank; ++k) idx[k] = box[k][0];
        do {
          const double diff = fabs(*bp_at(d, bp, a, idx) - *bp_at(d, bp, b, idx));
          if (n_s_of(d, idx) > 2) {
            if (diff > ms) ms = diff;
          } else if (diff > ss) {
            ss = diff;
          }
        } while (box_next(d->rank, box, idx));
      }
      if (ss > *jss) *jss = ss;
      if (ms > *jms) *jms = ms;
      if (pairs) {
        pairs[4 * np + 0] = a;
        pairs[4 * np + 1] = b;
        pairs[4 * np + 2] = ss;
        pairs[4 * np + 3] = ms;
      }
      ++np;
    }
  if (npairs) *npairs = np;
}

static double tlinf(const tensor_t* t) {
  double m = 0.0;
  const int64_t n = tsize(t);
  for (int64_t i = 0; i < n; ++i)
    if (fabs(t->data[i]) > m) m = fabs(t->data[i]);
  return m;
}

/* lsq.cpp:66-85 residual_error */
static void residual(const banded_t* r, const tensor_t* q, const tensor_t* p, double* l2, double* linf) {
  tensor_t dec = decode_rows(p, r);
  double sq = 0.0, mx = 0.0;
  const int64_t n = tsize(q);
  for (int64_t i = 0; i < n; ++i) {
    const double e = q->data[i] - dec.data[i];
    sq += e * e;
    if (fabs(e) > mx) mx = fabs(e);
  }
  *l2 = sqrt(sq);
  *linf = mx;
  free(dec.data);
}

int orc_solve(const orc_dec* d, const double* field, int max_iters, double tol, int log_errors, int enforce,
              orc_result** out) {
  if (max_iters < 1) return fail(1, "SolverConfig: max iterations must be >= 1");
  if (!(tol > 0.0)) return fail(1, "SolverConfig: tolerance must be > 0");
  const int D = d->rank, NB = d->nblocks, p = d->degree;
  int64_t gst[3];
  tstrides(D, d->grid, gst);
  banded_t* R = calloc((size_t)NB * D, sizeof(banded_t));
  tensor_t* Q = calloc((size_t)NB, sizeof(tensor_t));
  orc_result* res = calloc(1, sizeof *res);
  res->nblocks = NB;
  res->rank = D;
  res->bp = calloc((size_t)NB, sizeof(tensor_t));
  res->epochs = calloc((size_t)max_iters + 1, sizeof(epoch_t));
  int rc = 0;
  /* solver.cpp:48-95 make_block_state */
  for (int b = 0; b < NB && !rc; ++b) {
    Q[b].rank = D;
    for (int k = 0; k < D; ++k) {
      const int64_t* bd = BD(d, b, k);
      const int64_t m = bd[BD_IN_HI] - bd[BD_IN_LO];
      Q[b].ext[k] = m;
      double* u = malloc((size_t)m * sizeof(double));
      for (int64_t j = 0; j < m; ++j) u[j] = (double)(bd[BD_IN_LO] + j) / (double)(d->grid[k] - 1);
      rc = collocation_window(d->knots[k], d->nknots[k], p, u, m, bd[BD_DOF_LO], bd[BD_DOF_HI], &R[b * D + k]);
      free(u);
      if (rc) break;
      if (R[b * D + k].rows < R[b * D + k].cols) {
        rc = fail(1, "block %d: LocalProblem: underdetermined in dimension %d", b, k);
        break;
      }
    }
    if (rc) break;
    for (int k = D; k < 3; ++k) Q[b].ext[k] = 1;
    const int64_t n = tsize(&Q[b]);
    Q[b].data = malloc((size_t)n * sizeof(double));
    int64_t idx[3] = {0, 0, 0};
    for (int64_t i = 0; i < n; ++i) {
      int64_t g = 0;
      for (int k = 0; k < D; ++k) g += (BD(d, b, k)[BD_IN_LO] + idx[k]) * gst[k];
      Q[b].data[i] = field[g];
      for (int k = D - 1; k >= 0; --k) {
        if (++idx[k] < Q[b].ext[k]) break;
        idx[k] = 0;
      }
    }
  }
  /* solver.cpp:369-373 decoupled local fits */
  for (int b = 0; b < NB && !rc; ++b) rc = fit(&R[b * D], &Q[b], &res->bp[b]);

  if (!rc) {
    /* solver.cpp:349-366 record_epoch */
#define RECORD(it, dpv)                                                                   \
  do {                                                                                    \
    epoch_t* e_ = &res->epochs[res->nepochs++];                                           \
    e_->iteration = (it);                                                                 \
    e_->dp = (dpv);                                                                       \
    jumps(d, res->bp, &e_->jss, &e_->jms, NULL, NULL);                                    \
    if (log_errors) {                                                                     \
      e_->block_err = calloc((size_t)NB * 2, sizeof(double));                             \
      for (int b_ = 0; b_ < NB; ++b_)                                                     \
        residual(&R[b_ * D], &Q[b_], &res->bp[b_], &e_->block_err[2 * b_], &e_->block_err[2 * b_ + 1]); \
    }                                                                                     \
  } while (0)
    RECORD(0, 0.0);
    int any_shared = 0;
    for (int k = 0; k < D; ++k)
      for (int64_t i = 0; i < d->n_ctrl[k]; ++i)
        if (d->hr[k][2 * i + 1] > d->hr[k][2 * i]) any_shared = 1;
    res->converged = 1;
    if (enforce && any_shared) {
      res->converged = 0;
      tensor_t* snap = calloc((size_t)NB, sizeof(tensor_t));
      double* change = calloc((size_t)NB, sizeof(double));
      for (int iter = 1; iter <= max_iters; ++iter) {
        /* runtime.cpp:123-158: messages are a pre-epoch snapshot */
        for (int b = 0; b < NB; ++b) {
          snap[b] = res->bp[b];
          snap[b].data = malloc((size_t)tsize(&res->bp[b]) * sizeof(double));
          memcpy(snap[b].data, res->bp[b].data, (size_t)tsize(&res->bp[b]) * sizeof(double));
        }
        /* solver.cpp:112-164 enforce_constraints, per block */
        for (int b = 0; b < NB; ++b) {
          int64_t box[3][2], idx[3];
          for (int k = 0; k < D; ++k) {
            box[k][0] = BD(d, b, k)[BD_DOF_LO];
            box[k][1] = BD(d, b, k)[BD_DOF_HI];
            idx[k] = box[k][0];
          }
          double mc = 0.0;
          do {
            const int ns = n_s_of(d, idx);
            if (ns < 2) continue;
            int ids[27];
            holders_of(d, idx, ids);
            /* solver.cpp:134-141: contributions arrive only from neighbors
             * (coordinate distance <= 1, runtime.cpp:17-21); every other
             * holder must have sent, else runtime_error. */
            int received = 0;
            for (int h = 0; h < ns; ++h) {
              if (ids[h] == b) continue;
              int near = 1;
              for (int k = 0; k < D; ++k)
                if (abs(d->coords[ids[h] * D + k] - d->coords[b * D + k]) > 1) near = 0;
              received += near;
            }
            if (received != ns - 1) {
              for (int b2 = 0; b2 < NB; ++b2) free(snap[b2].data);
              free(snap);
              free(change);
              rc = fail(4, "enforce_constraints: block %d received %d contributions for a control shared by %d blocks",
                        b, received, ns);
              goto solve_failed;
            }
            if (iter < 2 && ns > 2) continue;
            double sum = 0.0;
            for (int h = 0; h < ns; ++h) sum += *bp_at(d, snap, ids[h], idx);
            const double avg = sum / (double)ns;
            double* own = bp_at(d, res->bp, b, idx);
            const double ch = fabs(avg - *own);
            if (ch > mc) mc = ch;
            *own = avg;
          } while (box_next(D, box, idx));
          change[b] = mc;
        }
        for (int b = 0; b < NB; ++b) free(snap[b].data);
        /* solver.cpp:402-414 */
        double dp = 0.0;
        for (int b = 0; b < NB; ++b) {
          const double l = tlinf(&res->bp[b]);
          const double v = change[b] / (l > 1.0 ? l : 1.0);
          if (v > dp) dp = v;
        }
        RECORD(iter, dp);
        res->final_dp = dp;
        if (dp < tol) {
          res->converged = 1;
          res->ci = iter - 1;
          break;
        }
        res->ci = iter;
      }
      free(snap);
      free(change);
    }
  solve_failed:
    if (rc) goto cleanup;
    /* solver.cpp:416 final jumps */
    int np = 0;
    for (int a = 0; a < NB; ++a) np += d->nbr_off[a + 1] - d->nbr_off[a];
    res->jumps = calloc((size_t)np * 4 + 4, sizeof(double));
    double js, jm;
    jumps(d, res->bp, &js, &jm, res->jumps, &res->njumps);
    /* solver.cpp:418-423 assemble_owned */
    res->controls.rank = D;
    for (int k = 0; k < 3; ++k) res->controls.ext[k] = k < D ? d->n_ctrl[k] : 1;
    res->controls.data = calloc((size_t)tsize(&res->controls), sizeof(double));
    int64_t cst[3];
    tstrides(D, res->controls.ext, cst);
    for (int b = 0; b < NB; ++b) {
      int64_t box[3][2], idx[3];
      for (int k = 0; k < D; ++k) {
        box[k][0] = BD(d, b, k)[BD_OWN_LO];
        box[k][1] = BD(d, b, k)[BD_OWN_HI];
        idx[k] = box[k][0];
        if (box[k][0] >= box[k][1]) goto next_block;
      }
      do {
        int64_t g = 0;
        for (int k = 0; k < D; ++k) g += idx[k] * cst[k];
        res->controls.data[g] = *bp_at(d, res->bp, b, idx);
      } while (box_next(D, box, idx));
    next_block:;
    }
    /* solver.cpp:298-328,425-438 block_error_slab over the global lattice */
    res->error.rank = D;
    for (int k = 0; k < 3; ++k) res->error.ext[k] = k < D ? d->grid[k] : 1;
    res->error.data = calloc((size_t)tsize(&res->error), sizeof(double));
    double sq = 0.0;
    for (int b = 0; b < NB; ++b) {
      banded_t rr[3];
      memset(rr, 0, sizeof rr);
      int empty = 0;
      for (int k = 0; k < D && !rc; ++k) {
        const int64_t lo = BD(d, b, k)[BD_OWNIN_LO], hi = BD(d, b, k)[BD_OWNIN_HI];
        if (hi <= lo) {
          empty = 1;
          break;
        }
        double* u = malloc((size_t)(hi - lo) * sizeof(double));
        for (int64_t j = lo; j < hi; ++j) u[j - lo] = (double)j / (double)(d->grid[k] - 1);
        rc = collocation_window(d->knots[k], d->nknots[k], p, u, hi - lo, 0, d->n_ctrl[k], &rr[k]);
        free(u);
      }
      if (!empty && !rc) {
        tensor_t dec = decode_rows(&res->controls, rr);
        double l2sq = 0.0, linf = 0.0;
        int64_t idx[3] = {0, 0, 0};
        const int64_t n = tsize(&dec);
        for (int64_t i = 0; i < n; ++i) {
          int64_t g = 0;
          for (int k = 0; k < D; ++k) g += (BD(d, b, k)[BD_OWNIN_LO] + idx[k]) * gst[k];
          const double e = field[g] - dec.data[i];
          res->error.data[g] = e;
          l2sq += e * e;
          if (fabs(e) > linf) linf = fabs(e);
          for (int k = D - 1; k >= 0; --k) {
            if (++idx[k] < dec.ext[k]) break;
            idx[k] = 0;
          }
        }
        free(dec.data);
        sq += l2sq;
        if (linf > res->linf) res->linf = linf;
      }
      for (int k = 0; k < D; ++k) banded_free(&rr[k]);
    }
    res->l2 = sqrt(sq);
  }
cleanup:
  for (int b = 0; b < NB; ++b) {
    for (int k = 0; k < D; ++k) banded_free(&R[b * D + k]);
    free(Q[b].data);
  }
  free(R);
  free(Q);
  if (rc) {
    orc_result_free(res);
    return rc;
  }
  *out = res;
  return 0;
}

void orc_result_scalars(const orc_result* r, int* ints4, double* dbl3) {
  ints4[0] = r->converged;
  ints4[1] = r->ci;
  ints4[2] = r->nepochs;
  ints4[3] = r->njumps;
  dbl3[0] = r->final_dp;
  dbl3[1] = r->l2;
  dbl3[2] = r->linf;
}
void orc_result_epochs(const orc_result* r, double* out) {
  for (int e = 0; e < r->nepochs; ++e) {
    out[4 * e + 0] = r->epochs[e].iteration;
    out[4 * e + 1] = r->epochs[e].dp;
    out[4 * e + 2] = r->epochs[e].jss;
    out[4 * e + 3] = r->epochs[e].jms;
  }
}
void orc_result_block_errors(const orc_result* r, int epoch, double* out) {
  if (r->epochs[epoch].block_err) memcpy(out, r->epochs[epoch].block_err, (size_t)r->nblocks * 2 * sizeof(double));
}
void orc_result_final_jumps(const orc_result* r, double* out) {
  memcpy(out, r->jumps, (size_t)r->njumps * 4 * sizeof(double));
}
void orc_result_controls(const orc_result* r, double* out) {
  memcpy(out, r->controls.data, (size_t)tsize(&r->controls) * sizeof(double));
}
void orc_result_error(const orc_result* r, double* out) {
  memcpy(out, r->error.data, (size_t)tsize(&r->error) * sizeof(double));
}
void orc_result_block_p(const orc_result* r, int block, double* out) {
  memcpy(out, r->bp[block].data, (size_t)tsize(&r->bp[block]) * sizeof(double));
}
