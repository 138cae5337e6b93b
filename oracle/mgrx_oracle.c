/* TEST INFRASTRUCTURE ONLY — CPU oracle for the parity tests (see
 * mgrx_oracle.h for who may load it and how it is pinned).
 *
 * A plain-C restatement of the reference algorithm, organised the way the
 * GPU path is (natural-order level blocks, a separate fp64 component buffer,
 * one load+Thomas sweep per axis) rather than the reference's in-place
 * reordered field.  Every floating-point operation is performed in the same
 * order and with the same constants as the reference, and the file is built
 * with -ffp-contract=off like the reference (proj/CMakeLists.txt:12-14), so
 * results are bit-identical to it (pinned in tests/test_oracle.py).
 *
 * Arithmetic is carried in double; `rt()` rounds a stored value to the field
 * type T exactly as the reference's static_cast<T> does. */
#include "mgrx_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define MO_MAXD 16
#define MO_MAXL 64

/* 1 + mgrx::errc (error.hpp:9-36) */
enum {
  E_INVALID_DIMS = 1,
  E_DEPTH_EXCEEDED = 2,
  E_INVALID_LEVEL = 3,
  E_DEGENERATE_LINE = 5,
  E_DEGENERATE_SYSTEM = 6,
  E_SHAPE = 7,
  E_INVALID_BUDGET = 8,
  E_NONFINITE = 9,
  E_INVALID_INPUT = 15,
  E_NOMEM = 98
};

/* Mass-matrix constants with the spacing cancelled (transform.hpp:17-21). */
static const double kOff = 1.0 / 3.0;
static const double kDiagB = 2.0 / 3.0;
static const double kDiagI = 4.0 / 3.0;

static double rt(double v, int f32) { return f32 ? (double)(float)v : v; }

/* ---------------------------------------------------------------- grid --
 * GridHierarchy::max_levels / create (grid.cpp:9-49). */
typedef struct {
  int d, L;
  uint64_t dims[MO_MAXL][MO_MAXD]; /* [level][axis], level 0 = coarsest */
  uint64_t node[MO_MAXL], delta[MO_MAXL];
} hier_t;

static int bit_width(uint64_t x) {
  int w = 0;
  while (x) {
    ++w;
    x >>= 1;
  }
  return w;
}

int mo_max_levels(int nd, const uint64_t* dims, int* out) {
  if (nd <= 0 || nd > MO_MAXD) return E_INVALID_DIMS;
  int depth = 1 << 30;
  for (int i = 0; i < nd; ++i) {
    if (dims[i] < 2) return E_INVALID_DIMS;
    int k = bit_width(dims[i] - 1) - 1; /* floor(log2(n-1)) */
    if (k < depth) depth = k;
  }
  *out = depth;
  return 0;
}

static int make_hier(int nd, const uint64_t* dims, int levels, hier_t* h) {
  int feasible, rc = mo_max_levels(nd, dims, &feasible);
  if (rc) return rc;
  int L = levels < 0 ? feasible : levels;
  if (L > feasible) return E_DEPTH_EXCEEDED;
  if (L + 1 > MO_MAXL) return E_DEPTH_EXCEEDED;
  h->d = nd;
  h->L = L;
  for (int i = 0; i < nd; ++i) h->dims[L][i] = dims[i];
  for (int l = L - 1; l >= 0; --l)
    for (int i = 0; i < nd; ++i) h->dims[l][i] = (h->dims[l + 1][i] + 1) / 2;
  for (int l = 0; l <= L; ++l) {
    uint64_t c = 1;
    for (int i = 0; i < nd; ++i) c *= h->dims[l][i];
    h->node[l] = c;
    h->delta[l] = c - (l ? h->node[l - 1] : 0);
  }
  return 0;
}

int mo_hierarchy(int nd, const uint64_t* dims, int levels, int* out_levels, uint64_t* level_dims,
                 uint64_t* delta_counts) {
  hier_t* h = malloc(sizeof(hier_t));
  if (!h) return E_NOMEM;
  int rc = make_hier(nd, dims, levels, h);
  if (!rc) {
    *out_levels = h->L;
    for (int l = 0; l <= h->L; ++l) {
      if (level_dims)
        for (int i = 0; i < nd; ++i) level_dims[l * nd + i] = h->dims[l][i];
      if (delta_counts) delta_counts[l] = h->delta[l];
    }
  }
  free(h);
  return rc;
}

/* make_plan (quantize.cpp:7-24). mode 0 = uniform, 1 = levelwise. */
int mo_make_plan(int mode, double budget, int nd, const uint64_t* dims, int levels, double* q) {
  if (!(budget > 0.0) || !isfinite(budget)) return E_INVALID_BUDGET;
  hier_t* h = malloc(sizeof(hier_t));
  if (!h) return E_NOMEM;
  int rc = make_hier(nd, dims, levels, h);
  if (!rc) {
    const int L = h->L;
    if (mode == 0) {
      const double qq = 2.0 * budget / (double)(L + 1);
      for (int l = 0; l <= L; ++l) q[l] = qq;
    } else {
      const double total = (double)h->node[L];
      for (int l = 0; l <= L; ++l) q[l] = 2.0 * budget * (double)h->delta[l] / total;
    }
  }
  free(h);
  return rc;
}

/* ------------------------------------------------------ 1-D kernels -- */

/* load_entry (transform.hpp:84-96): five-point stencil, terms summed in
 * stencil order. c is the natural-order line, `step` its element stride. */
static double load_entry(const double* c, uint64_t step, uint64_t i, uint64_t n) {
  const uint64_t m = (n + 1) / 2;
  double acc = 0.0;
  if (i >= 1) {
    acc += (1.0 / 12.0) * c[(2 * i - 2) * step];
    acc += 0.5 * c[(2 * i - 1) * step];
  }
  acc += ((i == 0 || i + 1 == m) ? 5.0 / 12.0 : 5.0 / 6.0) * c[(2 * i) * step];
  if (2 * i + 1 < n) acc += 0.5 * c[(2 * i + 1) * step];
  if (2 * i + 2 < n) acc += (1.0 / 12.0) * c[(2 * i + 2) * step];
  return acc;
}

/* ThomasAux::build (transform.hpp:29-43). */
int mo_thomas_aux(uint64_t m, double* w, double* inv_d) {
  if (m < 2) return E_DEGENERATE_SYSTEM;
  double d = kDiagB;
  w[0] = 0.0;
  inv_d[0] = 1.0 / d;
  for (uint64_t i = 1; i < m; ++i) {
    const double wi = kOff / d;
    w[i] = wi;
    d = (i + 1 == m ? kDiagB : kDiagI) - wi * kOff;
    inv_d[i] = 1.0 / d;
  }
  return 0;
}

/* batched_solve with b = 1 (transform.hpp:116-130). */
static void thomas_solve(double* f, uint64_t m, const double* w, const double* inv_d) {
  for (uint64_t i = 1; i < m; ++i) f[i] -= w[i] * f[i - 1];
  f[m - 1] *= inv_d[m - 1];
  for (uint64_t i = m - 1; i-- > 0;) f[i] = (f[i] - kOff * f[i + 1]) * inv_d[i];
}

/* load_vector_1d (transform.hpp:136-143). */
int mo_load_vector_1d(const double* line, uint64_t n, double* out) {
  if (n < 3) return E_DEGENERATE_LINE;
  for (uint64_t i = 0; i < (n + 1) / 2; ++i) out[i] = load_entry(line, 1, i, n);
  return 0;
}

/* solve_correction_1d (transform.hpp:146-154). */
int mo_solve_correction_1d(double* f, uint64_t m) {
  if (m < 2) return E_DEGENERATE_SYSTEM;
  double* w = malloc(m * sizeof(double));
  double* inv = malloc(m * sizeof(double));
  if (!w || !inv) {
    free(w);
    free(inv);
    return E_NOMEM;
  }
  mo_thomas_aux(m, w, inv);
  thomas_solve(f, m, w, inv);
  free(w);
  free(inv);
  return 0;
}

/* ------------------------------------------- nonuniform axis tables --
 * No reference counterpart.  Finite-element restatement
 * with real spacings; every table reduces to the
 * reference's constants when the spacing is uniform:
 *   interpolation  linear weights (x_{j+1}-x_j)/(x_{j+1}-x_{j-1}) etc.
 *                  (uniform: the 1/2 of corner_average, transform.hpp:207-212;
 *                  a degenerate even-axis end keeps its single neighbour)
 *   load vector    fine mass matrix (h/6, (h_l+h_r)/3) then restriction by
 *                  the coarse hat values (uniform: 1/12,1/2,5/6|5/12,1/2,1/12,
 *                  transform.hpp:84-96; even-axis end term 1/2 -> h/2)
 *   coarse mass    diag (H_{i-1}+H_i)/3, off H_i/6 (uniform, h cancelled:
 *                  2/3, 4/3, 1/3, transform.hpp:17-21). */
typedef struct {
  uint64_t n, m;
  double* wl;  /* [n] interpolation weight of the left neighbour (odd j) */
  double* wr;  /* [n] ... of the right neighbour */
  double* s;   /* [m*5] load stencil for coarse i over fine 2i-2..2i+2 */
  double* tw;  /* [m] Thomas w_i */
  double* tid; /* [m] Thomas 1/d_i */
  double* off; /* [m] super-diagonal H_i/6 */
} nu_axis_t;

static void nu_free(nu_axis_t* a) {
  free(a->wl);
  free(a->wr);
  free(a->s);
  free(a->tw);
  free(a->tid);
  free(a->off);
  memset(a, 0, sizeof(*a));
}

/* x: the n coordinates of this level along the axis. */
static int nu_build(nu_axis_t* a, const double* x, uint64_t n) {
  const uint64_t m = (n + 1) / 2;
  a->n = n;
  a->m = m;
  a->wl = calloc(n, sizeof(double));
  a->wr = calloc(n, sizeof(double));
  a->s = calloc(m * 5, sizeof(double));
  a->tw = calloc(m, sizeof(double));
  a->tid = calloc(m, sizeof(double));
  a->off = calloc(m, sizeof(double));
  if (!a->wl || !a->wr || !a->s || !a->tw || !a->tid || !a->off) return E_NOMEM;
  for (uint64_t j = 1; j < n; j += 2) {
    if (j + 1 < n) {
      const double span = x[j + 1] - x[j - 1];
      a->wl[j] = (x[j + 1] - x[j]) / span;
      a->wr[j] = (x[j] - x[j - 1]) / span;
    } else {
      a->wl[j] = 1.0;
      a->wr[j] = 0.0;
    }
  }
  /* h_j = x_{j+1} - x_j, zero outside [0, n-1) */
#define H(j) (((j) >= 0 && (uint64_t)(j) + 1 < n) ? x[(j) + 1] - x[(j)] : 0.0)
  for (uint64_t i = 0; i < m; ++i) {
    const int64_t c = (int64_t)(2 * i);
    double* s = a->s + i * 5;
    const int even_end = (n % 2 == 0) && (i + 1 == m);
    /* coarse hat value at fine c-1 and c+1 */
    const double al = i > 0 ? H(c - 2) / (H(c - 2) + H(c - 1)) : 0.0;
    const double ar = (!even_end && i + 1 < m) ? H(c + 1) / (H(c) + H(c + 1)) : 0.0;
    if (i > 0) {
      s[0] = al * H(c - 2) / 6.0;
      s[1] = al * (H(c - 2) + H(c - 1)) / 3.0 + H(c - 1) / 6.0;
    }
    if (even_end) {
      s[2] = al * H(c - 1) / 6.0 + H(c - 1) / 3.0;
      s[3] = H(c) / 2.0;
    } else {
      s[2] = al * H(c - 1) / 6.0 + (H(c - 1) + H(c)) / 3.0 + ar * H(c) / 6.0;
      if (i + 1 < m) {
        s[3] = H(c) / 6.0 + ar * (H(c) + H(c + 1)) / 3.0;
        s[4] = ar * H(c + 1) / 6.0;
      }
    }
  }
#undef H
  /* coarse mass matrix on X_i = x_{2i} */
  double* Hc = calloc(m, sizeof(double));
  if (!Hc) return E_NOMEM;
  for (uint64_t i = 0; i + 1 < m; ++i) Hc[i] = x[2 * i + 2] - x[2 * i];
  double d = Hc[0] / 3.0;
  a->tw[0] = 0.0;
  a->tid[0] = 1.0 / d;
  for (uint64_t i = 0; i + 1 < m; ++i) a->off[i] = Hc[i] / 6.0;
  for (uint64_t i = 1; i < m; ++i) {
    const double wi = a->off[i - 1] / d;
    a->tw[i] = wi;
    const double diag = (Hc[i - 1] + (i + 1 < m ? Hc[i] : 0.0)) / 3.0;
    d = diag - wi * a->off[i - 1];
    a->tid[i] = 1.0 / d;
  }
  free(Hc);
  return 0;
}

static double nu_load_entry(const nu_axis_t* a, const double* c, uint64_t step, uint64_t i) {
  const double* s = a->s + i * 5;
  double acc = 0.0;
  for (int k = 0; k < 5; ++k) {
    const int64_t j = (int64_t)(2 * i) + k - 2;
    if (j < 0 || (uint64_t)j >= a->n) continue;
    acc += s[k] * c[(uint64_t)j * step];
  }
  return acc;
}

static void nu_thomas_solve(const nu_axis_t* a, double* f) {
  const uint64_t m = a->m;
  for (uint64_t i = 1; i < m; ++i) f[i] -= a->tw[i] * f[i - 1];
  f[m - 1] *= a->tid[m - 1];
  for (uint64_t i = m - 1; i-- > 0;) f[i] = (f[i] - a->off[i] * f[i + 1]) * a->tid[i];
}

int mo_load_vector_nu_1d(const double* line, const double* x, uint64_t n, double* out) {
  if (n < 3) return E_DEGENERATE_LINE;
  nu_axis_t a;
  memset(&a, 0, sizeof(a));
  int rc = nu_build(&a, x, n);
  if (!rc)
    for (uint64_t i = 0; i < a.m; ++i) out[i] = nu_load_entry(&a, line, 1, i);
  nu_free(&a);
  return rc;
}

/* X: the m coarse coordinates; builds a fine line whose even nodes are X. */
int mo_solve_correction_nu_1d(double* f, const double* X, uint64_t m) {
  if (m < 2) return E_DEGENERATE_SYSTEM;
  const uint64_t n = 2 * m - 1;
  double* x = malloc(n * sizeof(double));
  if (!x) return E_NOMEM;
  for (uint64_t i = 0; i < m; ++i) x[2 * i] = X[i];
  for (uint64_t i = 0; i + 1 < m; ++i) x[2 * i + 1] = 0.5 * (X[i] + X[i + 1]);
  nu_axis_t a;
  memset(&a, 0, sizeof(a));
  int rc = nu_build(&a, x, n);
  if (!rc) nu_thomas_solve(&a, f);
  nu_free(&a);
  free(x);
  return rc;
}

/* ------------------------------------------------- level machinery -- */

typedef struct {
  int d;
  uint64_t n[MO_MAXD], m[MO_MAXD];
  const nu_axis_t* nu; /* per-axis tables, or NULL for the uniform path */
} level_t;

static uint64_t count_of(const uint64_t* e, int d) {
  uint64_t c = 1;
  for (int i = 0; i < d; ++i) c *= e[i];
  return c;
}

static void unravel(uint64_t p, const uint64_t* e, int d, uint64_t* j) {
  for (int i = d - 1; i >= 0; --i) {
    j[i] = p % e[i];
    p /= e[i];
  }
}

static uint64_t ravel(const uint64_t* j, const uint64_t* e, int d) {
  uint64_t p = 0;
  for (int i = 0; i < d; ++i) p = p * e[i] + j[i];
  return p;
}

/* Position of a coefficient node inside its level's shell in the
 * level-centric buffer (pack_level_centric, reorder.hpp:180-215): row-major
 * over the reordered level block, rows whose leading reordered indices are
 * all nodal contribute only their coefficient tail [m_{d-1}, n_{d-1}). */
static uint64_t shell_pos(const level_t* lv, const uint64_t* j) {
  const int d = lv->d;
  uint64_t r[MO_MAXD];
  for (int i = 0; i < d; ++i) r[i] = (j[i] % 2 == 0) ? j[i] / 2 : lv->m[i] + j[i] / 2;
  uint64_t row = 0, before = 0;
  int inside = 1;
  for (int i = 0; i + 1 < d; ++i) row = row * lv->n[i] + r[i];
  for (int i = 0; i + 1 < d; ++i) {
    uint64_t p = 1;
    for (int k = i + 1; k + 1 < d; ++k) p *= lv->m[k];
    if (r[i] < lv->m[i]) {
      before += r[i] * p;
    } else {
      before += lv->m[i] * p;
      inside = 0;
      break;
    }
  }
  const uint64_t last = lv->n[d - 1], mlast = lv->m[d - 1];
  return row * last - before * mlast + (inside ? r[d - 1] - mlast : r[d - 1]);
}

/* Multilinear prediction at a node with natural coords j from nodal values.
 * src holds the nodal values: natural level block (coarse_idx = 0) or the
 * compact coarse block (coarse_idx = 1).  Uniform path: corner_average
 * (transform.hpp:206-212) with the corner enumeration of
 * update_coefficients (:223-301): set axes ascending, cmask ascending, the
 * single neighbour of a degenerate even-axis end counted twice. */
static double predict(const level_t* lv, const double* src, int coarse_idx, const uint64_t* j) {
  const int d = lv->d;
  int set[MO_MAXD], k = 0;
  for (int i = 0; i < d; ++i)
    if (j[i] % 2 == 1) set[k++] = i;
  const uint64_t* ext = coarse_idx ? lv->m : lv->n;
  double sum = 0.0;
  for (unsigned cm = 0; cm < (1u << k); ++cm) {
    uint64_t c[MO_MAXD];
    double wprod = 1.0;
    for (int i = 0; i < d; ++i) c[i] = j[i];
    for (int b = 0; b < k; ++b) {
      const int ax = set[b];
      const int right = (cm >> b) & 1u;
      c[ax] = (right && j[ax] + 1 < lv->n[ax]) ? j[ax] + 1 : j[ax] - 1;
      if (lv->nu) wprod *= right ? lv->nu[ax].wr[j[ax]] : lv->nu[ax].wl[j[ax]];
    }
    if (coarse_idx)
      for (int i = 0; i < d; ++i) c[i] /= 2;
    const double v = src[ravel(c, ext, d)];
    if (lv->nu)
      sum += wprod * v;
    else
      sum += v;
  }
  return lv->nu ? sum : sum * (1.0 / (double)(1u << k));
}

/* compute_correction (transform.hpp:331-431) on a natural-order component:
 * load + Thomas along axis 0, 1, ..., d-1 on the shrinking extents.  Returns
 * a malloc'd coarse-extent array (row-major). */
static double* correction(const level_t* lv, double* comp) {
  const int d = lv->d;
  uint64_t cur[MO_MAXD];
  for (int i = 0; i < d; ++i) cur[i] = lv->n[i];
  double* x = comp;
  for (int a = 0; a < d; ++a) {
    const uint64_t n = cur[a], m = lv->m[a];
    uint64_t outer = 1, inner = 1;
    for (int i = 0; i < a; ++i) outer *= cur[i];
    for (int i = a + 1; i < d; ++i) inner *= cur[i];
    double* y = malloc(outer * m * inner * sizeof(double));
    double* f = malloc(m * sizeof(double));
    double *w = NULL, *inv = NULL;
    if (!lv->nu) {
      w = malloc(m * sizeof(double));
      inv = malloc(m * sizeof(double));
      mo_thomas_aux(m, w, inv);
    }
    for (uint64_t o = 0; o < outer; ++o)
      for (uint64_t t = 0; t < inner; ++t) {
        const double* line = x + o * n * inner + t;
        for (uint64_t i = 0; i < m; ++i)
          f[i] = lv->nu ? nu_load_entry(&lv->nu[a], line, inner, i) : load_entry(line, inner, i, n);
        if (lv->nu)
          nu_thomas_solve(&lv->nu[a], f);
        else
          thomas_solve(f, m, w, inv);
        for (uint64_t i = 0; i < m; ++i) y[(o * m + i) * inner + t] = f[i];
      }
    free(f);
    free(w);
    free(inv);
    if (x != comp) free(x);
    x = y;
    cur[a] = m;
  }
  return x;
}

static int build_nu_level(const hier_t* h, int l, const double* const* coords, nu_axis_t* axes) {
  const int L = h->L;
  for (int a = 0; a < h->d; ++a) {
    const uint64_t n = h->dims[l][a];
    const uint64_t stride = (uint64_t)1 << (L - l);
    double* x = malloc(n * sizeof(double));
    if (!x) return E_NOMEM;
    for (uint64_t j = 0; j < n; ++j) x[j] = coords[a][j * stride];
    int rc = nu_build(&axes[a], x, n);
    free(x);
    if (rc) return rc;
  }
  return 0;
}

static int check_coords(const hier_t* h, const double* const* coords) {
  if (!coords) return 0;
  for (int a = 0; a < h->d; ++a)
    for (uint64_t j = 0; j + 1 < h->dims[h->L][a]; ++j)
      if (!(coords[a][j + 1] > coords[a][j])) return E_INVALID_INPUT;
  return 0;
}

/* decompose (transform.hpp:509-515 -> decompose_with :485-506): per level
 * reorder + compute_coefficients + compute_correction + apply_correction(+1),
 * then pack_level_centric (reorder.hpp:162). */
static int decompose_core(int nd, const uint64_t* dims, int levels, int stop, const double* in,
                          double* out, int f32, const double* const* coords) {
  hier_t* h = malloc(sizeof(hier_t));
  if (!h) return E_NOMEM;
  int rc = make_hier(nd, dims, levels, h);
  if (!rc && (stop < 0 || stop > h->L)) rc = E_INVALID_LEVEL;
  if (!rc) rc = check_coords(h, coords);
  if (rc) {
    free(h);
    return rc;
  }
  const int L = h->L, d = nd;
  double* blk = malloc(h->node[L] * sizeof(double));
  memcpy(blk, in, h->node[L] * sizeof(double));
  for (int l = L; l > stop; --l) {
    level_t lv;
    nu_axis_t axes[MO_MAXD];
    memset(axes, 0, sizeof(axes));
    lv.d = d;
    for (int i = 0; i < d; ++i) {
      lv.n[i] = h->dims[l][i];
      lv.m[i] = h->dims[l - 1][i];
    }
    lv.nu = NULL;
    if (coords) {
      rc = build_nu_level(h, l, coords, axes);
      lv.nu = axes;
    }
    const uint64_t nl = h->node[l], nc = h->node[l - 1];
    double* comp = calloc(nl, sizeof(double));
    double* next = malloc(nc * sizeof(double));
    double* shell = out + h->node[l - 1];
    for (uint64_t p = 0; p < nl && !rc; ++p) {
      uint64_t j[MO_MAXD];
      unravel(p, lv.n, d, j);
      int nodal = 1;
      for (int i = 0; i < d; ++i) nodal &= (j[i] % 2 == 0);
      if (nodal) {
        uint64_t c[MO_MAXD];
        for (int i = 0; i < d; ++i) c[i] = j[i] / 2;
        next[ravel(c, lv.m, d)] = blk[p];
      } else {
        const double v = rt(blk[p] - predict(&lv, blk, 0, j), f32);
        comp[p] = v;
        shell[shell_pos(&lv, j)] = v;
      }
    }
    if (!rc) {
      double* z = correction(&lv, comp);
      for (uint64_t x = 0; x < nc; ++x) next[x] = rt(next[x] + z[x], f32);
      free(z);
    }
    free(comp);
    free(blk);
    blk = next;
    for (int a = 0; a < d; ++a) nu_free(&axes[a]);
    if (rc) break;
  }
  if (!rc) memcpy(out, blk, h->node[stop] * sizeof(double));
  free(blk);
  free(h);
  return rc;
}

/* recompose (transform.hpp:517-530): unpack, then per level
 * compute_correction, apply_correction(-1), add_interpolant, inverse
 * reorder. */
static int recompose_core(int nd, const uint64_t* dims, int levels, int stop, const double* in,
                          double* out, int f32, const double* const* coords) {
  hier_t* h = malloc(sizeof(hier_t));
  if (!h) return E_NOMEM;
  int rc = make_hier(nd, dims, levels, h);
  if (!rc && (stop < 0 || stop > h->L)) rc = E_INVALID_LEVEL;
  if (!rc) rc = check_coords(h, coords);
  if (rc) {
    free(h);
    return rc;
  }
  const int L = h->L, d = nd;
  double* cur = malloc(h->node[stop] * sizeof(double));
  memcpy(cur, in, h->node[stop] * sizeof(double));
  for (int l = stop + 1; l <= L && !rc; ++l) {
    level_t lv;
    nu_axis_t axes[MO_MAXD];
    memset(axes, 0, sizeof(axes));
    lv.d = d;
    for (int i = 0; i < d; ++i) {
      lv.n[i] = h->dims[l][i];
      lv.m[i] = h->dims[l - 1][i];
    }
    lv.nu = NULL;
    if (coords) {
      rc = build_nu_level(h, l, coords, axes);
      lv.nu = axes;
    }
    const uint64_t nl = h->node[l], nc = h->node[l - 1];
    const double* shell = in + h->node[l - 1];
    double* comp = calloc(nl, sizeof(double));
    for (uint64_t p = 0; p < nl; ++p) {
      uint64_t j[MO_MAXD];
      unravel(p, lv.n, d, j);
      int nodal = 1;
      for (int i = 0; i < d; ++i) nodal &= (j[i] % 2 == 0);
      if (!nodal) comp[p] = shell[shell_pos(&lv, j)];
    }
    double* z = correction(&lv, comp);
    for (uint64_t x = 0; x < nc; ++x) cur[x] = rt(cur[x] - z[x], f32);
    free(z);
    double* fine = malloc(nl * sizeof(double));
    for (uint64_t p = 0; p < nl; ++p) {
      uint64_t j[MO_MAXD], c[MO_MAXD];
      unravel(p, lv.n, d, j);
      int nodal = 1;
      for (int i = 0; i < d; ++i) nodal &= (j[i] % 2 == 0);
      if (nodal) {
        for (int i = 0; i < d; ++i) c[i] = j[i] / 2;
        fine[p] = cur[ravel(c, lv.m, d)];
      } else {
        fine[p] = rt(comp[p] + predict(&lv, cur, 1, j), f32);
      }
    }
    free(comp);
    free(cur);
    cur = fine;
    for (int a = 0; a < d; ++a) nu_free(&axes[a]);
  }
  if (!rc) memcpy(out, cur, h->node[L] * sizeof(double));
  free(cur);
  free(h);
  return rc;
}

static uint64_t total_of(int nd, const uint64_t* dims) { return count_of(dims, nd > 0 ? nd : 0); }

static double* widen_f32(const float* in, uint64_t n) {
  double* d = malloc(n * sizeof(double));
  if (d)
    for (uint64_t i = 0; i < n; ++i) d[i] = (double)in[i];
  return d;
}

static void narrow_f32(const double* in, uint64_t n, float* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = (float)in[i];
}

int mo_decompose_f64(int nd, const uint64_t* dims, int levels, int stop, const double* in, double* out) {
  return decompose_core(nd, dims, levels, stop, in, out, 0, NULL);
}
int mo_recompose_f64(int nd, const uint64_t* dims, int levels, int stop, const double* in, double* out) {
  return recompose_core(nd, dims, levels, stop, in, out, 0, NULL);
}
int mo_decompose_nu_f64(int nd, const uint64_t* dims, int levels, int stop, const double* const* coords,
                        const double* in, double* out) {
  return decompose_core(nd, dims, levels, stop, in, out, 0, coords);
}
int mo_recompose_nu_f64(int nd, const uint64_t* dims, int levels, int stop, const double* const* coords,
                        const double* in, double* out) {
  return recompose_core(nd, dims, levels, stop, in, out, 0, coords);
}

static int f32_wrap(int dec, int nd, const uint64_t* dims, int levels, int stop, const double* const* coords,
                    const float* in, float* out) {
  if (nd <= 0 || nd > MO_MAXD) return E_INVALID_DIMS;
  const uint64_t n = total_of(nd, dims);
  double* a = widen_f32(in, n);
  double* b = malloc(n * sizeof(double));
  if (!a || !b) {
    free(a);
    free(b);
    return E_NOMEM;
  }
  int rc = dec ? decompose_core(nd, dims, levels, stop, a, b, 1, coords)
               : recompose_core(nd, dims, levels, stop, a, b, 1, coords);
  if (!rc) narrow_f32(b, n, out);
  free(a);
  free(b);
  return rc;
}

int mo_decompose_f32(int nd, const uint64_t* dims, int levels, int stop, const float* in, float* out) {
  return f32_wrap(1, nd, dims, levels, stop, NULL, in, out);
}
int mo_recompose_f32(int nd, const uint64_t* dims, int levels, int stop, const float* in, float* out) {
  return f32_wrap(0, nd, dims, levels, stop, NULL, in, out);
}
int mo_decompose_nu_f32(int nd, const uint64_t* dims, int levels, int stop, const double* const* coords,
                        const float* in, float* out) {
  return f32_wrap(1, nd, dims, levels, stop, coords, in, out);
}
int mo_recompose_nu_f32(int nd, const uint64_t* dims, int levels, int stop, const double* const* coords,
                        const float* in, float* out) {
  return f32_wrap(0, nd, dims, levels, stop, coords, in, out);
}

/* --------------------------------------------------------- quantize --
 * quantize / quantize_tail (quantize.hpp:58-114): r = nearbyint(v / q_l)
 * (IEEE division, ties to even); outside [-32768, 32767] -> outlier
 * {position, value} + label 0; non-finite -> nonfinite_data.  labels is the
 * concatenation of the per-level vectors (levels stop+1..L for a tail). */
static int quantize_core(int nd, const uint64_t* dims, int levels, int stop, const double* q,
                         const double* c, int32_t* labels, uint64_t* opos, double* oval, uint64_t cap,
                         uint64_t* n_out) {
  hier_t* h = malloc(sizeof(hier_t));
  if (!h) return E_NOMEM;
  int rc = make_hier(nd, dims, levels, h);
  if (!rc && (stop < 0 || stop > h->L)) rc = E_INVALID_LEVEL;
  if (rc) {
    free(h);
    return rc;
  }
  uint64_t pos = stop == 0 ? 0 : h->node[stop];
  uint64_t lp = 0, no = 0;
  for (int l = stop == 0 ? 0 : stop + 1; l <= h->L; ++l) {
    const double ql = q[l];
    for (uint64_t i = 0; i < h->delta[l]; ++i, ++pos, ++lp) {
      const double v = c[pos];
      if (!isfinite(v)) {
        free(h);
        return E_NONFINITE;
      }
      const double r = nearbyint(v / ql);
      if (r < -32768.0 || r > 32767.0) {
        if (no < cap) {
          opos[no] = pos;
          oval[no] = v;
        }
        ++no;
        labels[lp] = 0;
      } else {
        labels[lp] = (int32_t)r;
      }
    }
  }
  *n_out = no;
  free(h);
  return 0;
}

/* dequantize / dequantize_tail (quantize.hpp:118-150). */
static int dequantize_core(int nd, const uint64_t* dims, int levels, int stop, const double* q,
                           const int32_t* labels, const uint64_t* opos, const double* oval, uint64_t n_out,
                           double* c, int f32) {
  hier_t* h = malloc(sizeof(hier_t));
  if (!h) return E_NOMEM;
  int rc = make_hier(nd, dims, levels, h);
  if (!rc && (stop < 0 || stop > h->L)) rc = E_INVALID_LEVEL;
  if (rc) {
    free(h);
    return rc;
  }
  uint64_t pos = stop == 0 ? 0 : h->node[stop], lp = 0;
  for (int l = stop == 0 ? 0 : stop + 1; l <= h->L; ++l)
    for (uint64_t i = 0; i < h->delta[l]; ++i, ++pos, ++lp) c[pos] = rt((double)labels[lp] * q[l], f32);
  for (uint64_t i = 0; i < n_out; ++i) c[opos[i]] = oval[i];
  free(h);
  return 0;
}

int mo_quantize_f64(int nd, const uint64_t* dims, int levels, int stop, const double* q, const double* c,
                    int32_t* labels, uint64_t* opos, double* oval, uint64_t cap, uint64_t* n_out) {
  return quantize_core(nd, dims, levels, stop, q, c, labels, opos, oval, cap, n_out);
}

int mo_quantize_f32(int nd, const uint64_t* dims, int levels, int stop, const double* q, const float* c,
                    int32_t* labels, uint64_t* opos, float* oval, uint64_t cap, uint64_t* n_out) {
  if (nd <= 0 || nd > MO_MAXD) return E_INVALID_DIMS;
  const uint64_t n = total_of(nd, dims);
  double* a = widen_f32(c, n);
  double* ov = malloc((cap ? cap : 1) * sizeof(double));
  if (!a || !ov) {
    free(a);
    free(ov);
    return E_NOMEM;
  }
  int rc = quantize_core(nd, dims, levels, stop, q, a, labels, opos, ov, cap, n_out);
  if (!rc)
    for (uint64_t i = 0; i < *n_out && i < cap; ++i) oval[i] = (float)ov[i];
  free(a);
  free(ov);
  return rc;
}

int mo_dequantize_f64(int nd, const uint64_t* dims, int levels, int stop, const double* q,
                      const int32_t* labels, const uint64_t* opos, const double* oval, uint64_t n_out,
                      double* c) {
  return dequantize_core(nd, dims, levels, stop, q, labels, opos, oval, n_out, c, 0);
}

int mo_dequantize_f32(int nd, const uint64_t* dims, int levels, int stop, const double* q,
                      const int32_t* labels, const uint64_t* opos, const float* oval, uint64_t n_out,
                      float* c) {
  if (nd <= 0 || nd > MO_MAXD) return E_INVALID_DIMS;
  const uint64_t n = total_of(nd, dims);
  double* a = widen_f32(c, n);
  double* ov = malloc((n_out ? n_out : 1) * sizeof(double));
  if (!a || !ov) {
    free(a);
    free(ov);
    return E_NOMEM;
  }
  for (uint64_t i = 0; i < n_out; ++i) ov[i] = (double)oval[i];
  int rc = dequantize_core(nd, dims, levels, stop, q, labels, opos, ov, n_out, a, 1);
  if (!rc) narrow_f32(a, n, c);
  free(a);
  free(ov);
  return rc;
}
