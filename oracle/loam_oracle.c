/*
 * loam_oracle.c -- CPU restatement of the reference par_loop hot path.
 * TEST INFRASTRUCTURE ONLY (see loam_oracle.h for the usage rule and pins).
 *
 * Reference: /root/reference/proj/include/loam (C++20).  Citations are
 * file:line into that tree.
 */
#include "loam_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

void orc_free(void* p) { free(p); }

/* ======================================================================== */
/* Colouring: topology.hpp:86-125                                            */
/* ======================================================================== */

int orc_color_iteration(int n, int nmaps, const int32_t* const* maps, const int32_t* arity,
                        const int32_t* target_size, int32_t* colors) {
  /* colors_at[m][t] is kept as a bitset of `words` 64-bit words per target
   * (the reference keeps a vector<int> per target; membership is the same). */
  int words = 1;
  uint64_t** at = (uint64_t**)calloc((size_t)(nmaps > 0 ? nmaps : 1), sizeof(uint64_t*));
  for (int m = 0; m < nmaps; ++m)
    at[m] = (uint64_t*)calloc((size_t)target_size[m] * words, sizeof(uint64_t));
  int num_colors = 0;
  uint64_t* forbidden = (uint64_t*)calloc(1, sizeof(uint64_t));
  for (int e = 0; e < n; ++e) {
    memset(forbidden, 0, sizeof(uint64_t) * words);
    for (int m = 0; m < nmaps; ++m) {
      const int32_t* tuple = maps[m] + (int64_t)e * arity[m];
      for (int k = 0; k < arity[m]; ++k) {
        const uint64_t* set = at[m] + (int64_t)tuple[k] * words;
        for (int w = 0; w < words; ++w) forbidden[w] |= set[w];
      }
    }
    int color = 0;
    while (color < 64 * words && (forbidden[color >> 6] >> (color & 63) & 1u)) ++color;
    colors[e] = color;
    if (color >= num_colors) num_colors = color + 1;
    if (num_colors > 64 * words) { /* grow every bitset by one word */
      int nw = words + 1;
      for (int m = 0; m < nmaps; ++m) {
        uint64_t* grown = (uint64_t*)calloc((size_t)target_size[m] * nw, sizeof(uint64_t));
        for (int64_t t = 0; t < target_size[m]; ++t)
          memcpy(grown + t * nw, at[m] + t * words, sizeof(uint64_t) * words);
        free(at[m]);
        at[m] = grown;
      }
      forbidden = (uint64_t*)realloc(forbidden, sizeof(uint64_t) * nw);
      words = nw;
    }
    for (int m = 0; m < nmaps; ++m) {
      const int32_t* tuple = maps[m] + (int64_t)e * arity[m];
      for (int k = 0; k < arity[m]; ++k)
        at[m][(int64_t)tuple[k] * words + (color >> 6)] |= (uint64_t)1 << (color & 63);
    }
  }
  for (int m = 0; m < nmaps; ++m) free(at[m]);
  free(at);
  free(forbidden);
  return num_colors;
}

/* ======================================================================== */
/* Sparsity: data.hpp:149-179                                                */
/* ======================================================================== */

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

int64_t orc_build_sparsity(int nsrc, const int32_t* row_map, int ar_r, int nrt,
                           const int32_t* col_map, int ar_c, int nct, int row_dim, int col_dim,
                           int64_t** row_ptr_out, int32_t** col_idx_out) {
  (void)nct;
  /* The reference pushes cn[b]*col_dim+cd into rows[rn[a]*row_dim+rd]
   * (data.hpp:157-166).  All row_dim sub-rows of a node see the same node
   * set and each node m expands to the ascending run m*col_dim+[0,col_dim),
   * so collecting per node row and expanding afterwards yields the identical
   * sorted/unique rows (data.hpp:169-174). */
  int64_t* cnt = (int64_t*)calloc((size_t)nrt + 1, sizeof(int64_t));
  for (int64_t e = 0; e < nsrc; ++e)
    for (int a = 0; a < ar_r; ++a) cnt[row_map[e * ar_r + a] + 1] += ar_c;
  for (int r = 0; r < nrt; ++r) cnt[r + 1] += cnt[r];
  int32_t* buf = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cnt[nrt] > 0 ? cnt[nrt] : 1));
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nrt > 0 ? nrt : 1));
  for (int r = 0; r < nrt; ++r) fill[r] = cnt[r];
  for (int64_t e = 0; e < nsrc; ++e)
    for (int a = 0; a < ar_r; ++a) {
      int r = row_map[e * ar_r + a];
      for (int b = 0; b < ar_c; ++b) buf[fill[r]++] = col_map[e * ar_c + b];
    }
  /* sort + unique per node row */
  int64_t* ulen = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nrt > 0 ? nrt : 1));
  for (int r = 0; r < nrt; ++r) {
    int32_t* row = buf + cnt[r];
    int64_t len = cnt[r + 1] - cnt[r];
    qsort(row, (size_t)len, sizeof(int32_t), cmp_i32);
    int64_t u = 0;
    for (int64_t k = 0; k < len; ++k)
      if (u == 0 || row[u - 1] != row[k]) row[u++] = row[k];
    ulen[r] = u;
  }
  const int64_t nrows = (int64_t)nrt * row_dim;
  int64_t* rp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nrows + 1));
  rp[0] = 0;
  for (int r = 0; r < nrt; ++r)
    for (int rd = 0; rd < row_dim; ++rd) {
      int64_t i = (int64_t)r * row_dim + rd;
      rp[i + 1] = rp[i] + ulen[r] * col_dim;
    }
  const int64_t nnz = rp[nrows];
  int32_t* ci = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
  for (int r = 0; r < nrt; ++r)
    for (int rd = 0; rd < row_dim; ++rd) {
      int64_t pos = rp[(int64_t)r * row_dim + rd];
      for (int64_t k = 0; k < ulen[r]; ++k)
        for (int cd = 0; cd < col_dim; ++cd) ci[pos++] = buf[cnt[r] + k] * col_dim + cd;
    }
  free(cnt);
  free(buf);
  free(fill);
  free(ulen);
  *row_ptr_out = rp;
  *col_idx_out = ci;
  return nnz;
}

int64_t orc_sparsity_find(const int64_t* row_ptr, const int32_t* col_idx, int nrows, int row,
                          int col) {
  if (row < 0 || row >= nrows) return -1;
  int64_t lo = row_ptr[row], hi = row_ptr[row + 1];
  while (lo < hi) { /* std::lower_bound */
    int64_t mid = lo + (hi - lo) / 2;
    if (col_idx[mid] < col) lo = mid + 1;
    else hi = mid;
  }
  if (lo == row_ptr[row + 1] || col_idx[lo] != col) return -1;
  return lo;
}

/* ======================================================================== */
/* P2 spaces: space.hpp:48-72 (triangles); tet extension                     */
/* ======================================================================== */

static int cmp_edge(const void* a, const void* b) {
  const int32_t* x = (const int32_t*)a;
  const int32_t* y = (const int32_t*)b;
  if (x[0] != y[0]) return (x[0] > y[0]) - (x[0] < y[0]);
  return (x[1] > y[1]) - (x[1] < y[1]);
}

/* local edge (vertex pair) list per cell, in cell-node-row order */
static const int TRI_EDGES[3][2] = {{1, 2}, {0, 2}, {0, 1}};                         /* space.hpp:66-71 */
static const int TET_EDGES[6][2] = {{2, 3}, {1, 3}, {1, 2}, {0, 3}, {0, 2}, {0, 1}}; /* extension */

int orc_p2_cell_node_map(int ncells, int nv, int gdim, const int32_t* cv, int32_t* cn) {
  const int nvc = gdim + 1;
  const int ne = gdim == 2 ? 3 : 6;
  const int (*edges)[2] = gdim == 2 ? TRI_EDGES : TET_EDGES;
  const int64_t total = (int64_t)ncells * ne;
  int32_t* keys = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)(total > 0 ? total : 1));
  for (int64_t c = 0; c < ncells; ++c)
    for (int k = 0; k < ne; ++k) {
      int32_t a = cv[c * nvc + edges[k][0]], b = cv[c * nvc + edges[k][1]];
      keys[2 * (c * ne + k)] = a < b ? a : b;
      keys[2 * (c * ne + k) + 1] = a < b ? b : a;
    }
  /* std::set<pair<int,int>> iteration order = lexicographic (space.hpp:51-57) */
  qsort(keys, (size_t)total, 2 * sizeof(int32_t), cmp_edge);
  int64_t u = 0;
  for (int64_t k = 0; k < total; ++k)
    if (u == 0 || cmp_edge(keys + 2 * (u - 1), keys + 2 * k) != 0) {
      keys[2 * u] = keys[2 * k];
      keys[2 * u + 1] = keys[2 * k + 1];
      ++u;
    }
  const int row = nvc + ne;
  for (int64_t c = 0; c < ncells; ++c) {
    for (int v = 0; v < nvc; ++v) cn[c * row + v] = cv[c * nvc + v];
    for (int k = 0; k < ne; ++k) {
      int32_t a = cv[c * nvc + edges[k][0]], b = cv[c * nvc + edges[k][1]];
      int32_t key[2] = {a < b ? a : b, a < b ? b : a};
      int64_t lo = 0, hi = u;
      while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (cmp_edge(keys + 2 * mid, key) < 0) lo = mid + 1;
        else hi = mid;
      }
      cn[c * row + nvc + k] = (int32_t)(nv + lo);
    }
  }
  free(keys);
  return (int)(nv + u);
}

/* ======================================================================== */
/* Quadrature: element.hpp:75-149 (+ the 14-point degree-5 tet rule)         */
/* ======================================================================== */

#define MAXQ 16
typedef struct {
  int nq;
  double pts[MAXQ][3];
  double w[MAXQ];
} rule_t;

static void tri_orbit(rule_t* r, double a, double b, double w) { /* element.hpp:48-54 */
  const double bary[3][3] = {{a, b, b}, {b, a, b}, {b, b, a}};
  for (int k = 0; k < 3; ++k) {
    r->pts[r->nq][0] = bary[k][1];
    r->pts[r->nq][1] = bary[k][2];
    r->w[r->nq++] = w;
  }
}
static void tri_point(rule_t* r, double l1, double l2, double w) { /* element.hpp:56-60 */
  r->pts[r->nq][0] = l1;
  r->pts[r->nq][1] = l2;
  r->w[r->nq++] = w;
}
static void tet_orbit(rule_t* r, double a, double b, double w) { /* element.hpp:62-68 */
  const double bary[4][4] = {{a, b, b, b}, {b, a, b, b}, {b, b, a, b}, {b, b, b, a}};
  for (int k = 0; k < 4; ++k) {
    r->pts[r->nq][0] = bary[k][1];
    r->pts[r->nq][1] = bary[k][2];
    r->pts[r->nq][2] = bary[k][3];
    r->w[r->nq++] = w;
  }
}

/* 14-point rule exact to degree 5 (tools/tet_rule14.py). */
static void tet_rule14(rule_t* r) {
  const double b1 = 0.0927352503108912, b2 = 0.3108859192633006, c = 0.4544962958743504;
  const double w1 = 0.01224884051939366, w2 = 0.01878132095300264, w3 = 0.007091003462846911;
  tet_orbit(r, 1.0 - 3.0 * b1, b1, w1);
  tet_orbit(r, 1.0 - 3.0 * b2, b2, w2);
  const double d = 0.5 - c;
  const double six[6][4] = {{c, c, d, d}, {c, d, c, d}, {c, d, d, c},
                            {d, c, c, d}, {d, c, d, c}, {d, d, c, c}};
  for (int k = 0; k < 6; ++k) {
    r->pts[r->nq][0] = six[k][1];
    r->pts[r->nq][1] = six[k][2];
    r->pts[r->nq][2] = six[k][3];
    r->w[r->nq++] = w3;
  }
}

static void quadrature_rule(int gdim, int degree, rule_t* r) {
  r->nq = 0;
  if (gdim == 2) {
    if (degree <= 1) tri_point(r, 1.0 / 3, 1.0 / 3, 0.5);
    else if (degree == 2) tri_orbit(r, 2.0 / 3, 1.0 / 6, 1.0 / 6);
    else if (degree == 3) {
      tri_orbit(r, 0.0, 0.5, 1.0 / 60);
      tri_orbit(r, 2.0 / 3, 1.0 / 6, 3.0 / 20);
    } else {
      tri_orbit(r, 0.108103018168070, 0.445948490915965, 0.223381589678011 / 2);
      tri_orbit(r, 0.816847572980459, 0.091576213509771, 0.109951743655322 / 2);
    }
    return;
  }
  if (degree <= 1) {
    r->pts[0][0] = r->pts[0][1] = r->pts[0][2] = 0.25;
    r->w[0] = 1.0 / 6;
    r->nq = 1;
  } else if (degree == 2) {
    const double a = (5.0 + 3.0 * sqrt(5.0)) / 20.0;
    const double b = (5.0 - sqrt(5.0)) / 20.0;
    tet_orbit(r, a, b, 1.0 / 24);
  } else if (degree == 3) {
    tet_orbit(r, 0.0, 1.0 / 3, 3.0 / 200);
    tet_orbit(r, 5.0 / 8, 1.0 / 8, 2.0 / 75);
  } else {
    tet_rule14(r); /* degree 4 requested by config 3; not in the reference */
  }
}

/* ======================================================================== */
/* Lagrange basis: element.hpp:196-235 (+ P2 tet extension)                  */
/* ======================================================================== */

static int nbasis(int gdim, int degree) {
  if (degree == 1) return gdim + 1;
  return gdim == 2 ? 6 : 10;
}

static double bary_grad(int li, int dir) { return li == 0 ? -1.0 : (li == dir + 1 ? 1.0 : 0.0); }

static void edge_of(int gdim, int i, int* j, int* k) {
  const int nv = gdim + 1;
  if (gdim == 2) { /* edge node opposite vertex o: (o+1)%3,(o+2)%3 (element.hpp:219-221) */
    int o = i - nv;
    *j = (o + 1) % nv;
    *k = (o + 2) % nv;
  } else {
    *j = TET_EDGES[i - nv][0];
    *k = TET_EDGES[i - nv][1];
  }
}

static double eval_basis(int gdim, int degree, int i, const double* x) {
  double l[4];
  l[0] = 1.0;
  for (int k = 0; k < gdim; ++k) {
    l[0] -= x[k];
    l[k + 1] = x[k];
  }
  const int nv = gdim + 1;
  if (degree == 1) return l[i];
  if (i < nv) return l[i] * (2.0 * l[i] - 1.0);
  int j, k;
  edge_of(gdim, i, &j, &k);
  return 4.0 * l[j] * l[k];
}

static double eval_basis_grad(int gdim, int degree, int i, const double* x, int d) {
  double l[4];
  l[0] = 1.0;
  for (int k = 0; k < gdim; ++k) {
    l[0] -= x[k];
    l[k + 1] = x[k];
  }
  const int nv = gdim + 1;
  if (degree == 1) return bary_grad(i, d);
  if (i < nv) return (4.0 * l[i] - 1.0) * bary_grad(i, d);
  int j, k;
  edge_of(gdim, i, &j, &k);
  return 4.0 * (l[k] * bary_grad(j, d) + l[j] * bary_grad(k, d));
}

typedef struct {
  int nq, nbf, gdim;
  double P[MAXQ][10];
  double D[3][MAXQ][10];
} tab_t;

static void tabulate(int gdim, int degree, const rule_t* r, tab_t* t) { /* element.hpp:247-264 */
  t->nq = r->nq;
  t->nbf = nbasis(gdim, degree);
  t->gdim = gdim;
  for (int q = 0; q < r->nq; ++q)
    for (int i = 0; i < t->nbf; ++i) {
      t->P[q][i] = eval_basis(gdim, degree, i, r->pts[q]);
      for (int d = 0; d < gdim; ++d) t->D[d][q][i] = eval_basis_grad(gdim, degree, i, r->pts[q], d);
    }
}

/* ======================================================================== */
/* Geometry: form.hpp:139-178                                                */
/* ======================================================================== */

typedef struct {
  double detJ, adetJ, K[3][3];
} geom_t;

static void geometry(int gdim, const double* X, geom_t* g) {
  double J[3][3];
  for (int a = 0; a < gdim; ++a)
    for (int b = 0; b < gdim; ++b) J[a][b] = X[(b + 1) * gdim + a] - X[a];
  if (gdim == 2) {
    g->detJ = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    g->K[0][0] = J[1][1] / g->detJ;
    g->K[0][1] = -(J[1][0] / g->detJ);
    g->K[1][0] = -(J[0][1] / g->detJ);
    g->K[1][1] = J[0][0] / g->detJ;
  } else {
    double c[3][3];
    c[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    c[0][1] = -(J[1][0] * J[2][2] - J[1][2] * J[2][0]);
    c[0][2] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    g->detJ = J[0][0] * c[0][0] + J[0][1] * c[0][1] + J[0][2] * c[0][2];
    c[1][0] = -(J[0][1] * J[2][2] - J[0][2] * J[2][1]);
    c[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    c[1][2] = -(J[0][0] * J[2][1] - J[0][1] * J[2][0]);
    c[2][0] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    c[2][1] = -(J[0][0] * J[1][2] - J[0][2] * J[1][0]);
    c[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) g->K[a][b] = c[a][b] / g->detJ;
  }
  g->adetJ = sqrt(g->detJ * g->detJ); /* form.hpp:157 */
}

/* physical gradient component a of basis i at q: sum_b K_ab D_b[q][i] (form.hpp:193-199) */
static double pgrad(const geom_t* g, const tab_t* t, int a, int q, int i) {
  double acc = g->K[a][0] * t->D[0][q][i];
  for (int b = 1; b < t->gdim; ++b) acc += g->K[a][b] * t->D[b][q][i];
  return acc;
}

/* form.hpp:117-121 */
static int form_degree(int form, int p) {
  switch (form) {
  case ORC_STIFFNESS:
  case ORC_STIFFNESS_ACTION: return 2 * (p - 1) > 1 ? 2 * (p - 1) : 1;
  case ORC_ELASTICITY: return 1;     /* constant integrand */
  case ORC_STOKES_A: return 2;       /* P2 gradients: degree 2 */
  case ORC_STOKES_B:
  case ORC_STOKES_BT: return 2;      /* P1 x grad P2 */
  default: return 2 * p;
  }
}

int orc_element_shape(int form, int degree, int gdim, int* rows, int* cols) {
  int m = nbasis(gdim, degree);
  switch (form) {
  case ORC_MASS:
  case ORC_STIFFNESS:
  case ORC_HELMHOLTZ: *rows = m; *cols = m; return 0;
  case ORC_MASS_ACTION:
  case ORC_STIFFNESS_ACTION:
  case ORC_HELMHOLTZ_ACTION: *rows = m; *cols = 1; return 0;
  case ORC_ELASTICITY:
    if (gdim != 3 || degree != 1) return ORC_ERR_UNSUPPORTED_FORM;
    *rows = 12; *cols = 12; return 0;
  case ORC_STOKES_A:
    if (gdim != 2 || degree != 2) return ORC_ERR_UNSUPPORTED_FORM;
    *rows = 12; *cols = 12; return 0;
  case ORC_STOKES_B:
    if (gdim != 2 || degree != 2) return ORC_ERR_UNSUPPORTED_FORM;
    *rows = 3; *cols = 12; return 0;
  case ORC_STOKES_BT:
    if (gdim != 2 || degree != 2) return ORC_ERR_UNSUPPORTED_FORM;
    *rows = 12; *cols = 3; return 0;
  default: return ORC_ERR_UNSUPPORTED_FORM;
  }
}

int orc_element(int form, int degree, int gdim, const double* params, const double* X,
                const double* C, double* out) {
  int rows, cols;
  int err = orc_element_shape(form, degree, gdim, &rows, &cols);
  if (err) return err;
  if (!(gdim == 2 || gdim == 3) || !(degree == 1 || degree == 2)) return ORC_ERR_UNSUPPORTED_FORM;
  memset(out, 0, sizeof(double) * (size_t)rows * cols);
  geom_t g;
  geometry(gdim, X, &g);
  rule_t r;
  quadrature_rule(gdim, form_degree(form, degree), &r);
  tab_t t;
  tabulate(gdim, degree, &r, &t);
  const int m = t.nbf;

  switch (form) {
  case ORC_MASS:
  case ORC_STIFFNESS:
  case ORC_HELMHOLTZ: /* form.hpp:263-283 */
    for (int q = 0; q < r.nq; ++q) {
      const double scale = r.w[q] * g.adetJ;
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) {
          double integrand = 0.0;
          if (form == ORC_MASS) {
            integrand = t.P[q][i] * t.P[q][j];
          } else {
            integrand = pgrad(&g, &t, 0, q, i) * pgrad(&g, &t, 0, q, j);
            for (int a = 1; a < gdim; ++a) integrand += pgrad(&g, &t, a, q, i) * pgrad(&g, &t, a, q, j);
            if (form == ORC_HELMHOLTZ) integrand += params[0] * t.P[q][i] * t.P[q][j];
          }
          out[i * m + j] += scale * integrand;
        }
    }
    return 0;
  case ORC_MASS_ACTION: /* form.hpp:306-312 */
    for (int q = 0; q < r.nq; ++q) {
      const double scale = r.w[q] * g.adetJ;
      double fq = 0.0;
      for (int k = 0; k < m; ++k) fq += C[k] * t.P[q][k];
      for (int i = 0; i < m; ++i) out[i] += scale * fq * t.P[q][i];
    }
    return 0;
  case ORC_STIFFNESS_ACTION: /* form.hpp:288-303 */
  case ORC_HELMHOLTZ_ACTION:
    for (int q = 0; q < r.nq; ++q) {
      const double scale = r.w[q] * g.adetJ;
      double ga[3] = {0, 0, 0};
      for (int k = 0; k < m; ++k)
        for (int a = 0; a < gdim; ++a) ga[a] += C[k] * pgrad(&g, &t, a, q, k);
      double fq = 0.0;
      if (form == ORC_HELMHOLTZ_ACTION)
        for (int k = 0; k < m; ++k) fq += C[k] * t.P[q][k];
      for (int i = 0; i < m; ++i) {
        double integrand = pgrad(&g, &t, 0, q, i) * ga[0];
        for (int a = 1; a < gdim; ++a) integrand += pgrad(&g, &t, a, q, i) * ga[a];
        if (form == ORC_HELMHOLTZ_ACTION) integrand += params[0] * fq * t.P[q][i];
        out[i] += scale * integrand;
      }
    }
    return 0;
  case ORC_ELASTICITY: { /* 2 mu eps(u):eps(v) + lambda div u div v, vector P1 tet */
    const double lam = params[0], mu = params[1];
    for (int q = 0; q < r.nq; ++q) {
      const double scale = r.w[q] * g.adetJ;
      for (int a = 0; a < 4; ++a)
        for (int d = 0; d < 3; ++d)
          for (int b = 0; b < 4; ++b)
            for (int e = 0; e < 3; ++e) {
              double gagb = 0.0;
              for (int k = 0; k < 3; ++k) gagb += pgrad(&g, &t, k, q, a) * pgrad(&g, &t, k, q, b);
              double v = mu * pgrad(&g, &t, e, q, a) * pgrad(&g, &t, d, q, b) +
                         lam * pgrad(&g, &t, d, q, a) * pgrad(&g, &t, e, q, b);
              if (d == e) v += mu * gagb;
              out[(a * 3 + d) * 12 + b * 3 + e] += scale * v;
            }
    }
    return 0;
  }
  case ORC_STOKES_A: { /* nu grad u : grad v, vector P2 tri (component-diagonal) */
    const double nu = params[0];
    for (int q = 0; q < r.nq; ++q) {
      const double scale = r.w[q] * g.adetJ;
      for (int a = 0; a < 6; ++a)
        for (int b = 0; b < 6; ++b) {
          double gg = pgrad(&g, &t, 0, q, a) * pgrad(&g, &t, 0, q, b) +
                      pgrad(&g, &t, 1, q, a) * pgrad(&g, &t, 1, q, b);
          for (int d = 0; d < 2; ++d) out[(a * 2 + d) * 12 + b * 2 + d] += scale * nu * gg;
        }
    }
    return 0;
  }
  case ORC_STOKES_B:
  case ORC_STOKES_BT: { /* b(u, q) = -int q div u ; pressure P1, velocity vector P2 */
    tab_t tp;
    tabulate(2, 1, &r, &tp);
    for (int q = 0; q < r.nq; ++q) {
      const double scale = r.w[q] * g.adetJ;
      for (int p = 0; p < 3; ++p)
        for (int b = 0; b < 6; ++b)
          for (int e = 0; e < 2; ++e) {
            double v = -scale * tp.P[q][p] * pgrad(&g, &t, e, q, b);
            if (form == ORC_STOKES_B) out[p * 12 + b * 2 + e] += v;
            else out[(b * 2 + e) * 3 + p] += v;
          }
    }
    return 0;
  }
  default: return ORC_ERR_UNSUPPORTED_FORM;
  }
}

/* ======================================================================== */
/* Assembly through the par_loop semantics: parloop.hpp:253-320              */
/* ======================================================================== */

int orc_assemble_vector(int form, int degree, int gdim, const double* params, int ncells,
                        const int32_t* test_map, int ar_t, const int32_t* coord_map,
                        const double* coords, const int32_t* coeff_map, int ar_coeff,
                        const double* coeff, int nout, double* out) {
  int rows, cols;
  int err = orc_element_shape(form, degree, gdim, &rows, &cols);
  if (err) return err;
  if (cols != 1 || rows != ar_t) return ORC_ERR_INVALID_ARGUMENT;
  const int nvc = gdim + 1;
  memset(out, 0, sizeof(double) * (size_t)nout); /* make_dat zero-fill (assemble.hpp:111) */
  double X[12], C[16], A[16];
  for (int64_t e = 0; e < ncells; ++e) {
    for (int v = 0; v < nvc; ++v) /* stage-in gather (parloop.hpp:268-273) */
      for (int d = 0; d < gdim; ++d) X[v * gdim + d] = coords[(int64_t)coord_map[e * nvc + v] * gdim + d];
    if (coeff)
      for (int k = 0; k < ar_coeff; ++k) C[k] = coeff[coeff_map[e * ar_coeff + k]];
    err = orc_element(form, degree, gdim, params, X, coeff ? C : NULL, A);
    if (err) return err;
    for (int t = 0; t < ar_t; ++t) out[test_map[e * ar_t + t]] += A[t]; /* INC (parloop.hpp:301-305) */
  }
  return 0;
}

static int addto_cell(int64_t e, const int32_t* row_map, int ar_r, const int32_t* col_map,
                      int ar_c, int nrows, const int64_t* row_ptr, const int32_t* col_idx,
                      const double* A, double* values) {
  for (int i = 0; i < ar_r; ++i) /* Mat::addto (data.hpp:211-221) */
    for (int j = 0; j < ar_c; ++j) {
      int64_t pos = orc_sparsity_find(row_ptr, col_idx, nrows, row_map[e * ar_r + i],
                                      col_map[e * ar_c + j]);
      if (pos < 0) return ORC_ERR_OUTSIDE_SPARSITY;
      values[pos] += A[i * ar_c + j];
    }
  return 0;
}

static int stage_cell(int form, int degree, int gdim, const double* params, int64_t e,
                      const int32_t* coord_map, const double* coords, double* A) {
  const int nvc = gdim + 1;
  double X[12];
  for (int v = 0; v < nvc; ++v)
    for (int d = 0; d < gdim; ++d) X[v * gdim + d] = coords[(int64_t)coord_map[e * nvc + v] * gdim + d];
  return orc_element(form, degree, gdim, params, X, NULL, A);
}

int orc_assemble_matrix(int form, int degree, int gdim, const double* params, int ncells,
                        const int32_t* row_map, int ar_r, const int32_t* col_map, int ar_c,
                        const int32_t* coord_map, const double* coords, int nrows,
                        const int64_t* row_ptr, const int32_t* col_idx, double* values) {
  int rows, cols;
  int err = orc_element_shape(form, degree, gdim, &rows, &cols);
  if (err) return err;
  if (rows != ar_r || cols != ar_c) return ORC_ERR_INVALID_ARGUMENT;
  memset(values, 0, sizeof(double) * (size_t)row_ptr[nrows]); /* data.hpp:187 */
  double A[144];
  for (int64_t e = 0; e < ncells; ++e) {
    err = stage_cell(form, degree, gdim, params, e, coord_map, coords, A);
    if (err) return err;
    err = addto_cell(e, row_map, ar_r, col_map, ar_c, nrows, row_ptr, col_idx, A, values);
    if (err) return err;
  }
  return 0;
}

int orc_assemble_matrix_colored(int form, int degree, int gdim, const double* params, int ncells,
                                const int32_t* row_map, int ar_r, const int32_t* col_map,
                                int ar_c, const int32_t* coord_map, const double* coords,
                                int nrows, const int64_t* row_ptr, const int32_t* col_idx,
                                const int32_t* colors, int ncolors, double* values) {
  int rows, cols;
  int err = orc_element_shape(form, degree, gdim, &rows, &cols);
  if (err) return err;
  if (rows != ar_r || cols != ar_c) return ORC_ERR_INVALID_ARGUMENT;
  memset(values, 0, sizeof(double) * (size_t)row_ptr[nrows]);
  double A[144];
  for (int c = 0; c < ncolors; ++c) /* parloop.hpp:234-235, 322-352 */
    for (int64_t e = 0; e < ncells; ++e) {
      if (colors[e] != c) continue;
      err = stage_cell(form, degree, gdim, params, e, coord_map, coords, A);
      if (err) return err;
      err = addto_cell(e, row_map, ar_r, col_map, ar_c, nrows, row_ptr, col_idx, A, values);
      if (err) return err;
    }
  return 0;
}


/* ---- consumers of the assembled matrix ------------------- */

/* data.hpp:236-250 mat_spmv / solver.hpp:33-58 block_spmv */
void orc_block_spmv(const int32_t* rs, const int32_t* cs, const int64_t* const* rp, const int32_t* const* ci,
                    const double* const* v, const double* x, double* y) {
  int out = 0;
  for (int bi = 0; bi < 2; ++bi)
    for (int r = 0; r < rs[bi]; ++r) {
      double acc = 0.0;
      int col_off = 0;
      for (int bj = 0; bj < 2; ++bj) {
        const int k = 2 * bi + bj;
        if (rp[k])
          for (int64_t e = rp[k][r]; e < rp[k][r + 1]; ++e) {
            const double prod = v[k][e] * x[col_off + ci[k][e]];
            acc = acc + prod;
          }
        col_off += cs[bj];
      }
      y[out++] = acc;
    }
}

static double orc_dot(const double* a, const double* c, int n) { /* solver.hpp:93-97 */
  double acc = 0.0;
  for (int i = 0; i < n; ++i) acc += a[i] * c[i];
  return acc;
}

/* solver.hpp:64-76: 1 / A(r, r), Mat::at = 0 outside the pattern */
static int orc_inv_diag(int n, const int64_t* rp, const int32_t* ci, const double* v, double* inv) {
  for (int r = 0; r < n; ++r) {
    double d = 0.0;
    for (int64_t e = rp[r]; e < rp[r + 1]; ++e)
      if (ci[e] == r) d = v[e];
    if (!(d > 0.0)) return r;
    inv[r] = 1.0 / d;
  }
  return -1;
}

int orc_cg(const int32_t* rs, const int32_t* cs, const int64_t* const* rp, const int32_t* const* ci,
           const double* const* v, int nested, const double* b, double* x, double rtol, double atol, int maxit,
           int jacobi, int32_t* report, double* rnorm_out, int32_t* fail) {
  const int n = rs[0] + rs[1];
  double *inv = NULL, *r = malloc(sizeof(double) * (n + 1)), *z = malloc(sizeof(double) * (n + 1)),
         *p = malloc(sizeof(double) * (n + 1)), *q = malloc(sizeof(double) * (n + 1));
  int rc = 0;
  report[0] = 0;
  report[1] = 0;
  report[2] = 2;
  if (jacobi) { /* solver.hpp:180-201 */
    inv = malloc(sizeof(double) * (n + 1));
    int off = 0;
    for (int i = 0; i < (nested ? 2 : 1); ++i) {
      const int k = 3 * i; /* diagonal block (i, i) */
      int bad = rp[k] ? orc_inv_diag(rs[i], rp[k], ci[k], v[k], inv + off) : 0;
      if (bad >= 0) {
        *fail = bad;
        rc = ORC_ERR_INDEFINITE;
        goto done;
      }
      off += rs[i];
    }
  }
  { /* cg_iterate, solver.hpp:88-167 */
    const double target = fmax(rtol * sqrt(orc_dot(b, b, n)), atol);
    orc_block_spmv(rs, cs, rp, ci, v, x, q);
    for (int i = 0; i < n; ++i) r[i] = b[i] - q[i];
    double rnorm = sqrt(orc_dot(r, r, n));
    if (rnorm <= target) {
      report[1] = 1;
      report[2] = rnorm <= atol ? 1 : 0;
      *rnorm_out = rnorm;
      goto done;
    }
    for (int i = 0; i < n; ++i) z[i] = inv ? inv[i] * r[i] : r[i];
    for (int i = 0; i < n; ++i) p[i] = z[i];
    double rz = orc_dot(r, z, n);
    for (int it = 1; it <= maxit; ++it) {
      orc_block_spmv(rs, cs, rp, ci, v, p, q);
      const double pq = orc_dot(p, q, n);
      if (!(pq > 0.0)) {
        *fail = it;
        rc = ORC_ERR_INDEFINITE;
        goto done;
      }
      const double alpha = rz / pq;
      for (int i = 0; i < n; ++i) x[i] += alpha * p[i];
      for (int i = 0; i < n; ++i) r[i] -= alpha * q[i];
      report[0] = it;
      rnorm = sqrt(orc_dot(r, r, n));
      if (rnorm <= target) {
        orc_block_spmv(rs, cs, rp, ci, v, x, q);
        for (int i = 0; i < n; ++i) r[i] = b[i] - q[i];
        rnorm = sqrt(orc_dot(r, r, n));
        if (rnorm <= target) {
          report[1] = 1;
          report[2] = rnorm <= atol ? 1 : 0;
          *rnorm_out = rnorm;
          goto done;
        }
      }
      for (int i = 0; i < n; ++i) z[i] = inv ? inv[i] * r[i] : r[i];
      const double rz_next = orc_dot(r, z, n);
      const double beta = rz_next / rz;
      rz = rz_next;
      for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
    *rnorm_out = rnorm;
  }
done:
  free(inv);
  free(r);
  free(z);
  free(p);
  free(q);
  return rc;
}

/* ---- around the assembly loop -------------------------------------------- */

/* fem/assemble.hpp:225-247 lower_pw + :252-314 pointwise: the reference lowers
 * the expression to one assignment per component; out += e stages INC (0 + e,
 * then out + staged), out -= e accumulates -e: both equal out (+|-) e. */
int orc_pointwise(double* out, int64_t n, int assign, const int32_t* ops, const int32_t* fidx,
                  const double* vals, int nprog, const double* const* fields) {
  double st[64];
  if (nprog <= 0 || nprog > 64) return ORC_ERR_INVALID_ARGUMENT;
  for (int64_t i = 0; i < n; ++i) {
    int sp = 0;
    for (int q = 0; q < nprog; ++q) {
      switch (ops[q]) {
      case 0: st[sp++] = vals[q]; break;
      case 1: st[sp++] = fidx[q] < 0 ? out[i] : fields[fidx[q]][i]; break;
      case 6: st[sp - 1] = -st[sp - 1]; break;
      default: {
        const double b = st[--sp], a = st[sp - 1];
        st[sp - 1] = ops[q] == 2 ? a + b : ops[q] == 3 ? a - b : ops[q] == 4 ? a * b : a / b;
      }
      }
    }
    const double v = st[0];
    out[i] = assign == 0 ? v : assign == 1 ? out[i] + v : out[i] - v;
  }
  return ORC_OK;
}

/* fem/assemble.hpp:54-79 with Sparsity::find (data.hpp:129-136). */
int orc_apply_dirichlet(int nrows, const int64_t* row_ptr, const int32_t* col_idx, double* values,
                        double* rhs, const int32_t* nodes, int nn, const double* node_values,
                        double constant, int32_t* fail) {
  for (int q = 0; q < nn; ++q) {
    const int r = nodes[q];
    if (r < 0 || r >= nrows) return ORC_ERR_INDEX_OUT_OF_RANGE;
    for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) values[k] = 0.0;
    const int64_t d = orc_sparsity_find(row_ptr, col_idx, nrows, r, r);
    if (d < 0) {
      if (fail) *fail = r;
      return ORC_ERR_MISSING_DIAGONAL;
    }
    values[d] = 1.0;
    if (rhs) rhs[r] = node_values ? node_values[r] : constant;
  }
  return ORC_OK;
}

/* topology.hpp:131-178.  The queue is order[] itself (head chases tail);
 * a dequeued vertex's new neighbours are insertion-sorted by (degree, index)
 * in place at the tail before they are enqueued. */
int orc_rcm_order(int n, const int64_t* row_ptr, const int32_t* col_idx, int32_t* order, int64_t* fail) {
  for (int u = 0; u < n; ++u)
    for (int64_t k = row_ptr[u]; k < row_ptr[u + 1]; ++k) {
      const int v = col_idx[k];
      if (v < 0 || v >= n) {
        if (fail) *fail = k;
        return ORC_ERR_INDEX_OUT_OF_RANGE;
      }
      int64_t q = row_ptr[v];
      while (q < row_ptr[v + 1] && col_idx[q] != u) ++q;
      if (q == row_ptr[v + 1]) {
        if (fail) *fail = k;
        return ORC_ERR_ASYMMETRIC_ADJACENCY;
      }
    }
  char* seen = (char*)calloc(n ? (size_t)n : 1, 1);
  if (!seen) return ORC_ERR_INVALID_ARGUMENT;
#define DEG(x) (row_ptr[(x) + 1] - row_ptr[(x)])
#define BEFORE(a, b) (DEG(a) != DEG(b) ? DEG(a) < DEG(b) : (a) < (b))
  int tail = 0;
  for (;;) {
    int seed = -1;
    for (int u = 0; u < n; ++u)
      if (!seen[u] && (seed < 0 || DEG(u) < DEG(seed))) seed = u;
    if (seed < 0) break;
    seen[seed] = 1;
    int head = tail;
    order[tail++] = seed;
    while (head < tail) {
      const int u = order[head++];
      const int first = tail;
      for (int64_t k = row_ptr[u]; k < row_ptr[u + 1]; ++k) {
        const int v = col_idx[k];
        if (seen[v]) continue;
        seen[v] = 1;
        int j = tail++;
        while (j > first && BEFORE(v, order[j - 1])) {
          order[j] = order[j - 1];
          --j;
        }
        order[j] = v;
      }
    }
  }
#undef BEFORE
#undef DEG
  free(seen);
  for (int i = 0, j = n - 1; i < j; ++i, --j) {
    const int32_t t = order[i];
    order[i] = order[j];
    order[j] = t;
  }
  return ORC_OK;
}

/* ---- seeded synthetic inputs (bench --impl reference) -------- */
/* The reference has no jitter / permutation / coefficient generator; the
 * meshes themselves restate unit_square_mesh (mesh.hpp:96-143: vertices
 * row-major, cells (a,b,c),(a,c,d) per square, a=SW b=SE c=NE d=NW) and
 * unit_cube_mesh (mesh.hpp:148-214: six Kuhn tets per cube, one per axis
 * permutation, odd permutations re-oriented).  The stream is splitmix64 with
 * u = (x >> 11) * 2^-53.  tests/test_oracle_cpu.py checks these
 * against the compiled reference's meshes and against the product's own
 * generator bit-for-bit. */
static uint64_t orc_sm64(uint64_t* st) {
  uint64_t z = (*st += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double orc_sm64_u(uint64_t* st) { return (double)(orc_sm64(st) >> 11) * 0x1.0p-53; }

int orc_unit_square_mesh(int n, double* coords, int32_t* cv) {
  if (n < 1) return ORC_ERR_INVALID_ARGUMENT;
  for (int j = 0; j <= n; ++j)
    for (int i = 0; i <= n; ++i) {
      const int64_t v = (int64_t)j * (n + 1) + i;
      coords[2 * v] = (double)i / n;
      coords[2 * v + 1] = (double)j / n;
    }
  int64_t w = 0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const int32_t a = j * (n + 1) + i, b = a + 1, c = a + n + 2, d = a + n + 1;
      const int32_t t[6] = {a, b, c, a, c, d};
      for (int q = 0; q < 6; ++q) cv[w++] = t[q];
    }
  return ORC_OK;
}

int orc_unit_cube_mesh(int n, double* coords, int32_t* cv) {
  static const int axes[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  if (n < 1) return ORC_ERR_INVALID_ARGUMENT;
  const int64_t s = n + 1;
  for (int k = 0; k <= n; ++k)
    for (int j = 0; j <= n; ++j)
      for (int i = 0; i <= n; ++i) {
        const int64_t v = ((int64_t)k * s + j) * s + i;
        coords[3 * v] = (double)i / n;
        coords[3 * v + 1] = (double)j / n;
        coords[3 * v + 2] = (double)k / n;
      }
  int64_t w = 0;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        for (int p = 0; p < 6; ++p) {
          int x[3] = {i, j, k};
          int32_t t[4];
          t[0] = (int32_t)(((int64_t)x[2] * s + x[1]) * s + x[0]);
          for (int q = 0; q < 3; ++q) {
            x[axes[p][q]]++;
            t[q + 1] = (int32_t)(((int64_t)x[2] * s + x[1]) * s + x[0]);
          }
          /* the odd axis permutations (one transposition from identity) give
             negatively oriented tets: swap the last two vertices */
          const int odd = (p == 1 || p == 2 || p == 5);
          if (odd) {
            const int32_t tmp = t[2];
            t[2] = t[3];
            t[3] = tmp;
          }
          for (int q = 0; q < 4; ++q) cv[w++] = t[q];
        }
  return ORC_OK;
}

int orc_jitter(int gdim, int n, double amp, uint64_t seed, double* coords) {
  if ((gdim != 2 && gdim != 3) || n < 1) return ORC_ERR_INVALID_ARGUMENT;
  const int64_t s = n + 1, nv = gdim == 2 ? s * s : s * s * s;
  const double h = 1.0 / n;
  uint64_t st = seed;
  for (int64_t v = 0; v < nv; ++v) {
    const int64_t i = v % s, j = (v / s) % s, k = gdim == 3 ? v / (s * s) : 1;
    if (!(i > 0 && i < n && j > 0 && j < n && (gdim == 2 || (k > 0 && k < n)))) continue;
    for (int d = 0; d < gdim; ++d) coords[v * gdim + d] += (2.0 * orc_sm64_u(&st) - 1.0) * amp * h;
  }
  return ORC_OK;
}

int orc_permute_cells(int ncells, int arity, uint64_t seed, int32_t* cv) {
  if (ncells < 0 || arity < 1) return ORC_ERR_INVALID_ARGUMENT;
  uint64_t st = seed;
  for (int64_t i = (int64_t)ncells - 1; i >= 1; --i) {
    const int64_t j = (int64_t)(orc_sm64(&st) % (uint64_t)(i + 1));
    if (j == i) continue;
    for (int a = 0; a < arity; ++a) {
      const int32_t tmp = cv[i * arity + a];
      cv[i * arity + a] = cv[j * arity + a];
      cv[j * arity + a] = tmp;
    }
  }
  return ORC_OK;
}

int orc_uniform(int64_t count, uint64_t seed, double lo, double hi, double* out) {
  uint64_t st = seed;
  for (int64_t k = 0; k < count; ++k) out[k] = lo + (hi - lo) * orc_sm64_u(&st);
  return ORC_OK;
}
