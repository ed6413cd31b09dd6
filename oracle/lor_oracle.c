/*
 * lor_oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously-correct CPU oracle for
 * low-order-refined (LOR) matrix assembly (arXiv 2210.12253, Step S1.2 "Low-order-refined matrix
 * assembly").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header, table
 * or constant generator with the CUDA path (paper_2210_12253_b200/csrc/).
 *
 * What it computes -- the plain definition the macro-element method reorganises
 * ("A = Lambda^T Ahat Lambda ... blocks local to each macro element"):
 *
 *     A_S = sum_{coarse e} sum_{LOR cells K in e} P_K^T diag(s_K) A_K(alpha,beta) diag(s_K) P_K
 *
 *   * LOR cells: each element is split into p^d sub-cells whose vertices are the element's
 *     coordinate E-vector entries at the tensor Gauss-Lobatto points (Sec 2.1;
 *     l.342-345: coordinates given as a high-order E-vector).  The E-vector is an INPUT.
 *   * A_K: the textbook lowest-order matrix of the cell: Q1 for H1 (l.107-117 "V_h is the p=1
 *     space on the refined mesh"), lowest-order Nedelec / Raviart-Thomas for H(curl)/H(div)
 *     ("the lowest-order case ... reduces exactly to the standard lowest-order Nedelec and
 *     Raviart-Thomas elements", l.150), evaluated generically at every quadrature point of the
 *     rule (vertex rule = SURVEY reading P-1, Gauss-2 optional), no sparsity tricks.
 *   * Pattern = every pair of dofs sharing a LOR cell, explicit zeros kept (reading P-3),
 *     both triangles stored (P-4), columns ascending (P-5).
 *   * Numbering, orientation and signs: SURVEY App. A (reading P-6/P-7), implemented here
 *     independently of the GPU library's setup code.
 *   * Discrete gradient: Algorithm 1; discrete curl: l.440-445 (truncated
 *     sentence; reading P-15 = right-hand-rule circulation about the face's global normal).
 *
 * Step order follows SURVEY 8(c) c.2: O2 numbering, O3 explicit refinement, O4 dense local
 * matrices, O5 scatter triplets, O6 sort-and-sum into CSR, O7 G and C, O10 row oracle.
 * Build:  gcc -O2 -ffp-contract=off -fPIC -shared -o liblor_oracle.so lor_oracle.c -lm
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_H1 = 0, ORC_ND = 1, ORC_RT = 2 };
enum { ORC_QUAD_VERTEX = 0, ORC_QUAD_GAUSS2 = 1 };
enum { ORC_OK = 0, ORC_ERR_ARG = 1, ORC_ERR_DEGENERATE = 2, ORC_ERR_MEM = 3, ORC_ERR_INCONSISTENT = 4 };

typedef struct {
  int dim, p;
  int64_t nv, nel;
  const int64_t *elem;  /* [nel][2^dim], local corner order a + 2b + 4c          */
  const double *X;      /* [nel][dim][(p+1)^dim] coordinate E-vector (GLL points) */
  int nranks;
  const int64_t *erb;   /* [nranks+1] contiguous element slabs (NULL: 1 rank)    */
  const double *ca, *cb; /* [nel][(p+1)^dim] coefficient E-vectors a(x), b(x) at the GLL points
                           (variable coefficients, reading P-28), or NULL: constants */
} orc_mesh;

typedef struct {
  int64_t n_rows, n_cols, nnz;
  int64_t *row_ptr;  /* [n_rows+1] */
  int64_t *row_id;   /* [n_rows] global row id of each stored row */
  int32_t *col;      /* [nnz] */
  double *val;       /* [nnz] */
} orc_csr;

static char g_err[512];
const char *orc_last_error(void) { return g_err; }

/* ======================================================================================
 * Gauss-Lobatto points ("the p+1 Gauss--Lobatto points").  Roots of
 * (1-x^2) P_p'(x) by Newton iteration in long double from Chebyshev-Gauss-Lobatto guesses.
 * Weights w_i = 2 / (p (p+1) P_p(x_i)^2).  Used only by the HO spectral self-check.
 * ==================================================================================== */
static void legendre(int n, long double x, long double *P, long double *dP) {
  long double p0 = 1.0L, p1 = x;
  if (n == 0) { *P = 1.0L; *dP = 0.0L; return; }
  for (int k = 2; k <= n; ++k) {
    long double p2 = ((2.0L * k - 1.0L) * x * p1 - (k - 1.0L) * p0) / k;
    p0 = p1; p1 = p2;
  }
  *P = p1;
  *dP = n * (x * p1 - p0) / (x * x - 1.0L); /* valid for |x| < 1 */
}

void orc_gll(int p, double *x, double *w) {
  for (int i = 0; i <= p; ++i) {
    long double xi = -cosl(3.14159265358979323846264338327950288L * i / p);
    if (i > 0 && i < p) {
      for (int it = 0; it < 100; ++it) {
        /* f = P_p'(x);  f' = P_p''(x) = (2x P_p' - p(p+1) P_p) / (1 - x^2) */
        long double P, dP;
        legendre(p, xi, &P, &dP);
        long double d2P = (2.0L * xi * dP - p * (p + 1.0L) * P) / (1.0L - xi * xi);
        long double dx = dP / d2P;
        xi -= dx;
        if (fabsl(dx) < 1e-30L) break;
      }
    }
    long double P = 1.0L, dP;
    if (i == 0) P = (p % 2) ? -1.0L : 1.0L;
    else if (i == p) P = 1.0L;
    else legendre(p, xi, &P, &dP);
    x[i] = (double)xi;
    w[i] = (double)(2.0L / (p * (p + 1.0L) * P * P));
  }
}

/* ======================================================================================
 * O4: textbook local matrices on one LOR cell.  Reference cell [0,1]^d (reading P-11),
 * quadrature: vertex rule (points {0,1}^d, w = 2^-d, reading P-1) or Gauss-2
 * (points 1/2 +- 1/(2 sqrt 3), w = 2^-d).  corners: [2^d][d] physical vertex coordinates
 * in local order a + 2b + 4c.  All reference basis functions and their derivatives are
 * evaluated generically at each point.
 * ==================================================================================== */
static int quad_points(int dim, int quad, double pts[8][3], double *w) {
  int nq = 1 << dim;
  double g0 = 0.5 - 0.5 / sqrt(3.0), g1 = 0.5 + 0.5 / sqrt(3.0);
  for (int q = 0; q < nq; ++q)
    for (int d = 0; d < dim; ++d) {
      int bit = (q >> d) & 1;
      pts[q][d] = (quad == ORC_QUAD_VERTEX) ? (double)bit : (bit ? g1 : g0);
    }
  *w = 1.0 / nq;
  return nq;
}

/* Q1 basis N_v(x) = prod_d (bit_d(v) ? x_d : 1 - x_d) and its reference gradient. */
static void q1_basis(int dim, const double *x, int v, double *N, double *grad) {
  double f[3], df[3];
  for (int d = 0; d < dim; ++d) {
    int bit = (v >> d) & 1;
    f[d] = bit ? x[d] : 1.0 - x[d];
    df[d] = bit ? 1.0 : -1.0;
  }
  double prod = 1.0;
  for (int d = 0; d < dim; ++d) prod *= f[d];
  *N = prod;
  for (int d = 0; d < dim; ++d) {
    double g = df[d];
    for (int e = 0; e < dim; ++e)
      if (e != d) g *= f[e];
    grad[d] = g;
  }
}

/* Jacobian of the (bi/tri)linear cell map at reference point x: J[k][d] = sum_v X_v[k] dN_v/dx_d */
static void jacobian(int dim, const double *corners, const double *x, double J[3][3]) {
  for (int k = 0; k < dim; ++k)
    for (int d = 0; d < dim; ++d) J[k][d] = 0.0;
  for (int v = 0; v < (1 << dim); ++v) {
    double N, g[3];
    q1_basis(dim, x, v, &N, g);
    for (int k = 0; k < dim; ++k)
      for (int d = 0; d < dim; ++d) J[k][d] += corners[v * dim + k] * g[d];
  }
}

/* determinant and inverse by explicit cofactors */
static double inverse(int dim, double J[3][3], double Ji[3][3]) {
  if (dim == 2) {
    double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    Ji[0][0] = J[1][1] / det; Ji[0][1] = -J[0][1] / det;
    Ji[1][0] = -J[1][0] / det; Ji[1][1] = J[0][0] / det;
    return det;
  }
  double c[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
      c[i][j] = J[i1][j1] * J[i2][j2] - J[i1][j2] * J[i2][j1]; /* cofactor C_ij */
    }
  double det = J[0][0] * c[0][0] + J[0][1] * c[0][1] + J[0][2] * c[0][2];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Ji[i][j] = c[j][i] / det; /* inverse = C^T / det */
  return det;
}

/* Reference lowest-order Nedelec function of cell edge eps (3D), local order
 * x-edges (b,c) -> b + 2c, y-edges (a,c) -> 4 + a + 2c, z-edges (a,b) -> 8 + a + 2b (App. A.3):
 * phi = e_a f_u(x_u) f_v(x_v), (u,v) the other axes increasing, f = bit ? x : 1-x;
 * curl phi = grad(f_u f_v) x e_a.  Its tangential integral along its own edge is 1. */
static void nd_basis(const double *x, int eps, double phi[3], double curl[3]) {
  int a = eps / 4, b1 = eps & 1, b2 = (eps >> 1) & 1;
  int u = (a == 0) ? 1 : 0, v = (a == 2) ? 1 : 2;
  double fu = b1 ? x[u] : 1.0 - x[u], dfu = b1 ? 1.0 : -1.0;
  double fv = b2 ? x[v] : 1.0 - x[v], dfv = b2 ? 1.0 : -1.0;
  double grad[3] = {0, 0, 0};
  grad[u] = dfu * fv;
  grad[v] = fu * dfv;
  phi[0] = phi[1] = phi[2] = 0.0;
  phi[a] = fu * fv;
  double ea[3] = {0, 0, 0};
  ea[a] = 1.0;
  curl[0] = grad[1] * ea[2] - grad[2] * ea[1];
  curl[1] = grad[2] * ea[0] - grad[0] * ea[2];
  curl[2] = grad[0] * ea[1] - grad[1] * ea[0];
}

/* Reference lowest-order Raviart-Thomas function of cell face 2a + side (normal +e_a):
 * phi = e_a (side ? x_a : 1 - x_a); div phi = side ? 1 : -1.  Unit flux through its face. */
static void rt_basis(const double *x, int f, double phi[3], double *div) {
  int a = f / 2, side = f & 1;
  phi[0] = phi[1] = phi[2] = 0.0;
  phi[a] = side ? x[a] : 1.0 - x[a];
  *div = side ? 1.0 : -1.0;
}

static int local_ndof(int dim, int space) {
  if (space == ORC_H1) return 1 << dim;
  if (dim == 2) return 4;
  if (space == ORC_ND) return 12;
  return 6;
}

/* A (n x n, row major) = local matrix of alpha*a(x)*(grad|curl|div) + beta*b(x)*(mass) on one cell;
 * a, b = the multilinear interpolants of the corner values ca8 / cb8 (vertex order), evaluated at each
 * quadrature point (reading P-28: coefficients sampled at the LOR vertices);
 * ca8 == cb8 == NULL: a = b = 1. */
int orc_local_matrix_vc(int dim, int space, int quad, double alpha, double beta, const double *corners,
                        const double *ca8, const double *cb8, double *A);
int orc_local_matrix(int dim, int space, int quad, double alpha, double beta, const double *corners,
                     double *A) {
  return orc_local_matrix_vc(dim, space, quad, alpha, beta, corners, NULL, NULL, A);
}

/* value at reference point x of the multilinear interpolant of the 2^dim corner values c (NULL: 1) */
static double corner_interp(int dim, const double *c, const double *x) {
  if (!c) return 1.0;
  double s = 0.0;
  for (int v = 0; v < (1 << dim); ++v) {
    double N, g[3];
    q1_basis(dim, x, v, &N, g);
    s += N * c[v];
  }
  return s;
}

int orc_local_matrix_vc(int dim, int space, int quad, double alpha, double beta, const double *corners,
                        const double *ca8, const double *cb8, double *A) {
  if (!(dim == 2 || dim == 3)) return ORC_ERR_ARG;
  int n = local_ndof(dim, space);
  for (int i = 0; i < n * n; ++i) A[i] = 0.0;
  double pts[8][3], w;
  int nq = quad_points(dim, quad, pts, &w);
  for (int q = 0; q < nq; ++q) {
    double J[3][3], Ji[3][3];
    jacobian(dim, corners, pts[q], J);
    double det = inverse(dim, J, Ji);
    if (!(det > 0.0)) return ORC_ERR_DEGENERATE;
    const double aq = alpha * corner_interp(dim, ca8, pts[q]), bq = beta * corner_interp(dim, cb8, pts[q]);
    if (dim == 2 && space != ORC_H1) { /* 2D lowest-order Nedelec / Raviart-Thomas on the quad */
      double phi[4][2], sc[4];
      for (int i = 0; i < 4; ++i) {
        double ph[2], dv;
        int fam = i / 2, off = i & 1;
        if (space == ORC_ND) { /* x-edge at y = off: (f(y), 0); y-edge at x = off: (0, f(x)) */
          int o = 1 - fam;
          double f = off ? pts[q][o] : 1.0 - pts[q][o], df = off ? 1.0 : -1.0;
          ph[fam] = f;
          ph[o] = 0.0;
          dv = fam == 0 ? -df : df; /* scalar curl = d phi_y/dx - d phi_x/dy */
          for (int c = 0; c < 2; ++c) phi[i][c] = Ji[0][c] * ph[0] + Ji[1][c] * ph[1]; /* J^{-T} phi-hat */
        } else { /* face normal e_fam at side off: e_fam (off ? x_fam : 1 - x_fam), div = off ? 1 : -1 */
          ph[fam] = off ? pts[q][fam] : 1.0 - pts[q][fam];
          ph[1 - fam] = 0.0;
          dv = off ? 1.0 : -1.0;
          for (int c = 0; c < 2; ++c) phi[i][c] = (J[c][0] * ph[0] + J[c][1] * ph[1]) / det; /* J phi-hat / det */
        }
        sc[i] = dv / det;
      }
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j)
          A[i * 4 + j] += w * (aq * sc[i] * sc[j] + bq * (phi[i][0] * phi[j][0] + phi[i][1] * phi[j][1])) * det;
    } else if (space == ORC_H1) {
      double N[8], g[8][3];
      for (int i = 0; i < n; ++i) {
        double gr[3];
        q1_basis(dim, pts[q], i, &N[i], gr);
        for (int k = 0; k < dim; ++k) { /* physical gradient J^{-T} grad-hat */
          g[i][k] = 0.0;
          for (int d = 0; d < dim; ++d) g[i][k] += Ji[d][k] * gr[d];
        }
      }
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          double gg = 0.0;
          for (int k = 0; k < dim; ++k) gg += g[i][k] * g[j][k];
          A[i * n + j] += w * (aq * gg + bq * N[i] * N[j]) * det;
        }
    } else if (space == ORC_ND) {
      double phi[12][3], cu[12][3];
      for (int i = 0; i < 12; ++i) {
        double ph[3], ch[3];
        nd_basis(pts[q], i, ph, ch);
        for (int k = 0; k < 3; ++k) {
          phi[i][k] = 0.0; /* covariant Piola: J^{-T} phi-hat */
          cu[i][k] = 0.0;  /* curl: J curl-hat / det */
          for (int d = 0; d < 3; ++d) {
            phi[i][k] += Ji[d][k] * ph[d];
            cu[i][k] += J[k][d] * ch[d];
          }
          cu[i][k] /= det;
        }
      }
      for (int i = 0; i < 12; ++i)
        for (int j = 0; j < 12; ++j) {
          double cc = 0.0, pp = 0.0;
          for (int k = 0; k < 3; ++k) {
            cc += cu[i][k] * cu[j][k];
            pp += phi[i][k] * phi[j][k];
          }
          A[i * 12 + j] += w * (aq * cc + bq * pp) * det;
        }
    } else {
      double phi[6][3], dv[6];
      for (int i = 0; i < 6; ++i) {
        double ph[3];
        rt_basis(pts[q], i, ph, &dv[i]);
        for (int k = 0; k < 3; ++k) { /* contravariant Piola: J phi-hat / det */
          phi[i][k] = 0.0;
          for (int d = 0; d < 3; ++d) phi[i][k] += J[k][d] * ph[d];
          phi[i][k] /= det;
        }
        dv[i] /= det;
      }
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) {
          double pp = 0.0;
          for (int k = 0; k < 3; ++k) pp += phi[i][k] * phi[j][k];
          A[i * 6 + j] += w * (aq * dv[i] * dv[j] + bq * pp) * det;
        }
    }
  }
  return ORC_OK;
}

/* ======================================================================================
 * O2: numbering, implemented from the text.
 * ==================================================================================== */
typedef struct { int64_t k[4]; } key4;

static int cmp_key2(const void *a, const void *b) {
  const int64_t *x = (const int64_t *)a, *y = (const int64_t *)b;
  for (int i = 0; i < 2; ++i) {
    if (x[i] < y[i]) return -1;
    if (x[i] > y[i]) return 1;
  }
  return 0;
}
static int cmp_key4(const void *a, const void *b) {
  const int64_t *x = (const int64_t *)a, *y = (const int64_t *)b;
  for (int i = 0; i < 4; ++i) {
    if (x[i] < y[i]) return -1;
    if (x[i] > y[i]) return 1;
  }
  return 0;
}
static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}

typedef struct {
  int dim, p;
  int64_t nv, ne, nf, nel;
  int64_t *edges;   /* [ne][2] sorted unique (min vid, max vid)          */
  int64_t *faces;   /* [nf][4] sorted unique sorted vertex 4-tuples      */
  int64_t *el_edge; /* [nel][12 or 4] global edge id of each local edge  */
  int64_t *el_face; /* [nel][6] global face id of each local face        */
} topo_t;

/* local edge (axis d, bits (b1,b2) of the other axes increasing) = 4d + b1 + 2b2 (App. A.2);
 * in 2D: 2d + b1.  tail = corner with d-bit 0, head = d-bit 1. */
static void edge_corners(int dim, int le, int *tail, int *head) {
  if (dim == 3) {
    int d = le / 4, b1 = le & 1, b2 = (le >> 1) & 1;
    int u = (d == 0) ? 1 : 0, v = (d == 2) ? 1 : 2;
    int c = (b1 << u) | (b2 << v);
    *tail = c;
    *head = c | (1 << d);
  } else {
    int d = le / 2, b1 = le & 1;
    int u = 1 - d;
    int c = b1 << u;
    *tail = c;
    *head = c | (1 << d);
  }
}

/* corners of local face 2d + side listed by face-local (alpha, beta) along (u, v) increasing */
static void face_corners(int lf, int fc[2][2]) {
  int d = lf / 2, side = lf & 1;
  int u = (d == 0) ? 1 : 0, v = (d == 2) ? 1 : 2;
  for (int al = 0; al < 2; ++al)
    for (int be = 0; be < 2; ++be) fc[al][be] = (side << d) | (al << u) | (be << v);
}

static int64_t find_key2(const int64_t *arr, int64_t n, int64_t a, int64_t b) {
  int64_t lo = 0, hi = n - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) / 2;
    const int64_t *m = arr + 2 * mid;
    if (m[0] == a && m[1] == b) return mid;
    if (m[0] < a || (m[0] == a && m[1] < b)) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}
static int64_t find_key4(const int64_t *arr, int64_t n, const int64_t *k) {
  int64_t lo = 0, hi = n - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) / 2;
    int c = cmp_key4(arr + 4 * mid, k);
    if (c == 0) return mid;
    if (c < 0) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}

static void topo_free(topo_t *t) {
  free(t->edges); free(t->faces); free(t->el_edge); free(t->el_face);
  memset(t, 0, sizeof(*t));
}

static int topo_build(const orc_mesh *m, topo_t *t) {
  memset(t, 0, sizeof(*t));
  t->dim = m->dim; t->p = m->p; t->nv = m->nv; t->nel = m->nel;
  int nc = 1 << m->dim, nle = (m->dim == 3) ? 12 : 4;
  int64_t *keys = (int64_t *)malloc(sizeof(int64_t) * 2 * m->nel * nle);
  if (!keys) return ORC_ERR_MEM;
  for (int64_t e = 0; e < m->nel; ++e)
    for (int le = 0; le < nle; ++le) {
      int tl, hd;
      edge_corners(m->dim, le, &tl, &hd);
      int64_t a = m->elem[e * nc + tl], b = m->elem[e * nc + hd];
      keys[2 * (e * nle + le)] = a < b ? a : b;
      keys[2 * (e * nle + le) + 1] = a < b ? b : a;
    }
  qsort(keys, m->nel * nle, 2 * sizeof(int64_t), cmp_key2);
  int64_t ne = 0;
  for (int64_t i = 0; i < m->nel * nle; ++i)
    if (i == 0 || cmp_key2(keys + 2 * i, keys + 2 * (ne - 1)) != 0) {
      keys[2 * ne] = keys[2 * i]; keys[2 * ne + 1] = keys[2 * i + 1]; ++ne;
    }
  t->ne = ne;
  t->edges = keys;
  t->el_edge = (int64_t *)malloc(sizeof(int64_t) * m->nel * nle);
  for (int64_t e = 0; e < m->nel; ++e)
    for (int le = 0; le < nle; ++le) {
      int tl, hd;
      edge_corners(m->dim, le, &tl, &hd);
      int64_t a = m->elem[e * nc + tl], b = m->elem[e * nc + hd];
      t->el_edge[e * nle + le] = find_key2(t->edges, ne, a < b ? a : b, a < b ? b : a);
    }
  if (m->dim == 3) {
    int64_t *fk = (int64_t *)malloc(sizeof(int64_t) * 4 * m->nel * 6);
    for (int64_t e = 0; e < m->nel; ++e)
      for (int lf = 0; lf < 6; ++lf) {
        int fc[2][2];
        face_corners(lf, fc);
        int64_t *k = fk + 4 * (e * 6 + lf);
        k[0] = m->elem[e * 8 + fc[0][0]]; k[1] = m->elem[e * 8 + fc[1][0]];
        k[2] = m->elem[e * 8 + fc[0][1]]; k[3] = m->elem[e * 8 + fc[1][1]];
        qsort(k, 4, sizeof(int64_t), cmp_i64);
      }
    int64_t *sorted = (int64_t *)malloc(sizeof(int64_t) * 4 * m->nel * 6);
    memcpy(sorted, fk, sizeof(int64_t) * 4 * m->nel * 6);
    qsort(sorted, m->nel * 6, 4 * sizeof(int64_t), cmp_key4);
    int64_t nf = 0;
    for (int64_t i = 0; i < m->nel * 6; ++i)
      if (i == 0 || cmp_key4(sorted + 4 * i, sorted + 4 * (nf - 1)) != 0) {
        memmove(sorted + 4 * nf, sorted + 4 * i, 4 * sizeof(int64_t));
        ++nf;
      }
    t->nf = nf;
    t->faces = sorted;
    t->el_face = (int64_t *)malloc(sizeof(int64_t) * m->nel * 6);
    for (int64_t i = 0; i < m->nel * 6; ++i) t->el_face[i] = find_key4(sorted, nf, fk + 4 * i);
    free(fk);
  }
  return ORC_OK;
}

/* Face frame (App. A.2/A.4) of local face lf of element e: o = min vid on the face; n1 = the
 * smaller-id face-neighbour of o, n2 the other; axis1: o->n1, axis2: o->n2.  Output: swap = 0 if
 * axis1 <-> u (u < v the two in-face axes), 1 if axis1 <-> v; s1, s2 = +-1 directions. */
typedef struct { int swap, s1, s2; } frame_t;

static frame_t face_frame(const orc_mesh *m, int64_t e, int lf) {
  int fc[2][2];
  face_corners(lf, fc);
  const int64_t *ev = m->elem + e * 8;
  int a0 = 0, b0 = 0;
  int64_t best = ev[fc[0][0]];
  for (int al = 0; al < 2; ++al)
    for (int be = 0; be < 2; ++be)
      if (ev[fc[al][be]] < best) { best = ev[fc[al][be]]; a0 = al; b0 = be; }
  int64_t nu = ev[fc[1 - a0][b0]]; /* neighbour across u */
  int64_t nvv = ev[fc[a0][1 - b0]]; /* neighbour across v */
  frame_t f;
  if (nu < nvv) { /* n1 at (1-a0, b0): axis1 <-> u */
    f.swap = 0; f.s1 = (a0 == 0) ? 1 : -1; f.s2 = (b0 == 0) ? 1 : -1;
  } else {        /* axis1 <-> v, axis2 <-> u */
    f.swap = 1; f.s1 = (b0 == 0) ? 1 : -1; f.s2 = (a0 == 0) ? 1 : -1;
  }
  return f;
}

static int64_t ipow(int64_t b, int e) { int64_t r = 1; while (e--) r *= b; return r; }

static int64_t space_ndof_canonical(const topo_t *t, int space) {
  int p = t->p;
  if (t->dim == 2 && space != ORC_H1) return t->ne * p + t->nel * 2 * (int64_t)p * (p - 1); /* 2D ND / RT */
  if (t->dim == 2) return t->nv + t->ne * (p - 1) + t->nel * (int64_t)(p - 1) * (p - 1);
  if (space == ORC_H1)
    return t->nv + t->ne * (p - 1) + t->nf * (int64_t)(p - 1) * (p - 1) + t->nel * ipow(p - 1, 3);
  if (space == ORC_ND)
    return t->ne * p + t->nf * 2 * (int64_t)p * (p - 1) + t->nel * 3 * (int64_t)p * (p - 1) * (p - 1);
  return t->nf * (int64_t)p * p + t->nel * 3 * (int64_t)p * p * (p - 1);
}

static int ndof_per_el(int dim, int p, int space) {
  if (space == ORC_H1) return (int)ipow(p + 1, dim);
  if (dim == 2) return 2 * p * (p + 1); /* 2D ND / RT: two families of lattice edges */
  if (space == ORC_ND) return 3 * p * (p + 1) * (p + 1);
  return 3 * p * p * (p + 1);
}

/* Canonical (single-rank) global id and sign of local dof `l` of element e (App. A.3/A.4). */
static void canonical_dof(const orc_mesh *m, const topo_t *t, int space, int64_t e, int l,
                          int64_t *gid, int *sgn) {
  int p = m->p, dim = m->dim;
  int nc = 1 << dim;
  const int64_t *ev = m->elem + e * nc;
  *sgn = 1;
  if (space == ORC_H1) {
    int x[3] = {0, 0, 0};
    int r = l;
    for (int d = 0; d < dim; ++d) { x[d] = r % (p + 1); r /= (p + 1); }
    int nb = 0, bd[3];
    for (int d = 0; d < dim; ++d) { bd[d] = (x[d] == 0 || x[d] == p); nb += bd[d]; }
    if (nb == dim) { /* vertex */
      int c = 0;
      for (int d = 0; d < dim; ++d) c |= (x[d] == p) << d;
      *gid = ev[c];
      return;
    }
    if (nb == dim - 1) { /* edge interior: the one free axis d */
      int d = 0;
      for (int a = 0; a < dim; ++a) if (!bd[a]) d = a;
      int le;
      if (dim == 3) {
        int u = (d == 0) ? 1 : 0, v = (d == 2) ? 1 : 2;
        le = 4 * d + (x[u] == p) + 2 * (x[v] == p);
      } else {
        le = 2 * d + (x[1 - d] == p);
      }
      int tl, hd;
      edge_corners(dim, le, &tl, &hd);
      int64_t E = t->el_edge[e * (dim == 3 ? 12 : 4) + le];
      int tt = (ev[tl] < ev[hd]) ? x[d] : p - x[d];
      *gid = t->nv + E * (p - 1) + (tt - 1);
      return;
    }
    if (dim == 3 && nb == 1) { /* face interior */
      int d = 0;
      for (int a = 0; a < 3; ++a) if (bd[a]) d = a;
      int lf = 2 * d + (x[d] == p);
      int u = (d == 0) ? 1 : 0, v = (d == 2) ? 1 : 2;
      frame_t f = face_frame(m, e, lf);
      int c1 = f.swap ? x[v] : x[u], c2 = f.swap ? x[u] : x[v];
      int i1 = f.s1 > 0 ? c1 : p - c1, i2 = f.s2 > 0 ? c2 : p - c2;
      int64_t F = t->el_face[e * 6 + lf];
      *gid = t->nv + t->ne * (p - 1) + F * (int64_t)(p - 1) * (p - 1) + (i1 - 1) + (int64_t)(p - 1) * (i2 - 1);
      return;
    }
    /* element interior */
    int64_t base = t->nv + t->ne * (p - 1) + (dim == 3 ? t->nf * (int64_t)(p - 1) * (p - 1) : 0);
    int64_t lex = 0, stride = 1;
    for (int d = 0; d < dim; ++d) { lex += (x[d] - 1) * stride; stride *= (p - 1); }
    *gid = base + e * ipow(p - 1, dim) + lex;
    return;
  }
  if (dim == 2) { /* 2D ND / RT (reading P-29): dofs on lattice edges */
    int blk = p * (p + 1);
    int d = l / blk, r = l % blk, o = 1 - d, x[2];
    int ext0 = (space == ORC_ND) ? (d == 0 ? p : p + 1) : (d == 0 ? p + 1 : p);
    x[0] = r % ext0;
    x[1] = r / ext0;
    /* ND family d: edges along d (cell index along d); RT family d: normal e_d, edges along o */
    int along = (space == ORC_ND) ? d : o, across = 1 - along;
    if (x[across] == 0 || x[across] == p) { /* on a coarse edge along `along` */
      int le = 2 * along + (x[across] == p);
      int tl, hd;
      edge_corners(2, le, &tl, &hd);
      int aligned = ev[tl] < ev[hd];
      int k = aligned ? x[along] : p - 1 - x[along];
      *gid = t->el_edge[e * 4 + le] * p + k;
      /* ND: tangent in the global orientation; RT: global normal = the global tangent turned by
       * +90 degrees, against the local normal +e_d (= the local +axis tangent turned: +1 for d = y,
       * -1 for d = x) */
      *sgn = (aligned ? 1 : -1) * ((space == ORC_RT && d == 0) ? -1 : 1);
      return;
    }
    int lex = (space == ORC_ND) ? (d == 0 ? x[0] + p * (x[1] - 1) : (x[0] - 1) + (p - 1) * x[1])
                                : (d == 0 ? (x[0] - 1) + (p - 1) * x[1] : x[0] + p * (x[1] - 1));
    *gid = t->ne * p + e * 2 * (int64_t)p * (p - 1) + d * (int64_t)p * (p - 1) + lex;
    return;
  }
  if (space == ORC_ND) {
    int blk = p * (p + 1) * (p + 1);
    int d = l / blk, r = l % blk;
    int ext[3], x[3];
    for (int a = 0; a < 3; ++a) ext[a] = (a == d) ? p : p + 1;
    for (int a = 0; a < 3; ++a) { x[a] = r % ext[a]; r /= ext[a]; }
    int u = (d == 0) ? 1 : 0, v = (d == 2) ? 1 : 2;
    int bu = (x[u] == 0 || x[u] == p), bv = (x[v] == 0 || x[v] == p);
    if (bu && bv) { /* on a coarse edge along d */
      int le = 4 * d + (x[u] == p) + 2 * (x[v] == p);
      int tl, hd;
      edge_corners(3, le, &tl, &hd);
      int aligned = ev[tl] < ev[hd];
      int k = aligned ? x[d] : p - 1 - x[d];
      *gid = t->el_edge[e * 12 + le] * p + k;
      *sgn = aligned ? 1 : -1;
      return;
    }
    if (bu || bv) { /* interior of a coarse face with normal n */
      int n = bu ? u : v;
      int lf = 2 * n + (x[n] == p);
      int fu = (n == 0) ? 1 : 0, fv = (n == 2) ? 1 : 2; /* in-face axes, increasing */
      frame_t f = face_frame(m, e, lf);
      int ax1 = f.swap ? fv : fu, ax2 = f.swap ? fu : fv;
      int64_t base = t->ne * p + t->el_face[e * 6 + lf] * 2 * (int64_t)p * (p - 1);
      if (d == ax1) { /* axis1-parallel: cell index along axis1, vertex index along axis2 */
        int i1c = f.s1 > 0 ? x[ax1] : p - 1 - x[ax1];
        int i2 = f.s2 > 0 ? x[ax2] : p - x[ax2];
        *gid = base + i1c + (int64_t)p * (i2 - 1);
        *sgn = f.s1;
      } else {        /* axis2-parallel */
        int i2c = f.s2 > 0 ? x[ax2] : p - 1 - x[ax2];
        int i1 = f.s1 > 0 ? x[ax1] : p - x[ax1];
        *gid = base + (int64_t)p * (p - 1) + i2c + (int64_t)p * (i1 - 1);
        *sgn = f.s2;
      }
      return;
    }
    /* element interior: lex_d x-fastest over (cell along d: range p; vertex-1 elsewhere: p-1) */
    int64_t lex = 0, stride = 1;
    for (int a = 0; a < 3; ++a) {
      int c = (a == d) ? x[a] : x[a] - 1, rg = (a == d) ? p : p - 1;
      lex += c * stride;
      stride *= rg;
    }
    *gid = t->ne * p + t->nf * 2 * (int64_t)p * (p - 1) + e * 3 * (int64_t)p * (p - 1) * (p - 1) +
           d * (int64_t)p * (p - 1) * (p - 1) + lex;
    return;
  }
  /* RT */
  {
    int blk = (p + 1) * p * p;
    int d = l / blk, r = l % blk;
    int ext[3], x[3];
    for (int a = 0; a < 3; ++a) ext[a] = (a == d) ? p + 1 : p;
    for (int a = 0; a < 3; ++a) { x[a] = r % ext[a]; r /= ext[a]; }
    if (x[d] == 0 || x[d] == p) { /* on coarse face (d, side) */
      int lf = 2 * d + (x[d] == p);
      int u = (d == 0) ? 1 : 0, v = (d == 2) ? 1 : 2;
      frame_t f = face_frame(m, e, lf);
      int c1 = f.swap ? x[v] : x[u], c2 = f.swap ? x[u] : x[v];
      int i1c = f.s1 > 0 ? c1 : p - 1 - c1, i2c = f.s2 > 0 ? c2 : p - 1 - c2;
      static const int eps_d[3] = {1, -1, 1};
      *gid = t->el_face[e * 6 + lf] * (int64_t)p * p + i1c + (int64_t)p * i2c;
      *sgn = f.s1 * f.s2 * (f.swap ? -1 : 1) * eps_d[d];
      return;
    }
    int64_t lex = 0, stride = 1;
    for (int a = 0; a < 3; ++a) {
      int c = (a == d) ? x[a] - 1 : x[a], rg = (a == d) ? p - 1 : p;
      lex += c * stride;
      stride *= rg;
    }
    *gid = t->nf * (int64_t)p * p + e * 3 * (int64_t)p * p * (p - 1) + d * (int64_t)p * p * (p - 1) + lex;
  }
}

/* Full numbering with ownership and rank-major renumbering (App. A.6):
 * owner(g) = rank of the minimal element containing g;
 * new id  = offset[owner] + position of g among the owner's dofs in canonical order. */
typedef struct {
  int64_t n;          /* global dofs */
  int ndpe;
  int64_t *map;       /* [nel][ndpe] new global ids */
  int8_t *sign;       /* [nel][ndpe] */
  int64_t *rank_off;  /* [nranks+1] */
} numbering_t;

static void numbering_free(numbering_t *nb) {
  free(nb->map); free(nb->sign); free(nb->rank_off);
  memset(nb, 0, sizeof(*nb));
}

static int elem_rank(const orc_mesh *m, int64_t e) {
  if (m->nranks <= 1 || !m->erb) return 0;
  for (int r = 0; r < m->nranks; ++r)
    if (e >= m->erb[r] && e < m->erb[r + 1]) return r;
  return m->nranks - 1;
}

static int numbering_build(const orc_mesh *m, const topo_t *t, int space, numbering_t *nb) {
  memset(nb, 0, sizeof(*nb));
  int nr = (m->nranks > 0) ? m->nranks : 1;
  int64_t n = space_ndof_canonical(t, space);
  int ndpe = ndof_per_el(m->dim, m->p, space);
  nb->n = n; nb->ndpe = ndpe;
  nb->map = (int64_t *)malloc(sizeof(int64_t) * m->nel * ndpe);
  nb->sign = (int8_t *)malloc(m->nel * ndpe);
  nb->rank_off = (int64_t *)calloc(nr + 1, sizeof(int64_t));
  int *owner = (int *)malloc(sizeof(int) * n);
  int8_t *seen_sign = (int8_t *)calloc(n, 1);
  if (!nb->map || !nb->sign || !owner || !seen_sign) return ORC_ERR_MEM;
  for (int64_t g = 0; g < n; ++g) owner[g] = -1;
  for (int64_t e = 0; e < m->nel; ++e) { /* increasing e: first visit = minimal element */
    int r = elem_rank(m, e);
    for (int l = 0; l < ndpe; ++l) {
      int64_t g; int s;
      canonical_dof(m, t, space, e, l, &g, &s);
      if (g < 0 || g >= n) {
        snprintf(g_err, sizeof g_err, "dof id out of range e=%lld l=%d", (long long)e, l);
        free(owner); free(seen_sign);
        return ORC_ERR_INCONSISTENT;
      }
      nb->map[e * ndpe + l] = g;
      nb->sign[e * ndpe + l] = (int8_t)s;
      if (owner[g] < 0) owner[g] = r;
    }
  }
  int64_t *cnt = (int64_t *)calloc(nr, sizeof(int64_t));
  for (int64_t g = 0; g < n; ++g) {
    if (owner[g] < 0) {
      snprintf(g_err, sizeof g_err, "dof %lld never visited", (long long)g);
      free(owner); free(seen_sign); free(cnt);
      return ORC_ERR_INCONSISTENT;
    }
    cnt[owner[g]]++;
  }
  for (int r = 0; r < nr; ++r) nb->rank_off[r + 1] = nb->rank_off[r] + cnt[r];
  int64_t *newid = (int64_t *)malloc(sizeof(int64_t) * n);
  int64_t *pos = (int64_t *)calloc(nr, sizeof(int64_t));
  for (int64_t g = 0; g < n; ++g) newid[g] = nb->rank_off[owner[g]] + pos[owner[g]]++;
  for (int64_t i = 0; i < m->nel * ndpe; ++i) nb->map[i] = newid[nb->map[i]];
  free(owner); free(seen_sign); free(cnt); free(newid); free(pos);
  return ORC_OK;
}

/* ======================================================================================
 * O3: explicit refinement -- the LOR cells of element e and their dofs.
 * ==================================================================================== */
static int h1_lidx(int dim, int p, int i, int j, int k) {
  return (dim == 3) ? i + (p + 1) * (j + (p + 1) * k) : i + (p + 1) * j;
}
/* ND local index of the edge along axis a at cell index c_a, vertex indices elsewhere */
static int nd_lidx(int p, int a, const int *x) {
  int ext[3], r = 0, s = 1;
  for (int b = 0; b < 3; ++b) ext[b] = (b == a) ? p : p + 1;
  for (int b = 0; b < 3; ++b) { r += x[b] * s; s *= ext[b]; }
  return a * p * (p + 1) * (p + 1) + r;
}
/* RT local index of the face with normal a at vertex index x_a, cell indices elsewhere */
static int rt_lidx(int p, int a, const int *x) {
  int ext[3], r = 0, s = 1;
  for (int b = 0; b < 3; ++b) ext[b] = (b == a) ? p + 1 : p;
  for (int b = 0; b < 3; ++b) { r += x[b] * s; s *= ext[b]; }
  return a * (p + 1) * p * p + r;
}

/* The local dofs (macro-element local indices) of LOR cell (kx,ky,kz), in cell-local order. */
static int cell_dofs(int dim, int p, int space, const int *k, int *ldof) {
  if (space == ORC_H1) {
    for (int v = 0; v < (1 << dim); ++v) {
      int a = v & 1, b = (v >> 1) & 1, c = (v >> 2) & 1;
      ldof[v] = h1_lidx(dim, p, k[0] + a, k[1] + b, dim == 3 ? k[2] + c : 0);
    }
    return 1 << dim;
  }
  if (dim == 2) { /* ND: x-edges (b) -> b, y-edges (a) -> 2 + a; RT: faces 2d + side, normal +e_d */
    for (int i = 0; i < 4; ++i) {
      int fam = i / 2, off = i & 1, x[2] = {k[0], k[1]};
      if (space == ORC_ND) x[1 - fam] += off;
      else x[fam] += off;
      int ext0 = (space == ORC_ND) ? (fam == 0 ? p : p + 1) : (fam == 0 ? p + 1 : p);
      ldof[i] = fam * p * (p + 1) + x[0] + ext0 * x[1];
    }
    return 4;
  }
  if (space == ORC_ND) {
    for (int eps = 0; eps < 12; ++eps) {
      int a = eps / 4, b1 = eps & 1, b2 = (eps >> 1) & 1;
      int u = (a == 0) ? 1 : 0, v = (a == 2) ? 1 : 2;
      int x[3] = {k[0], k[1], k[2]};
      x[u] += b1;
      x[v] += b2;
      ldof[eps] = nd_lidx(p, a, x);
    }
    return 12;
  }
  for (int f = 0; f < 6; ++f) {
    int a = f / 2, side = f & 1;
    int x[3] = {k[0], k[1], k[2]};
    x[a] += side;
    ldof[f] = rt_lidx(p, a, x);
  }
  return 6;
}

/* the 2^d corner coordinates of LOR cell k of element e, copied from the E-vector */
static void cell_corners(const orc_mesh *m, int64_t e, const int *k, double *corners) {
  int p = m->p, dim = m->dim;
  int64_t np = ipow(p + 1, dim);
  const double *Xe = m->X + e * dim * np;
  for (int v = 0; v < (1 << dim); ++v) {
    int a = v & 1, b = (v >> 1) & 1, c = (v >> 2) & 1;
    int li = h1_lidx(dim, p, k[0] + a, k[1] + b, dim == 3 ? k[2] + c : 0);
    for (int d = 0; d < dim; ++d) corners[v * dim + d] = Xe[d * np + li];
  }
}

/* the 2^d corner values of LOR cell k of element e of a scalar E-vector c [nel][(p+1)^dim] (NULL:
 * returns NULL -- constant coefficients) */
static const double *cell_coefs(const orc_mesh *m, const double *c, int64_t e, const int *k, double *out) {
  if (!c) return NULL;
  int p = m->p, dim = m->dim;
  int64_t np = ipow(p + 1, dim);
  for (int v = 0; v < (1 << dim); ++v) {
    int a = v & 1, b = (v >> 1) & 1, cc = (v >> 2) & 1;
    out[v] = c[e * np + h1_lidx(dim, p, k[0] + a, k[1] + b, dim == 3 ? k[2] + cc : 0)];
  }
  return out;
}

/* ======================================================================================
 * O5/O6: triplets and sort-and-sum into CSR.
 * ==================================================================================== */
typedef struct { int64_t r, c; double v; } trip_t;

static int cmp_trip(const void *a, const void *b) {
  const trip_t *x = (const trip_t *)a, *y = (const trip_t *)b;
  if (x->r != y->r) return (x->r > y->r) - (x->r < y->r);
  if (x->c != y->c) return (x->c > y->c) - (x->c < y->c);
  return 0;
}

/* Reduce sorted triplets into CSR over the distinct rows present.  Sums each run of equal
 * (row, col) left-to-right; never prunes zeros (reading P-3). */
static int triplets_to_csr(trip_t *T, int64_t nt, orc_csr *out) {
  qsort(T, nt, sizeof(trip_t), cmp_trip);
  int64_t nnz = 0, nrows = 0;
  for (int64_t i = 0; i < nt; ++i) {
    if (i == 0 || T[i].r != T[i - 1].r || T[i].c != T[i - 1].c) nnz++;
    if (i == 0 || T[i].r != T[i - 1].r) nrows++;
  }
  out->n_rows = nrows;
  out->nnz = nnz;
  out->row_ptr = (int64_t *)malloc(sizeof(int64_t) * (nrows + 1));
  out->row_id = (int64_t *)malloc(sizeof(int64_t) * (nrows > 0 ? nrows : 1));
  out->col = (int32_t *)malloc(sizeof(int32_t) * (nnz > 0 ? nnz : 1));
  out->val = (double *)malloc(sizeof(double) * (nnz > 0 ? nnz : 1));
  if (!out->row_ptr || !out->row_id || !out->col || !out->val) return ORC_ERR_MEM;
  int64_t k = -1, r = -1;
  for (int64_t i = 0; i < nt; ++i) {
    if (i == 0 || T[i].r != T[i - 1].r) {
      ++r;
      out->row_id[r] = T[i].r;
      out->row_ptr[r] = k + 1;
    }
    if (i == 0 || T[i].r != T[i - 1].r || T[i].c != T[i - 1].c) {
      ++k;
      out->col[k] = (int32_t)T[i].c;
      out->val[k] = T[i].v;
    } else {
      out->val[k] += T[i].v;
    }
  }
  out->row_ptr[nrows] = nnz;
  return ORC_OK;
}

void orc_free(orc_csr *c) {
  if (!c) return;
  free(c->row_ptr); free(c->row_id); free(c->col); free(c->val);
  memset(c, 0, sizeof(*c));
}

static int ncells_dim(int p, int dim) { return (int)ipow(p, dim); }

static void cell_index(int p, int dim, int ic, int *k) {
  k[0] = ic % p; k[1] = (ic / p) % p; k[2] = (dim == 3) ? ic / (p * p) : 0;
}

static int check_mesh(const orc_mesh *m, int space) {
  if (!m || !(m->dim == 2 || m->dim == 3) || m->p < 1 || m->nel < 1 || !m->elem || !m->X) {
    snprintf(g_err, sizeof g_err, "invalid mesh");
    return ORC_ERR_ARG;
  }
  (void)space;
  return ORC_OK;
}

/* The full matrix A_S over all global rows (new, rank-major ids). */
int orc_assemble(const orc_mesh *m, int space, int quad, double alpha, double beta, orc_csr *out) {
  memset(out, 0, sizeof(*out));
  int rc = check_mesh(m, space);
  if (rc) return rc;
  topo_t t;
  if ((rc = topo_build(m, &t))) return rc;
  numbering_t nb;
  if ((rc = numbering_build(m, &t, space, &nb))) { topo_free(&t); return rc; }
  int nloc = local_ndof(m->dim, space), nc = ncells_dim(m->p, m->dim);
  int64_t nt = m->nel * (int64_t)nc * nloc * nloc;
  trip_t *T = (trip_t *)malloc(sizeof(trip_t) * nt);
  if (!T) { topo_free(&t); numbering_free(&nb); return ORC_ERR_MEM; }
  int64_t it = 0;
  double A[144], corners[24], ca8[8], cb8[8];
  int ldof[12];
  for (int64_t e = 0; e < m->nel; ++e)
    for (int ic = 0; ic < nc; ++ic) {
      int k[3];
      cell_index(m->p, m->dim, ic, k);
      cell_corners(m, e, k, corners);
      if (orc_local_matrix_vc(m->dim, space, quad, alpha, beta, corners, cell_coefs(m, m->ca, e, k, ca8),
                              cell_coefs(m, m->cb, e, k, cb8), A)) {
        snprintf(g_err, sizeof g_err, "degenerate-geometry(e=%lld, kx=%d, ky=%d, kz=%d)", (long long)e, k[0],
                 k[1], k[2]);
        free(T); topo_free(&t); numbering_free(&nb);
        return ORC_ERR_DEGENERATE;
      }
      cell_dofs(m->dim, m->p, space, k, ldof);
      for (int i = 0; i < nloc; ++i)
        for (int j = 0; j < nloc; ++j) {
          int64_t gi = nb.map[e * nb.ndpe + ldof[i]], gj = nb.map[e * nb.ndpe + ldof[j]];
          double s = (double)nb.sign[e * nb.ndpe + ldof[i]] * (double)nb.sign[e * nb.ndpe + ldof[j]];
          T[it].r = gi; T[it].c = gj; T[it].v = s * A[i * nloc + j];
          ++it;
        }
    }
  rc = triplets_to_csr(T, nt, out);
  out->n_cols = nb.n;
  free(T); topo_free(&t); numbering_free(&nb);
  return rc;
}

/* O10: row oracle.  For each requested global row g, visit only the LOR cells incident to g
 * (via the oracle's own transpose) and run O4-O6 restricted to row g. */
int orc_assemble_rows(const orc_mesh *m, int space, int quad, double alpha, double beta, int64_t nreq,
                      const int64_t *rows, orc_csr *out) {
  memset(out, 0, sizeof(*out));
  int rc = check_mesh(m, space);
  if (rc) return rc;
  topo_t t;
  if ((rc = topo_build(m, &t))) return rc;
  numbering_t nb;
  if ((rc = numbering_build(m, &t, space, &nb))) { topo_free(&t); return rc; }
  /* transpose: dof -> list of (e*ndpe + l) by counting sort */
  int64_t n = nb.n, ne_l = m->nel * (int64_t)nb.ndpe;
  int64_t *off = (int64_t *)calloc(n + 1, sizeof(int64_t));
  int64_t *ent = (int64_t *)malloc(sizeof(int64_t) * ne_l);
  for (int64_t i = 0; i < ne_l; ++i) off[nb.map[i] + 1]++;
  for (int64_t g = 0; g < n; ++g) off[g + 1] += off[g];
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * n);
  memcpy(fill, off, sizeof(int64_t) * n);
  for (int64_t i = 0; i < ne_l; ++i) ent[fill[nb.map[i]]++] = i;
  free(fill);
  int nloc = local_ndof(m->dim, space), nc = ncells_dim(m->p, m->dim);
  int64_t cap = 1024, nt = 0;
  trip_t *T = (trip_t *)malloc(sizeof(trip_t) * cap);
  double A[144], corners[24], ca8[8], cb8[8];
  int ldof[12];
  for (int64_t q = 0; q < nreq; ++q) {
    int64_t g = rows[q];
    if (g < 0 || g >= n) { rc = ORC_ERR_ARG; snprintf(g_err, sizeof g_err, "row out of range"); break; }
    for (int64_t s = off[g]; s < off[g + 1]; ++s) {
      int64_t e = ent[s] / nb.ndpe;
      int l = (int)(ent[s] % nb.ndpe);
      /* cells of e containing local dof l: scan all cells of e (slow and obviously complete) */
      for (int ic = 0; ic < nc; ++ic) {
        int k[3];
        cell_index(m->p, m->dim, ic, k);
        cell_dofs(m->dim, m->p, space, k, ldof);
        int li = -1;
        for (int i = 0; i < nloc; ++i) if (ldof[i] == l) li = i;
        if (li < 0) continue;
        cell_corners(m, e, k, corners);
        if (orc_local_matrix_vc(m->dim, space, quad, alpha, beta, corners, cell_coefs(m, m->ca, e, k, ca8),
                                cell_coefs(m, m->cb, e, k, cb8), A)) { rc = ORC_ERR_DEGENERATE; break; }
        for (int j = 0; j < nloc; ++j) {
          if (nt == cap) { cap *= 2; T = (trip_t *)realloc(T, sizeof(trip_t) * cap); }
          int64_t gj = nb.map[e * nb.ndpe + ldof[j]];
          double sg = (double)nb.sign[e * nb.ndpe + l] * (double)nb.sign[e * nb.ndpe + ldof[j]];
          T[nt].r = g; T[nt].c = gj; T[nt].v = sg * A[li * nloc + j];
          ++nt;
        }
      }
    }
  }
  if (!rc) rc = triplets_to_csr(T, nt, out);
  out->n_cols = n;
  free(T); free(off); free(ent); topo_free(&t); numbering_free(&nb);
  return rc;
}

/* ======================================================================================
 * O2 outputs for T1: the element->dof map, signs and per-rank row ranges.
 * ==================================================================================== */
int orc_space_size(const orc_mesh *m, int space, int64_t *n, int *ndpe, int64_t *rank_off) {
  int rc = check_mesh(m, space);
  if (rc) return rc;
  topo_t t;
  if ((rc = topo_build(m, &t))) return rc;
  numbering_t nb;
  if ((rc = numbering_build(m, &t, space, &nb))) { topo_free(&t); return rc; }
  *n = nb.n;
  *ndpe = nb.ndpe;
  int nr = m->nranks > 0 ? m->nranks : 1;
  if (rank_off) memcpy(rank_off, nb.rank_off, sizeof(int64_t) * (nr + 1));
  topo_free(&t); numbering_free(&nb);
  return ORC_OK;
}

int orc_dof_map(const orc_mesh *m, int space, int32_t *map, int8_t *sign) {
  int rc = check_mesh(m, space);
  if (rc) return rc;
  topo_t t;
  if ((rc = topo_build(m, &t))) return rc;
  numbering_t nb;
  if ((rc = numbering_build(m, &t, space, &nb))) { topo_free(&t); return rc; }
  for (int64_t i = 0; i < m->nel * (int64_t)nb.ndpe; ++i) {
    map[i] = (int32_t)nb.map[i];
    if (sign) sign[i] = nb.sign[i];
  }
  topo_free(&t); numbering_free(&nb);
  return ORC_OK;
}

/* coarse entity counts (nv, ne, nf) for pins */
int orc_topology_counts(const orc_mesh *m, int64_t *counts) {
  topo_t t;
  int rc = topo_build(m, &t);
  if (rc) return rc;
  counts[0] = t.nv; counts[1] = t.ne; counts[2] = t.nf;
  topo_free(&t);
  return ORC_OK;
}

/* ======================================================================================
 * O7: discrete gradient (Algorithm 1) and discrete curl (l.440-445).
 * which = 0: G (rows = ND dofs, cols = H1 dofs): row of LOR edge i: -sigma at the H1 id of
 *            its local tail, +sigma at its head; columns sorted (reading P-5).
 * which = 1: C (rows = RT dofs, cols = ND dofs): row of LOR face (d, side): cyclic in-face axes
 *            (u',v') = (d+1, d+2) mod 3; local circulation signs +1 (u'-edge at v'=0),
 *            +1 (v'-edge at u'=1), -1 (u'-edge at v'=1), -1 (v'-edge at u'=0); times
 *            sigma_face * sigma_edge (App. A.5, reading P-15).
 * Every revisit of a row from another cell/element must produce the identical row.
 * ==================================================================================== */
static int discrete_2d(const orc_mesh *m, int which, orc_csr *out);
int orc_discrete(const orc_mesh *m, int which, orc_csr *out) {
  memset(out, 0, sizeof(*out));
  if (m && m->dim == 2 && m->p >= 1 && (which == 0 || which == 2)) return discrete_2d(m, which, out);
  if (!m || m->dim != 3 || m->p < 1 || which == 2) { snprintf(g_err, sizeof g_err, "3D only"); return ORC_ERR_ARG; }
  topo_t t;
  int rc = topo_build(m, &t);
  if (rc) return rc;
  int rsp = which == 0 ? ORC_ND : ORC_RT, csp = which == 0 ? ORC_H1 : ORC_ND;
  numbering_t nr, ncn;
  if ((rc = numbering_build(m, &t, rsp, &nr))) { topo_free(&t); return rc; }
  if ((rc = numbering_build(m, &t, csp, &ncn))) { topo_free(&t); numbering_free(&nr); return rc; }
  int w = which == 0 ? 2 : 4;
  int64_t n = nr.n;
  int64_t *cols = (int64_t *)malloc(sizeof(int64_t) * n * w);
  double *vals = (double *)malloc(sizeof(double) * n * w);
  char *done = (char *)calloc(n, 1);
  int p = m->p, nc = ncells_dim(p, 3);
  for (int64_t e = 0; e < m->nel && !rc; ++e)
    for (int ic = 0; ic < nc && !rc; ++ic) {
      int k[3];
      cell_index(p, 3, ic, k);
      int nloc_r = which == 0 ? 12 : 6;
      int ldof_r[12];
      cell_dofs(3, p, rsp, k, ldof_r);
      for (int i = 0; i < nloc_r; ++i) {
        int64_t row = nr.map[e * nr.ndpe + ldof_r[i]];
        double sr = nr.sign[e * nr.ndpe + ldof_r[i]];
        int64_t c[4];
        double v[4];
        if (which == 0) {
          int tl, hd;
          edge_corners(3, i, &tl, &hd); /* cell-local edge order == 4a + b1 + 2b2 */
          int ta = tl & 1, tb = (tl >> 1) & 1, tc = (tl >> 2) & 1;
          int ha = hd & 1, hb = (hd >> 1) & 1, hc = (hd >> 2) & 1;
          c[0] = ncn.map[e * ncn.ndpe + h1_lidx(3, p, k[0] + ta, k[1] + tb, k[2] + tc)];
          c[1] = ncn.map[e * ncn.ndpe + h1_lidx(3, p, k[0] + ha, k[1] + hb, k[2] + hc)];
          v[0] = -sr;
          v[1] = sr;
        } else {
          int d = i / 2, side = i & 1;
          int up = (d + 1) % 3, vp = (d + 2) % 3;
          /* the four edges: (axis, offset along the other in-face axis, local sign) */
          int eax[4] = {up, vp, up, vp};
          int eoff[4] = {0, 1, 1, 0};
          double es[4] = {1.0, 1.0, -1.0, -1.0};
          for (int q = 0; q < 4; ++q) {
            int x[3] = {k[0], k[1], k[2]};
            x[d] += side;
            int other = (eax[q] == up) ? vp : up;
            x[other] += eoff[q];
            int le = nd_lidx(p, eax[q], x);
            c[q] = ncn.map[e * ncn.ndpe + le];
            v[q] = es[q] * sr * (double)ncn.sign[e * ncn.ndpe + le];
          }
        }
        /* sort the w entries by column (insertion sort) */
        for (int a = 1; a < w; ++a)
          for (int b = a; b > 0 && c[b] < c[b - 1]; --b) {
            int64_t tc = c[b]; c[b] = c[b - 1]; c[b - 1] = tc;
            double tv = v[b]; v[b] = v[b - 1]; v[b - 1] = tv;
          }
        if (done[row]) {
          for (int a = 0; a < w; ++a)
            if (cols[row * w + a] != c[a] || vals[row * w + a] != v[a]) {
              snprintf(g_err, sizeof g_err, "inconsistent %s row %lld", which ? "C" : "G", (long long)row);
              rc = ORC_ERR_INCONSISTENT;
            }
        } else {
          done[row] = 1;
          for (int a = 0; a < w; ++a) { cols[row * w + a] = c[a]; vals[row * w + a] = v[a]; }
        }
      }
    }
  if (!rc) {
    out->n_rows = n;
    out->n_cols = ncn.n;
    out->nnz = n * w;
    out->row_ptr = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    out->row_id = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    out->col = (int32_t *)malloc(sizeof(int32_t) * n * w);
    out->val = (double *)malloc(sizeof(double) * n * w);
    for (int64_t r = 0; r <= n; ++r) out->row_ptr[r] = r * w;
    for (int64_t r = 0; r < n; ++r) {
      out->row_id[r] = r;
      if (!done[r]) { rc = ORC_ERR_INCONSISTENT; snprintf(g_err, sizeof g_err, "row never visited"); }
    }
    for (int64_t i = 0; i < n * w; ++i) { out->col[i] = (int32_t)cols[i]; out->val[i] = vals[i]; }
  }
  free(cols); free(vals); free(done);
  topo_free(&t); numbering_free(&nr); numbering_free(&ncn);
  return rc;
}

/* 2D discrete gradient (which = 0: rows ND, Algorithm 1: -sigma at the LOR edge's tail, +sigma at its
 * head) and rotated gradient (which = 2: rows RT; grad-perp = (-d/dy, d/dx): the
 * flux of grad-perp u through an edge with normal n = tau turned by +90 degrees is u(head of tau) -
 * u(tail of tau); the local normal +e_d has tau = +e_x for d = y and tau = -e_y for d = x), times the
 * row's sign; columns sorted; every revisit of a row must give the identical row (reading P-29). */
static int discrete_2d(const orc_mesh *m, int which, orc_csr *out) {
  topo_t t;
  int rc = topo_build(m, &t);
  if (rc) return rc;
  int rsp = which == 0 ? ORC_ND : ORC_RT;
  numbering_t nr, ncn;
  if ((rc = numbering_build(m, &t, rsp, &nr))) { topo_free(&t); return rc; }
  if ((rc = numbering_build(m, &t, ORC_H1, &ncn))) { topo_free(&t); numbering_free(&nr); return rc; }
  int64_t n = nr.n;
  int64_t *cols = (int64_t *)malloc(sizeof(int64_t) * n * 2);
  double *vals = (double *)malloc(sizeof(double) * n * 2);
  char *done = (char *)calloc(n, 1);
  int p = m->p, nc = ncells_dim(p, 2);
  for (int64_t e = 0; e < m->nel && !rc; ++e)
    for (int ic = 0; ic < nc && !rc; ++ic) {
      int k[3];
      cell_index(p, 2, ic, k);
      int ldof[12];
      cell_dofs(2, p, rsp, k, ldof);
      for (int i = 0; i < 4; ++i) {
        int64_t row = nr.map[e * nr.ndpe + ldof[i]];
        double sr = nr.sign[e * nr.ndpe + ldof[i]];
        int fam = i / 2, off = i & 1, ta[2], ha[2]; /* cell-local corners (x, y) of the edge's tail / head */
        if (which == 0) { /* ND edge along fam at offset off across: tail lower end */
          ta[fam] = 0; ha[fam] = 1; ta[1 - fam] = ha[1 - fam] = off;
        } else if (fam == 1) { /* RT normal y: horizontal edge y = off, tau = +e_x */
          ta[0] = 0; ha[0] = 1; ta[1] = ha[1] = off;
        } else { /* RT normal x: vertical edge x = off, tau = -e_y */
          ta[1] = 1; ha[1] = 0; ta[0] = ha[0] = off;
        }
        int64_t c[2] = {ncn.map[e * ncn.ndpe + h1_lidx(2, p, k[0] + ta[0], k[1] + ta[1], 0)],
                        ncn.map[e * ncn.ndpe + h1_lidx(2, p, k[0] + ha[0], k[1] + ha[1], 0)]};
        double v[2] = {-sr, sr};
        if (c[1] < c[0]) {
          int64_t tc = c[0]; c[0] = c[1]; c[1] = tc;
          double tv = v[0]; v[0] = v[1]; v[1] = tv;
        }
        if (done[row]) {
          for (int a = 0; a < 2; ++a)
            if (cols[row * 2 + a] != c[a] || vals[row * 2 + a] != v[a]) {
              snprintf(g_err, sizeof g_err, "inconsistent 2D %s row %lld", which ? "rotated gradient" : "G",
                       (long long)row);
              rc = ORC_ERR_INCONSISTENT;
            }
        } else {
          done[row] = 1;
          for (int a = 0; a < 2; ++a) { cols[row * 2 + a] = c[a]; vals[row * 2 + a] = v[a]; }
        }
      }
    }
  if (!rc) {
    out->n_rows = n;
    out->n_cols = ncn.n;
    out->nnz = n * 2;
    out->row_ptr = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    out->row_id = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    out->col = (int32_t *)malloc(sizeof(int32_t) * n * 2);
    out->val = (double *)malloc(sizeof(double) * n * 2);
    for (int64_t r = 0; r <= n; ++r) out->row_ptr[r] = r * 2;
    for (int64_t r = 0; r < n; ++r) {
      out->row_id[r] = r;
      if (!done[r]) { rc = ORC_ERR_INCONSISTENT; snprintf(g_err, sizeof g_err, "row never visited"); }
    }
    for (int64_t i = 0; i < n * 2; ++i) { out->col[i] = (int32_t)cols[i]; out->val[i] = vals[i]; }
  }
  free(cols); free(vals); free(done);
  topo_free(&t); numbering_free(&nr); numbering_free(&ncn);
  return rc;
}
