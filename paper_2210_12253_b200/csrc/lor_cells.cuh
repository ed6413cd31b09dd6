// lor_cells.cuh -- LOR sub-cell matrices (Step A1), packed symmetric.
//
// Vertex rule (reading P-1: geometric factors at the sub-element vertices):
// at corner q the Jacobian's columns are the cell's edge vectors through q, and only the basis
// functions attached to q are non-zero there, so the cell matrix is a sum of small per-corner
// tensors:
//   H1:  Q = w a adj(J) adj(J)^T / det J;  (q,q) += s^T Q s + w b det J,  (q,q^d) += -s_d (Qs)_d,
//        (q^d,q^d') += s_d s_d' Q_dd'   (s = +-1 reference gradient of N_q, q^d = neighbour along d)
//   ND:  mass  M[E_d(q)][E_d'(q)] += w b (adj adj^T / det)_dd'   (E_d(q): the d-edge through q)
//        curl  K = C^T Mrt C,  Mrt[F_d(q)][F_d'(q)] += w a (J^T J / det)_dd'   (F_d(q): d-face at q)
//   RT:  mass  M[F_d(q)][F_d'(q)] += w b (J^T J / det)_dd';  div  K = (sum_q w a / det_q) d d^T
// The de Rham factorisations used for ND (K_ND = C^T M_RT C) and RT (rank one) hold pointwise for
// the lowest-order reference elements and are pinned against the oracle's textbook matrices
// (tests/test_oracle_pins.py::test_cell_derham_factorizations).
// Gauss-2: the same tensors at the 2^d interior points with all basis values.
#pragma once
#include <utility>

#include "lor_device.cuh"

#ifndef ND_FENCE
#define ND_FENCE 1  // cell_nd_vertex_to: corners between compiler fences
#endif

namespace lorb {

// ---------------------------------------------------------------- reference cell tables (ND/RT)
// cell-local edge eps = 4a + b1 + 2 b2 (direction a, bits b1/b2 along the other axes u < v)
__host__ __device__ constexpr int e_dir(int eps) { return eps / 4; }
__host__ __device__ constexpr int e_u(int eps) { return e_dir(eps) == 0 ? 1 : 0; }
__host__ __device__ constexpr int e_v(int eps) { return e_dir(eps) == 2 ? 1 : 2; }
__host__ __device__ constexpr int e_b1(int eps) { return eps & 1; }
__host__ __device__ constexpr int e_b2(int eps) { return (eps >> 1) & 1; }
// the two cell faces containing edge eps: (u, b1) and (v, b2)
__host__ __device__ constexpr int e_face(int eps, int k) { return k == 0 ? 2 * e_u(eps) + e_b1(eps) : 2 * e_v(eps) + e_b2(eps); }
// circulation sign C[f][eps] (App. A.5): cyclic in-face axes (u', v') = (d+1, d+2) mod 3;
// +1 u'-edge at v'=0, +1 v'-edge at u'=1, -1 u'-edge at v'=1, -1 v'-edge at u'=0.
__host__ __device__ constexpr int c_sign(int f, int eps) {
  // f contains eps; d = normal, the edge's position along the other in-face axis decides
  return ((f / 2) == e_u(eps))
             ? ((e_dir(eps) == (e_u(eps) + 1) % 3) ? (e_b2(eps) == 0 ? 1 : -1) : (e_b2(eps) == 1 ? 1 : -1))
             : ((e_dir(eps) == (e_v(eps) + 1) % 3) ? (e_b1(eps) == 0 ? 1 : -1) : (e_b1(eps) == 1 ? 1 : -1));
}
// d-edge through corner q: bits of q along the other two axes
__host__ __device__ constexpr int corner_edge(int q, int d) {
  return 4 * d + ((q >> (d == 0 ? 1 : 0)) & 1) + 2 * ((q >> (d == 2 ? 1 : 2)) & 1);
}

struct Jac3 {
  double j[3][3];  // j[d] = column d of J (edge vector along d)
  double r[3][3];  // r[d] = row d of adj(J) = j[d+1] x j[d+2]
  double det;
};

__device__ __forceinline__ void cross3(const double *a, const double *b, double *c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}
__device__ __forceinline__ double dot3(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

__device__ __forceinline__ void finish_jac(Jac3 &J) {
  cross3(J.j[1], J.j[2], J.r[0]);
  cross3(J.j[2], J.j[0], J.r[1]);
  cross3(J.j[0], J.j[1], J.r[2]);
  J.det = dot3(J.j[0], J.r[0]);
}

// Jacobian at corner q under the vertex rule: column d = X(q with bit d = 1) - X(q with bit d = 0)
__device__ __forceinline__ void jac_corner(const double X[8][3], int q, Jac3 &J) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int hi = q | (1 << d), lo = q & ~(1 << d);
#pragma unroll
    for (int k = 0; k < 3; ++k) J.j[d][k] = X[hi][k] - X[lo][k];
  }
  finish_jac(J);
}

// Jacobian of the trilinear map at reference point (t0, t1, t2)
__device__ __forceinline__ void jac_point(const double X[8][3], const double *t, Jac3 &J) {
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int k = 0; k < 3; ++k) J.j[d][k] = 0.0;
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    double f[3], df[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int b = (v >> a) & 1;
      f[a] = b ? t[a] : 1.0 - t[a];
      df[a] = b ? 1.0 : -1.0;
    }
    const double g0 = df[0] * f[1] * f[2], g1 = f[0] * df[1] * f[2], g2 = f[0] * f[1] * df[2];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      J.j[0][k] += X[v][k] * g0;
      J.j[1][k] += X[v][k] * g1;
      J.j[2][k] += X[v][k] * g2;
    }
  }
  finish_jac(J);
}

__device__ __forceinline__ double gauss2_pt(int bit) { return bit ? 0.78867513459481288225 : 0.21132486540518711775; }

// Variable coefficients ("time-dependent variable coefficients";
// DESIGN.md reading P-28): the multiplier of alpha / beta at quadrature point q of a cell with corner
// values c[NV] (vertex order a + 2b + 4c) -- the corner value under the vertex rule, the multilinear
// interpolant at the Gauss point under Gauss-2.  c == nullptr: constant coefficients, multiplier
// exactly 1.0 (x * 1.0 == x, so the constant-coefficient results are unchanged bit for bit).
template <int QUAD, int NV>
__device__ __forceinline__ double coef_q(const double *c, int q) {
  if (!c) return 1.0;
  if (QUAD == 0) return c[q];
  double s = 0.0;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double f = 1.0;
#pragma unroll
    for (int a = 0; a < (NV == 8 ? 3 : 2); ++a) {
      const double t = gauss2_pt((q >> a) & 1);
      f *= ((v >> a) & 1) ? t : 1.0 - t;
    }
    s += f * c[v];
  }
  return s;
}

// ---------------------------------------------------------------------------- H1, 3D
template <int QUAD>
__device__ __forceinline__ bool cell_h1_3d(const double X[8][3], double alpha, double beta, double *A /*36*/,
                                           const double *ca = nullptr, const double *cb = nullptr) {
#pragma unroll
  for (int i = 0; i < 36; ++i) A[i] = 0.0;
  const double w = 0.125;
  bool ok = true;
  if (QUAD == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      Jac3 J;
      jac_corner(X, q, J);
      ok &= J.det > 0.0;
      const double sa = w * alpha * coef_q<0, 8>(ca, q) / J.det;
      double Q[3][3];
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int e = d; e < 3; ++e) Q[d][e] = Q[e][d] = sa * dot3(J.r[d], J.r[e]);
      double sg[3], Qs[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) sg[d] = ((q >> d) & 1) ? 1.0 : -1.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) Qs[d] = Q[d][0] * sg[0] + Q[d][1] * sg[1] + Q[d][2] * sg[2];
      A[tri(8, q, q)] += (sg[0] * Qs[0] + sg[1] * Qs[1] + sg[2] * Qs[2]) + w * beta * coef_q<0, 8>(cb, q) * J.det;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int qd = q ^ (1 << d);
        A[tri(8, q, qd)] += -sg[d] * Qs[d];
        A[tri(8, qd, qd)] += Q[d][d];
#pragma unroll
        for (int e = d + 1; e < 3; ++e) A[tri(8, qd, q ^ (1 << e))] += sg[d] * sg[e] * Q[d][e];
      }
    }
  } else {
#pragma unroll
    for (int pt = 0; pt < 8; ++pt) {
      const double t[3] = {gauss2_pt(pt & 1), gauss2_pt((pt >> 1) & 1), gauss2_pt((pt >> 2) & 1)};
      Jac3 J;
      jac_point(X, t, J);
      ok &= J.det > 0.0;
      const double sa = w * alpha * coef_q<1, 8>(ca, pt) / J.det;
      double Q[3][3];
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int e = d; e < 3; ++e) Q[d][e] = Q[e][d] = sa * dot3(J.r[d], J.r[e]);
      double N[8], G[8][3];
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        double f[3], df[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const int b = (v >> a) & 1;
          f[a] = b ? t[a] : 1.0 - t[a];
          df[a] = b ? 1.0 : -1.0;
        }
        N[v] = f[0] * f[1] * f[2];
        G[v][0] = df[0] * f[1] * f[2];
        G[v][1] = f[0] * df[1] * f[2];
        G[v][2] = f[0] * f[1] * df[2];
      }
      const double wb = w * beta * coef_q<1, 8>(cb, pt) * J.det;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double QG[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) QG[d] = Q[d][0] * G[i][0] + Q[d][1] * G[i][1] + Q[d][2] * G[i][2];
#pragma unroll
        for (int j = i; j < 8; ++j) A[tri(8, i, j)] += QG[0] * G[j][0] + QG[1] * G[j][1] + QG[2] * G[j][2] + wb * N[i] * N[j];
      }
    }
  }
  return ok;
}

// ---------------------------------------------------------------------------- H1, 2D
template <int QUAD>
__device__ __forceinline__ bool cell_h1_2d(const double X[4][2], double alpha, double beta, double *A /*10*/,
                                           const double *ca = nullptr, const double *cb = nullptr) {
#pragma unroll
  for (int i = 0; i < 10; ++i) A[i] = 0.0;
  const double w = 0.25;
  bool ok = true;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double j0[2], j1[2];
    double t[2] = {0, 0};
    if (QUAD == 0) {
      const int h0 = q | 1, l0 = q & ~1, h1 = q | 2, l1 = q & ~2;
      j0[0] = X[h0][0] - X[l0][0]; j0[1] = X[h0][1] - X[l0][1];
      j1[0] = X[h1][0] - X[l1][0]; j1[1] = X[h1][1] - X[l1][1];
    } else {
      t[0] = gauss2_pt(q & 1);
      t[1] = gauss2_pt((q >> 1) & 1);
      j0[0] = j0[1] = j1[0] = j1[1] = 0.0;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int b0 = v & 1, b1 = (v >> 1) & 1;
        const double f0 = b0 ? t[0] : 1 - t[0], f1 = b1 ? t[1] : 1 - t[1];
        const double g0 = (b0 ? 1.0 : -1.0) * f1, g1 = f0 * (b1 ? 1.0 : -1.0);
        j0[0] += X[v][0] * g0; j0[1] += X[v][1] * g0;
        j1[0] += X[v][0] * g1; j1[1] += X[v][1] * g1;
      }
    }
    const double det = j0[0] * j1[1] - j0[1] * j1[0];
    ok &= det > 0.0;
    const double r0[2] = {j1[1], -j1[0]}, r1[2] = {-j0[1], j0[0]};  // rows of adj(J)
    const double aq = coef_q<QUAD, 4>(ca, q), bq = coef_q<QUAD, 4>(cb, q);
    const double sa = w * alpha * aq / det;
    const double Q00 = sa * (r0[0] * r0[0] + r0[1] * r0[1]);
    const double Q01 = sa * (r0[0] * r1[0] + r0[1] * r1[1]);
    const double Q11 = sa * (r1[0] * r1[0] + r1[1] * r1[1]);
    if (QUAD == 0) {
      const double s0 = (q & 1) ? 1.0 : -1.0, s1 = (q & 2) ? 1.0 : -1.0;
      const double Qs0 = Q00 * s0 + Q01 * s1, Qs1 = Q01 * s0 + Q11 * s1;
      A[tri(4, q, q)] += s0 * Qs0 + s1 * Qs1 + w * beta * bq * det;
      A[tri(4, q, q ^ 1)] += -s0 * Qs0;
      A[tri(4, q, q ^ 2)] += -s1 * Qs1;
      A[tri(4, q ^ 1, q ^ 1)] += Q00;
      A[tri(4, q ^ 2, q ^ 2)] += Q11;
      A[tri(4, q ^ 1, q ^ 2)] += s0 * s1 * Q01;
    } else {
      double N[4], G[4][2];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int b0 = v & 1, b1 = (v >> 1) & 1;
        const double f0 = b0 ? t[0] : 1 - t[0], f1 = b1 ? t[1] : 1 - t[1];
        N[v] = f0 * f1;
        G[v][0] = (b0 ? 1.0 : -1.0) * f1;
        G[v][1] = f0 * (b1 ? 1.0 : -1.0);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = i; j < 4; ++j)
          A[tri(4, i, j)] += G[i][0] * (Q00 * G[j][0] + Q01 * G[j][1]) + G[i][1] * (Q01 * G[j][0] + Q11 * G[j][1]) +
                             w * beta * bq * det * N[i] * N[j];
    }
  }
  return ok;
}

// ------------------------------------------------------------------------ ND (3D): 12 x 12
template <int QUAD>
__device__ __forceinline__ bool cell_nd(const double X[8][3], double alpha, double beta, double *A /*78*/,
                                        const double *ca = nullptr, const double *cb = nullptr) {
#pragma unroll
  for (int i = 0; i < 78; ++i) A[i] = 0.0;
  double M[21];  // 6x6 face "mass" with alpha: curl-curl = C^T M C
#pragma unroll
  for (int i = 0; i < 21; ++i) M[i] = 0.0;
  const double w = 0.125;
  bool ok = true;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    Jac3 J;
    double t[3];
    if (QUAD == 0) jac_corner(X, q, J);
    else {
      t[0] = gauss2_pt(q & 1); t[1] = gauss2_pt((q >> 1) & 1); t[2] = gauss2_pt((q >> 2) & 1);
      jac_point(X, t, J);
    }
    ok &= J.det > 0.0;
    const double sm = w * beta * coef_q<QUAD, 8>(cb, q) / J.det, sc = w * alpha * coef_q<QUAD, 8>(ca, q) / J.det;
    double Qm[3][3], R[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int e = d; e < 3; ++e) {
        Qm[d][e] = Qm[e][d] = sm * dot3(J.r[d], J.r[e]);
        R[d][e] = R[e][d] = sc * dot3(J.j[d], J.j[e]);
      }
    if (QUAD == 0) {
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int e = d; e < 3; ++e) {
          A[tri(12, corner_edge(q, d), corner_edge(q, e))] += Qm[d][e];
          M[tri(6, 2 * d + ((q >> d) & 1), 2 * e + ((q >> e) & 1))] += R[d][e];
        }
    } else {
      double fe[12], hf[6];
#pragma unroll
      for (int eps = 0; eps < 12; ++eps) {
        const double fu = e_b1(eps) ? t[e_u(eps)] : 1 - t[e_u(eps)];
        const double fv = e_b2(eps) ? t[e_v(eps)] : 1 - t[e_v(eps)];
        fe[eps] = fu * fv;
      }
#pragma unroll
      for (int f = 0; f < 6; ++f) hf[f] = (f & 1) ? t[f / 2] : 1 - t[f / 2];
#pragma unroll
      for (int i = 0; i < 12; ++i)
#pragma unroll
        for (int j = i; j < 12; ++j) A[tri(12, i, j)] += fe[i] * fe[j] * Qm[e_dir(i)][e_dir(j)];
#pragma unroll
      for (int f = 0; f < 6; ++f)
#pragma unroll
        for (int g = f; g < 6; ++g) M[tri(6, f, g)] += hf[f] * hf[g] * R[f / 2][g / 2];
    }
  }
  // curl-curl: K_ij = sum_{f in F(i), g in F(j)} C_fi M_fg C_gj
#pragma unroll
  for (int i = 0; i < 12; ++i)
#pragma unroll
    for (int j = i; j < 12; ++j) {
      double k = 0.0;
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int f = e_face(i, a), g = e_face(j, b);
          k += (double)(c_sign(f, i) * c_sign(g, j)) * M[tri(6, f, g)];
        }
      A[tri(12, i, j)] += k;
    }
  return ok;
}

// ND vertex rule straight into the cell's packed slots out[t * NC] (t = tri(12, i, j)): the corner
// coordinates are read from shared memory per corner (X(v, k): component k of cell vertex v), the
// mass part accumulates in place (first corner stores, the second adds; an off-diagonal mass entry
// has exactly one corner), the 6x6 face matrix of the curl part stays in registers and K = C^T M C
// is added at the end.  Same terms as cell_nd<0> without its 78 + 21 register arrays.
__host__ __device__ constexpr bool nd_share_corner(int i, int j) {
  for (int q = 0; q < 8; ++q)
    for (int d = 0; d < 3; ++d)
      for (int e = 0; e < 3; ++e)
        if (d != e && corner_edge(q, d) == i && corner_edge(q, e) == j) return true;
  return false;
}
// first corner (lowest q) on edge eps: the edge's end with bit dir = 0
__host__ __device__ constexpr bool nd_first_end(int q, int d) { return ((q >> d) & 1) == 0; }

// packed index t -> (i, j), i <= j, of a symmetric 12 x 12 matrix
__host__ __device__ constexpr int tri_i(int n, int t) {
  int i = 0;
  while (t >= n - i) { t -= n - i; ++i; }
  return i;
}
__host__ __device__ constexpr int tri_j(int n, int t) {
  int i = 0;
  while (t >= n - i) { t -= n - i; ++i; }
  return i + t;
}
template <int T>
__device__ __forceinline__ void nd_curl_one(const double (&M)[21], double *__restrict__ out, int NC) {
  constexpr int i = tri_i(12, T), j = tri_j(12, T);
  constexpr int f0 = e_face(i, 0), f1 = e_face(i, 1), g0 = e_face(j, 0), g1 = e_face(j, 1);
  constexpr double s00 = c_sign(f0, i) * c_sign(g0, j), s01 = c_sign(f0, i) * c_sign(g1, j);
  constexpr double s10 = c_sign(f1, i) * c_sign(g0, j), s11 = c_sign(f1, i) * c_sign(g1, j);
  static_assert(tri(12, i, j) == T, "packed index");
  const double k = s00 * M[tri(6, f0, g0)] + s01 * M[tri(6, f0, g1)] + s10 * M[tri(6, f1, g0)] + s11 * M[tri(6, f1, g1)];
  double &dst = out[T * NC];
  if constexpr (i == j || nd_share_corner(i, j)) dst += k;
  else dst = k;
}
template <int... T>
__device__ __forceinline__ void nd_curl_all(const double (&M)[21], double *__restrict__ out, int NC,
                                            std::integer_sequence<int, T...>) {
  (nd_curl_one<T>(M, out, NC), ...);
}

template <typename XF>
__device__ __forceinline__ bool cell_nd_vertex_to(XF X, double alpha, double beta, double *__restrict__ out, int NC,
                                                  const double *ca = nullptr, const double *cb = nullptr) {
  double M[21];
#pragma unroll
  for (int i = 0; i < 21; ++i) M[i] = 0.0;
  const double w = 0.125;
  bool ok = true;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q % ND_FENCE == 0) asm volatile("" ::: "memory");  // ND_FENCE corners at a time (registers vs ILP)
    Jac3 J;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int hi = q | (1 << d), lo = q & ~(1 << d);
#pragma unroll
      for (int k = 0; k < 3; ++k) J.j[d][k] = X(hi, k) - X(lo, k);
    }
    finish_jac(J);
    ok &= J.det > 0.0;
    const double rdet = 1.0 / J.det, sm = w * beta * coef_q<0, 8>(cb, q) * rdet,
                 sc = w * alpha * coef_q<0, 8>(ca, q) * rdet;
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int e = d; e < 3; ++e) {
        const double qm = sm * dot3(J.r[d], J.r[e]);
        double &dst = out[tri(12, corner_edge(q, d), corner_edge(q, e)) * NC];
        if (d != e || nd_first_end(q, d)) dst = qm;
        else dst += qm;
        M[tri(6, 2 * d + ((q >> d) & 1), 2 * e + ((q >> e) & 1))] += sc * dot3(J.j[d], J.j[e]);
      }
  }
  // curl-curl: K_ij = sum_{f in F(i), g in F(j)} C_fi M_fg C_gj, added to the mass part; one
  // compile-time instance per packed entry (nested unrolled loops left M in local memory)
  nd_curl_all(M, out, NC, std::make_integer_sequence<int, 78>{});
  return ok;
}

// ------------------------------------------------------------------------ RT (3D): 6 x 6
template <int QUAD>
__device__ __forceinline__ bool cell_rt(const double X[8][3], double alpha, double beta, double *A /*21*/,
                                        const double *ca = nullptr, const double *cb = nullptr) {
#pragma unroll
  for (int i = 0; i < 21; ++i) A[i] = 0.0;
  const double w = 0.125;
  double sdiv = 0.0;
  bool ok = true;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    Jac3 J;
    double t[3];
    if (QUAD == 0) jac_corner(X, q, J);
    else {
      t[0] = gauss2_pt(q & 1); t[1] = gauss2_pt((q >> 1) & 1); t[2] = gauss2_pt((q >> 2) & 1);
      jac_point(X, t, J);
    }
    ok &= J.det > 0.0;
    const double sm = w * beta * coef_q<QUAD, 8>(cb, q) / J.det;
    sdiv += w * alpha * coef_q<QUAD, 8>(ca, q) / J.det;
    double R[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int e = d; e < 3; ++e) R[d][e] = R[e][d] = sm * dot3(J.j[d], J.j[e]);
    if (QUAD == 0) {
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int e = d; e < 3; ++e) A[tri(6, 2 * d + ((q >> d) & 1), 2 * e + ((q >> e) & 1))] += R[d][e];
    } else {
      double hf[6];
#pragma unroll
      for (int f = 0; f < 6; ++f) hf[f] = (f & 1) ? t[f / 2] : 1 - t[f / 2];
#pragma unroll
      for (int f = 0; f < 6; ++f)
#pragma unroll
        for (int g = f; g < 6; ++g) A[tri(6, f, g)] += hf[f] * hf[g] * R[f / 2][g / 2];
    }
  }
#pragma unroll
  for (int f = 0; f < 6; ++f)
#pragma unroll
    for (int g = f; g < 6; ++g) A[tri(6, f, g)] += sdiv * (double)(((f & 1) ? 1 : -1) * ((g & 1) ? 1 : -1));
  return ok;
}

}  // namespace lorb
