// lor_device.cuh -- device-side building blocks of the B200 LOR assembly kernels.
//
// Geometry of one macro element (Step A1): the element is refined into p^d
// LOR cells whose vertices are the element's coordinate E-vector entries (tensor GLL points).
// Local dofs live on "sub-lattices": H1 = lattice points; ND = edges along axis s (cell index
// along s, vertex index along the others); RT = faces with normal s (vertex index along s,
// cell indices along the others).  Each dof lies on one coarse entity ("slot" tau, see
// lor_internal.h) and the global ids of the dofs of sub-lattice s' on slot tau ("block") are an
// affine function of the local lattice coordinates (App. A numbering) -- this is what lets the
// kernels emit columns in ascending global order without sorting.
#pragma once
#include <stdint.h>

#include "lor_internal.h"

namespace lorb {

// ------------------------------------------------------------------------------ space traits
template <int DIM, int SP>
struct Tr;
template <>
struct Tr<3, SP_H1> {
  static constexpr int S = 1, W = 27, MAXL = 18, NLOC = 8, NENT = 36, NSLOT = 27;
};
template <>
struct Tr<2, SP_H1> {
  static constexpr int S = 1, W = 9, MAXL = 6, NLOC = 4, NENT = 10, NSLOT = 9;
};
template <>
struct Tr<3, SP_ND> {
  static constexpr int S = 3, W = 33, MAXL = 20, NLOC = 12, NENT = 78, NSLOT = 27;
};
template <>
struct Tr<3, SP_RT> {
  static constexpr int S = 3, W = 11, MAXL = 6, NLOC = 6, NENT = 21, NSLOT = 27;
};

// kind of axis a in sub-lattice s: true = vertex index (range [0,p]), false = cell index ([0,p-1])
template <int SP>
__host__ __device__ constexpr bool vkind(int s, int a) {
  return SP == SP_H1 ? true : (SP == SP_ND ? (a != s) : (a == s));
}

// stencil box of column sub-lattice s2 around a row of sub-lattice s, along axis a
// (offsets relative to the row's lattice coordinate, before clipping to the lattice).
template <int SP>
__host__ __device__ constexpr int st_lo(int s, int s2, int a) {
  return SP == SP_H1 ? -1
                     : (SP == SP_ND ? (s2 == s ? (a == s ? 0 : -1) : (a == s2 ? -1 : (a == s ? 0 : -1)))
                                    : (s2 == s ? (a == s ? -1 : 0) : (a == s2 ? 0 : (a == s ? -1 : 0))));
}
template <int SP>
__host__ __device__ constexpr int st_hi(int s, int s2, int a) {
  return SP == SP_H1 ? 1
                     : (SP == SP_ND ? (s2 == s ? (a == s ? 0 : 1) : (a == s2 ? 0 : (a == s ? 1 : 1)))
                                    : (s2 == s ? (a == s ? 1 : 0) : (a == s2 ? 1 : (a == s ? 0 : 0))));
}
template <int DIM, int SP>
__host__ __device__ constexpr int st_n(int s, int s2) {
  int n = 1;
  for (int a = 0; a < DIM; ++a) n *= st_hi<SP>(s, s2, a) - st_lo<SP>(s, s2, a) + 1;
  return n;
}
// slot offset of column sub-lattice s2 in the natural stencil order of a row in sub-lattice s
template <int DIM, int SP>
__host__ __device__ constexpr int st_off(int s, int s2) {
  int o = 0;
  for (int t = 0; t < s2; ++t) o += st_n<DIM, SP>(s, t);
  return o;
}
// natural slot of relative offset d (in sub-lattice s2) for a row of sub-lattice s
template <int DIM, int SP>
__host__ __device__ constexpr int st_slot(int s, int s2, int dx, int dy, int dz) {
  int nx = st_hi<SP>(s, s2, 0) - st_lo<SP>(s, s2, 0) + 1;
  int ny = st_hi<SP>(s, s2, 1) - st_lo<SP>(s, s2, 1) + 1;
  int r = st_off<DIM, SP>(s, s2) + (dx - st_lo<SP>(s, s2, 0)) + nx * (dy - st_lo<SP>(s, s2, 1));
  if (DIM == 3) r += nx * ny * (dz - st_lo<SP>(s, s2, 2));
  return r;
}

// packed symmetric index of (i, j), n x n, upper triangle row-major
__host__ __device__ constexpr int tri(int n, int i, int j) {
  return i <= j ? i * n - i * (i - 1) / 2 + (j - i) : j * n - j * (j - 1) / 2 + (i - j);
}

// ---------------------------------------------------------------------- element block table
// One entry per block b = s' * 27 + tau (2D H1: tau < 9).
struct Blk {
  int32_t g0;       // gid = g0 + sum_a str[a] * x[a]
  int32_t str[3];
  int32_t base;     // min gid over the block (sort key)
  int16_t size;     // number of dofs in the block (0 = empty)
  int8_t sigma;     // orientation sign of all dofs in the block
  uint8_t ord;      // axis order by |stride|: fast | mid << 2 | slow << 4
};

__host__ __device__ inline int cls_of(int tau, int a) { return a == 0 ? tau % 3 : (a == 1 ? (tau / 3) % 3 : tau / 9); }

// class of coordinate x along an axis of the given kind (0 = min side, 1 = interior, 2 = max side)
__device__ __forceinline__ int coord_cls(bool vk, int x, int p) { return vk ? (x == 0 ? 0 : (x == p ? 2 : 1)) : 1; }

// Block affine map from App. A.  T: the element's topology record,
// base[t]: global id of the first dof of entity t of each type for this space.
// eb: global id of the first dof of the entity at slot tau (base[type][T.ent[tau]])
template <int DIM, int SP>
__device__ void block_affine_eb(int p, int s, int tau, const ElemTopo &T, int eb, Blk &B) {
  int c[3] = {cls_of(tau, 0), cls_of(tau, 1), DIM == 3 ? cls_of(tau, 2) : 1};
  B.g0 = 0;
  B.str[0] = B.str[1] = B.str[2] = 0;
  B.sigma = 1;
  B.size = 0;
  // box extent check: cell-index axes must be interior class; vertex-index interior needs p >= 2
  int sz = 1;
  for (int a = 0; a < DIM; ++a) {
    bool vk = vkind<SP>(s, a);
    int len;
    if (!vk) len = (c[a] == 1) ? p : 0;
    else len = (c[a] == 1) ? p - 1 : 1;
    sz *= len;
  }
  if (sz <= 0) { B.base = 0; B.ord = 0; return; }
  B.size = (int16_t)sz;
  int nI = 0;
  for (int a = 0; a < DIM; ++a) nI += (c[a] == 1);
  const int ent = T.ent[tau];
  const int o = T.orient[tau];
  if (SP == SP_H1) {
    if (nI == 0) {
      B.g0 = eb;
    } else if (nI == 1) {  // edge along the interior axis d
      int d = (c[0] == 1) ? 0 : (c[1] == 1 ? 1 : 2);
      bool rev = o & 1;
      B.g0 = eb + (rev ? p - 1 : -1);
      B.str[d] = rev ? -1 : 1;
    } else if (DIM == 3 && nI == 2) {  // face with normal n
      int n = (c[0] != 1) ? 0 : (c[1] != 1 ? 1 : 2);
      int u = (n == 0) ? 1 : 0, v = (n == 2) ? 1 : 2;
      int swp = o & 1, s1n = (o >> 1) & 1, s2n = (o >> 2) & 1;
      int ax1 = swp ? v : u, ax2 = swp ? u : v;
      B.str[ax1] = s1n ? -1 : 1;
      B.str[ax2] = s2n ? -(p - 1) : (p - 1);
      B.g0 = eb + (s1n ? p - 1 : -1) + (p - 1) * (s2n ? p - 1 : -1);
    } else {  // interior, lexicographic
      B.str[0] = 1;
      B.str[1] = p - 1;
      B.str[2] = DIM == 3 ? (p - 1) * (p - 1) : 0;
      B.g0 = eb - 1 - (p - 1) - (DIM == 3 ? (p - 1) * (p - 1) : 0);
    }
  } else if (SP == SP_ND) {
    int u = (s == 0) ? 1 : 0, v = (s == 2) ? 1 : 2;  // axes other than the edge direction
    bool bu = c[u] != 1, bv = c[v] != 1;
    if (bu && bv) {  // coarse edge along s
      bool rev = o & 1;
      B.g0 = eb + (rev ? p - 1 : 0);
      B.str[s] = rev ? -1 : 1;
      B.sigma = rev ? -1 : 1;
    } else if (bu || bv) {  // coarse face with normal n (the boundary axis), s in-face
      int n = bu ? u : v;
      int fu = (n == 0) ? 1 : 0, fv = (n == 2) ? 1 : 2;
      int swp = o & 1, s1n = (o >> 1) & 1, s2n = (o >> 2) & 1;
      int ax1 = swp ? fv : fu, ax2 = swp ? fu : fv;
      int fb = eb;
      if (s == ax1) {  // axis1-parallel: base + i1c + p (i2 - 1)
        B.str[s] = s1n ? -1 : 1;
        B.str[ax2] = s2n ? -p : p;
        B.g0 = fb + (s1n ? p - 1 : 0) + p * (s2n ? p - 1 : -1);
        B.sigma = s1n ? -1 : 1;
      } else {  // axis2-parallel: base + p(p-1) + i2c + p (i1 - 1)
        B.str[s] = s2n ? -1 : 1;
        B.str[ax1] = s1n ? -p : p;
        B.g0 = fb + p * (p - 1) + (s2n ? p - 1 : 0) + p * (s1n ? p - 1 : -1);
        B.sigma = s2n ? -1 : 1;
      }
    } else {  // interior block s: x-fastest over (cell along s: p; vertex-1 elsewhere: p-1)
      int rg[3];
      for (int a = 0; a < 3; ++a) rg[a] = (a == s) ? p : p - 1;
      B.str[0] = 1;
      B.str[1] = rg[0];
      B.str[2] = rg[0] * rg[1];
      int g = eb + s * p * (p - 1) * (p - 1);
      for (int a = 0; a < 3; ++a)
        if (a != s) g -= B.str[a];
      B.g0 = g;
    }
  } else {  // RT
    if (c[s] != 1) {  // coarse face (s, side)
      int u = (s == 0) ? 1 : 0, v = (s == 2) ? 1 : 2;
      int swp = o & 1, s1n = (o >> 1) & 1, s2n = (o >> 2) & 1;
      int ax1 = swp ? v : u, ax2 = swp ? u : v;
      B.str[ax1] = s1n ? -1 : 1;
      B.str[ax2] = s2n ? -p : p;
      B.g0 = eb + (s1n ? p - 1 : 0) + (s2n ? p * (p - 1) : 0);
      const int eps = (s == 1) ? -1 : 1;
      B.sigma = (int8_t)((s1n ? -1 : 1) * (s2n ? -1 : 1) * (swp ? -1 : 1) * eps);
    } else {  // interior block s: x-fastest over (vertex-1 along s: p-1; cells elsewhere: p)
      int rg[3];
      for (int a = 0; a < 3; ++a) rg[a] = (a == s) ? p - 1 : p;
      B.str[0] = 1;
      B.str[1] = rg[0];
      B.str[2] = rg[0] * rg[1];
      B.g0 = eb + s * p * p * (p - 1) - B.str[s];
    }
  }
  // min gid over the box and the axis order by |stride| (length-1 axes sort first, any order)
  int lo[3], hi[3];
  for (int a = 0; a < 3; ++a) { lo[a] = 0; hi[a] = 0; }
  for (int a = 0; a < DIM; ++a) {
    bool vk = vkind<SP>(s, a);
    if (!vk) { lo[a] = 0; hi[a] = p - 1; }
    else if (c[a] == 0) { lo[a] = hi[a] = 0; }
    else if (c[a] == 2) { lo[a] = hi[a] = p; }
    else { lo[a] = 1; hi[a] = p - 1; }
  }
  int bmin = B.g0;
  for (int a = 0; a < DIM; ++a) bmin += B.str[a] >= 0 ? B.str[a] * lo[a] : B.str[a] * hi[a];
  B.base = bmin;
  int key[3];
  for (int a = 0; a < 3; ++a) key[a] = (a < DIM && hi[a] > lo[a]) ? abs(B.str[a]) : 0;
  int ord[3] = {0, 1, 2};
  for (int i = 1; i < 3; ++i)
    for (int j = i; j > 0 && key[ord[j]] < key[ord[j - 1]]; --j) { int t = ord[j]; ord[j] = ord[j - 1]; ord[j - 1] = t; }
  B.ord = (uint8_t)(ord[0] | (ord[1] << 2) | (ord[2] << 4));
}

template <int DIM, int SP>
__device__ __forceinline__ void block_affine(int p, int s, int tau, const ElemTopo &T, const int32_t *const *base, Blk &B) {
  const int c0 = cls_of(tau, 0), c1 = cls_of(tau, 1), c2 = DIM == 3 ? cls_of(tau, 2) : 1;
  const int nI = (c0 == 1) + (c1 == 1) + (DIM == 3 ? (c2 == 1) : 0);
  const int type = (nI == 0) ? 0 : (nI == DIM ? 3 : (DIM == 3 ? nI : 1));
  block_affine_eb<DIM, SP>(p, s, tau, T, base[type][T.ent[tau]], B);
}

// ------------------------------------------------------------------------- row geometry
// Row (local dof) of sub-lattice s at lattice position x.  For each column sub-lattice s2 and
// axis a: the clipped column range [blo, bhi] and, per class c, the segment [slo, shi] (empty if
// slo > shi).
struct AxisSeg {
  int8_t lo[3], hi[3];  // per class 0/1/2
};

template <int SP>
__device__ __forceinline__ void axis_segments(int p, int s, int s2, int a, int x, AxisSeg &g) {
  const bool vk = vkind<SP>(s2, a);
  const int ext = vk ? p + 1 : p;
  int blo = x + st_lo<SP>(s, s2, a), bhi = x + st_hi<SP>(s, s2, a);
  blo = blo < 0 ? 0 : blo;
  bhi = bhi > ext - 1 ? ext - 1 : bhi;
  if (!vk) {
    g.lo[0] = 1; g.hi[0] = 0;
    g.lo[1] = (int8_t)blo; g.hi[1] = (int8_t)bhi;
    g.lo[2] = 1; g.hi[2] = 0;
    return;
  }
  // m: {0}, I: [1, p-1], M: {p}
  if (blo == 0) { g.lo[0] = 0; g.hi[0] = 0; } else { g.lo[0] = 1; g.hi[0] = 0; }
  int ilo = blo < 1 ? 1 : blo, ihi = bhi > p - 1 ? p - 1 : bhi;
  g.lo[1] = (int8_t)ilo; g.hi[1] = (int8_t)ihi;
  if (bhi == p) { g.lo[2] = (int8_t)p; g.hi[2] = (int8_t)p; } else { g.lo[2] = 1; g.hi[2] = 0; }
}

}  // namespace lorb
