// lor_asm.cuh -- templates of the fused element assembly kernel (k_assemble) and the shared-row
// merge (finalize_ose).  Instantiated per (dim, space, p) in generated translation units
// (build.py) so the sm_100a build runs in parallel.  See lor_kernels.cu for the pipeline.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "lor_cells.cuh"
#include "lor_device.cuh"
#include "lor_kernels.h"

namespace lorb {

__host__ __device__ constexpr int ipow_c(int b, int e) { return e == 0 ? 1 : b * ipow_c(b, e - 1); }

// ------------------------------------------------------------------------ small helpers
// L2 eviction priorities: the CSR output is written once and never re-read by this kernel
// (the hinted stores carry no "memory" clobber: nothing in the issuing thread reads them back, and
// leaving it off lets the compiler hoist the shared-memory loads of later slots above them)
// (evict_first); partial rows wait in L2 for the last contributor of their entity (evict_last).
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_hint(int32_t *a, int32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol));
}
__device__ __forceinline__ void st_hint(double *a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol));
}
// streaming reads (coordinates, merge plan, row offsets): read once per call, so they must not
// push the waiting partial rows out of L2
__device__ __forceinline__ uint4 ld_stream(const uint4 *a, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld_stream(const double2 *a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int64_t ld_stream(const int64_t *a, uint64_t pol) {
  int64_t v;
  asm volatile("ld.global.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint2(double *a, double v0, double v1, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a), "d"(v0), "d"(v1), "l"(pol));
}
// debug: per-CTA phase clocks (A.tstamp, LOR_PHASE_TIMING=1)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid_() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
#define LOR_TSTAMP(cond, k)                                                                \
  do {                                                                                     \
    if (A.tstamp && (cond)) A.tstamp[(int64_t)blockIdx.x * 16 + (k)] = clock64();        \
  } while (0)
#define LOR_STAMP(k)                                                                       \
  do {                                                                                     \
    if (A.tstamp && threadIdx.x == 0) A.tstamp[(int64_t)blockIdx.x * 16 + (k)] = clock64(); \
  } while (0)

__device__ __forceinline__ void report_error(int *err, int code, int64_t e, int cell) {
  if (atomicCAS(err, 0, code) == 0) {
    err[1] = (int)e;
    err[2] = cell;
  }
}

// bounds of the class-c segment of the clipped stencil range of column sub-lattice s2 along axis a
template <int SP>
__device__ __forceinline__ void seg_bounds(int p, int s, int s2, int a, int x, int c, int &lo, int &hi) {
  const bool vk = vkind<SP>(s2, a);
  const int ext = vk ? p + 1 : p;
  int blo = x + st_lo<SP>(s, s2, a), bhi = x + st_hi<SP>(s, s2, a);
  blo = blo < 0 ? 0 : blo;
  bhi = bhi > ext - 1 ? ext - 1 : bhi;
  if (!vk) {
    if (c == 1) { lo = blo; hi = bhi; } else { lo = 1; hi = 0; }
    return;
  }
  if (c == 0) { lo = 0; hi = (blo == 0) ? 0 : -1; }
  else if (c == 2) { lo = p; hi = (bhi == p) ? p : p - 1; }
  else { lo = blo < 1 ? 1 : blo; hi = bhi > p - 1 ? p - 1 : bhi; }
}

// lattice extent of sub-lattice s along axis a
template <int SP>
__host__ __device__ constexpr int ext_of(int p, int s, int a) { return vkind<SP>(s, a) ? p + 1 : p; }

// decode a local dof index (macro-element local order) into (sub-lattice, lattice coords)
template <int DIM, int SP>
__device__ __forceinline__ void decode_local(int p, int l, int &s, int x[3]) {
  if (SP == SP_H1) {
    s = 0;
    x[0] = l % (p + 1);
    x[1] = (l / (p + 1)) % (p + 1);
    x[2] = DIM == 3 ? l / ((p + 1) * (p + 1)) : 0;
    return;
  }
  const int blk = (SP == SP_ND) ? p * (p + 1) * (p + 1) : (p + 1) * p * p;
  s = l / blk;
  int r = l - s * blk;
  const int e0 = ext_of<SP>(p, s, 0), e1 = ext_of<SP>(p, s, 1);
  x[0] = r % e0;
  r /= e0;
  x[1] = r % e1;
  x[2] = r / e1;
}

template <int DIM, int SP>
__device__ __forceinline__ int row_tau(int p, int s, const int x[3]) {
  int t = coord_cls(vkind<SP>(s, 0), x[0], p) + 3 * coord_cls(vkind<SP>(s, 1), x[1], p);
  if (DIM == 3) t += 9 * coord_cls(vkind<SP>(s, 2), x[2], p);
  return t;
}

// row key: per axis (min(x,2), min(ext-1-x,2)) -> 0..8, combined base 9
template <int DIM, int SP>
__device__ __forceinline__ int row_key(int p, int s, const int x[3]) {
  int k = 0, m = 1;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const int ext = ext_of<SP>(p, s, a);
    const int kl = x[a] < 2 ? x[a] : 2, d = ext - 1 - x[a], kh = d < 2 ? d : 2;
    k += (kl * 3 + kh) * m;
    m *= 9;
  }
  return k;
}

// join entity of a row (classes cr) and a column (classes cc): fixed where both sit on the same side
__device__ __forceinline__ int join_cls(int cr, int cc) { return (cr == cc && cr != 1) ? cr : 1; }

// ================================================================================ k_assemble
// natural-order partial-row records (values only; columns and column signs of shared rows are
// topological and live in the setup merge plan): row strides padded to whole 128-byte lines, so a
// record line can be dropped from L2 with discard.global.L2 once the finalizer has consumed it
// (no write-back to HBM)
__host__ __device__ constexpr int rec_w8(int W) { return (W + 15) / 16 * 16; }  // doubles per row

// H1 stencil slot j <-> neighbour offset (dx, dy, dz) in {-1,0,1}^d, x fastest (st_slot order)
template <int DIM>
__host__ __device__ constexpr int h1_off(int j, int a) { return a == 0 ? j % 3 - 1 : (a == 1 ? (j / 3) % 3 - 1 : (DIM == 3 ? j / 9 - 1 : 0)); }
template <int DIM, int P>
__host__ __device__ constexpr int h1_dl(int j) { return h1_off<DIM>(j, 0) + (P + 1) * (h1_off<DIM>(j, 1) + (P + 1) * h1_off<DIM>(j, 2)); }

template <int DIM, int SP, int P, int KZ>
struct AsmCfg {
  using T_ = Tr<DIM, SP>;
  static constexpr int S = T_::S, W = T_::W, NENT = T_::NENT, NSLOT = T_::NSLOT, MAXL = T_::MAXL;
  static constexpr int NB = S * 27;                               // block table entries
  static constexpr int NPTS = ipow_c(P + 1, DIM);                 // lattice points (coords)
  static constexpr int NDPE = SP == SP_H1 ? NPTS : (SP == SP_ND ? 3 * P * (P + 1) * (P + 1) : 3 * P * P * (P + 1));
  static constexpr int CPL = P * P;                               // cells per layer (2D: all)
  static constexpr int NRING = DIM == 3 ? (KZ == P ? P : KZ + 1) : 1;
  static constexpr int NCELL = NRING * CPL;                       // cells resident in smem
  static constexpr int NCP = NCELL | 1;                           // cell-matrix pitch (odd: the 8 corner
                                                                  // lanes of a cell hit different banks)
  static constexpr int NW = 4;                                    // warps per CTA
  static constexpr int NT = NW * 32;
  static constexpr int TZS = tab_tzs(NB);                         // block-size table row (bytes)
  static constexpr int TSB = TZS + (NB + 15) / 16 * 16;           // per-thread row scratch: sizes -> positions | P0
  // shared memory layout (bytes); everything from OFF_X on is reused by the finalizer
  static constexpr int OFF_BLK = 0;
  static constexpr int OFF_OS = OFF_BLK + NB * (int)sizeof(Blk);            // ordsig[NB] uint16
  static constexpr int OFF_BL = OFF_OS + NB * 2;                           // blist[NB] uint8
  static constexpr int OFF_GM = (OFF_BL + NB + 15) / 16 * 16;              // gmap[NDPE] int32
  static constexpr int OFF_BS = OFF_GM + NDPE * 4;                         // bsg[NDPE] uint8
  static constexpr int OFF_DL = (OFF_BS + NDPE + 15) / 16 * 16;            // dl[S][W] int16: local offset | s2 << 8
  static constexpr int OFF_X = (OFF_DL + S * W * 2 + 15) / 16 * 16;
  static constexpr int OFF_CM = (OFF_X + DIM * NPTS * 8 + 15) / 16 * 16;
  static constexpr int OFF_TS = (OFF_CM + NENT * NCP * 8 + 15) / 16 * 16;    // row scratch [TSB][NT] bytes
  static constexpr int MAXR = DIM == 3 ? S * (P + 1) * (P + 1) * (KZ + 1) : (P + 1) * (P + 1);  // rows per chunk
  static constexpr int OFF_RL = OFF_TS + NT * TSB;                         // row order list uint16[MAXR]
  static constexpr int SMEM = (OFF_RL + 2 * MAXR + 15) / 16 * 16;
  static_assert(TZS >= W, "slot positions overwrite the block-size bytes");
  // CTAs per SM the shared memory allows (228 KB per SM, 1 KB reserved per CTA), 2..5: the
  // register budget of __launch_bounds__ follows it (ND: 3 -> 168 registers, no spills)
  static constexpr int MINB_FIT = (228 * 1024) / (SMEM + 1024);
  static constexpr int MINB_CAP = (DIM == 3 && SP == SP_H1) ? 5 : 4;  // measured best caps (RT at 5: 0.918 -> 0.956 ms)
  static constexpr int MINB_SMEM = MINB_FIT > MINB_CAP ? MINB_CAP : (MINB_FIT < 2 ? 2 : MINB_FIT);
};


// per-row value accumulation: acc[slot] = sum over cells containing the row of the cell matrix row
template <int DIM, int SP, int P, int RS, int NC>
__device__ __forceinline__ void row_values(const double *__restrict__ cm, const int x[3], int nring, double *acc) {
  constexpr int W = Tr<DIM, SP>::W;
#pragma unroll
  for (int j = 0; j < W; ++j) acc[j] = 0.0;
  auto cidx = [&](int cx, int cy, int cz) -> int {
    if (DIM == 2) return cy * P + cx;
    return (((cz % nring) * P) + cy) * P + cx;
  };
  auto cvalid = [&](int c) { return c >= 0 && c < P; };
  if (SP == SP_H1 && DIM == 3) {
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      const int ox = o & 1, oy = (o >> 1) & 1, oz = (o >> 2) & 1;
      const int cx = x[0] - ox, cy = x[1] - oy, cz = x[2] - oz;
      if (!(cvalid(cx) && cvalid(cy) && cvalid(cz))) continue;
      const int ci = cidx(cx, cy, cz);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int dx = (j & 1) - ox, dy = ((j >> 1) & 1) - oy, dz = ((j >> 2) & 1) - oz;
        acc[st_slot<3, SP_H1>(0, 0, dx, dy, dz)] += cm[tri(8, o, j) * NC + ci];
      }
    }
  } else if (SP == SP_H1 && DIM == 2) {
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      const int ox = o & 1, oy = (o >> 1) & 1;
      const int cx = x[0] - ox, cy = x[1] - oy;
      if (!(cvalid(cx) && cvalid(cy))) continue;
      const int ci = cidx(cx, cy, 0);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int dx = (j & 1) - ox, dy = ((j >> 1) & 1) - oy;
        acc[st_slot<2, SP_H1>(0, 0, dx, dy, 0)] += cm[tri(4, o, j) * NC + ci];
      }
    }
  } else if (SP == SP_ND) {
    constexpr int u = (RS == 0) ? 1 : 0, v = (RS == 2) ? 1 : 2;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int b1 = b & 1, b2 = b >> 1;
      int c[3];
      c[RS] = x[RS];
      c[u] = x[u] - b1;
      c[v] = x[v] - b2;
      if (!(cvalid(c[0]) && cvalid(c[1]) && cvalid(c[2]))) continue;
      const int ci = cidx(c[0], c[1], c[2]);
      const int er = 4 * RS + b1 + 2 * b2;
#pragma unroll
      for (int ep = 0; ep < 12; ++ep) {
        int d[3] = {0, 0, 0};
        d[u] -= b1;
        d[v] -= b2;
        d[e_u(ep)] += e_b1(ep);
        d[e_v(ep)] += e_b2(ep);
        acc[st_slot<3, SP_ND>(RS, e_dir(ep), d[0], d[1], d[2])] += cm[tri(12, er, ep) * NC + ci];
      }
    }
  } else {  // RT
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      int c[3] = {x[0], x[1], x[2]};
      c[RS] -= side;
      if (!(cvalid(c[0]) && cvalid(c[1]) && cvalid(c[2]))) continue;
      const int ci = cidx(c[0], c[1], c[2]);
      const int fr = 2 * RS + side;
#pragma unroll
      for (int fp = 0; fp < 6; ++fp) {
        int d[3] = {0, 0, 0};
        d[RS] -= side;
        d[fp / 2] += fp & 1;
        acc[st_slot<3, SP_RT>(RS, fp / 2, d[0], d[1], d[2])] += cm[tri(6, fr, fp) * NC + ci];
      }
    }
  }
}

// H1 (3D, vertex rule): one thread per (cell, corner); the eight corners of a cell are eight
// consecutive lanes.  Corner q forms its Jacobian from the cell's edge vectors through q, the
// tensor Q = w a adj adj^T / det and the ten corner contributions of SURVEY C.5; the 36 packed
// entries of the cell matrix are then assembled with xor-shuffles inside the 8-lane group:
//   (q,q)       = s^T Q_q s + w b det_q + sum_d Q_{q^d}[d][d]
//   (q,q^d)     = -s_d (Q_q s)_d - s'_d (Q_{q^d} s')_d
//   (q^d,q^d')  = s_d s_d' Q_q[d][d'] + (same at corner q^d^d')        (face diagonal)
//   body diagonal = 0
template <int P, int NC, int NRING_>
__device__ __forceinline__ void cells_h1_corner(const double *__restrict__ X, double *__restrict__ cm, int k0, int ncell,
                                                double alpha, double beta, int &bad, const double *ca = nullptr,
                                                const double *cb = nullptr) {
  constexpr int NP1 = P + 1, NPT = NP1 * NP1 * NP1;
  const int lane = threadIdx.x & 31;
  const int items = ncell * 8;
  const int ceil32 = (items + 31) / 32 * 32;
  for (int it = threadIdx.x; it < ceil32; it += blockDim.x) {
    const bool act = it < items;
    const int c = act ? it >> 3 : 0, q = it & 7;
    const int cx = c % P, cy = (c / P) % P, cz = k0 + c / (P * P);
    auto pt = [&](int v, int d) -> double {
      const int l = (cx + (v & 1)) + NP1 * ((cy + ((v >> 1) & 1)) + NP1 * (cz + ((v >> 2) & 1)));
      return X[d * NPT + l];
    };
    double j[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int hi = q | (1 << d), lo = q & ~(1 << d);
#pragma unroll
      for (int k = 0; k < 3; ++k) j[d][k] = pt(hi, k) - pt(lo, k);
    }
    double r[3][3];
    cross3(j[1], j[2], r[0]);
    cross3(j[2], j[0], r[1]);
    cross3(j[0], j[1], r[2]);
    const double det = dot3(j[0], r[0]);
    if (act && !(det > 0.0)) bad = 1 + c;
    // variable coefficients (NEXT-3): the element's coefficient E-vectors at this corner's point
    const int lq = (cx + (q & 1)) + NP1 * ((cy + ((q >> 1) & 1)) + NP1 * (cz + ((q >> 2) & 1)));
    const double sa = 0.125 * alpha * (ca ? __ldg(ca + lq) : 1.0) / det;
    double Q[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int e = d; e < 3; ++e) Q[d][e] = Q[e][d] = sa * dot3(r[d], r[e]);
    double sg[3], Qs[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) sg[d] = ((q >> d) & 1) ? 1.0 : -1.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) Qs[d] = Q[d][0] * sg[0] + Q[d][1] * sg[1] + Q[d][2] * sg[2];
    double diag = sg[0] * Qs[0] + sg[1] * Qs[1] + sg[2] * Qs[2] + 0.125 * beta * (cb ? __ldg(cb + lq) : 1.0) * det;
    double edge[3], fdg[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      diag += __shfl_xor_sync(0xffffffffu, Q[d][d], 1 << d);
      const double e = -sg[d] * Qs[d];
      edge[d] = e + __shfl_xor_sync(0xffffffffu, e, 1 << d);
    }
    // face diagonals (d,d') = (0,1), (0,2), (1,2)
    {
      const double f01 = sg[0] * sg[1] * Q[0][1], f02 = sg[0] * sg[2] * Q[0][2], f12 = sg[1] * sg[2] * Q[1][2];
      fdg[0] = f01 + __shfl_xor_sync(0xffffffffu, f01, 3);
      fdg[1] = f02 + __shfl_xor_sync(0xffffffffu, f02, 5);
      fdg[2] = f12 + __shfl_xor_sync(0xffffffffu, f12, 6);
    }
    (void)lane;
    if (act) {
      const int ci = (((cz % NRING_) * P) + cy) * P + cx;
      double *o = cm + ci;
      // packed upper-triangle index of (i, j), i <= j < 8: i*8 - i(i-1)/2 + (j - i) = i(15-i)/2 + j
      const int rq = (q * (15 - q)) >> 1;
      o[(rq + q) * NC] = diag;
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (!((q >> d) & 1)) o[(rq + (q | (1 << d))) * NC] = edge[d];
      // face diagonal of (d,d') is written by the lower of its two corners q, q^d^d'
      auto tp = [](int a, int b) { const int i = a < b ? a : b, j = a < b ? b : a; return ((i * (15 - i)) >> 1) + j; };
      if (q < (q ^ 3)) o[tp(q ^ 1, q ^ 2) * NC] = fdg[0];
      if (q < (q ^ 5)) o[tp(q ^ 1, q ^ 4) * NC] = fdg[1];
      if (q < (q ^ 6)) o[tp(q ^ 2, q ^ 4) * NC] = fdg[2];
      if (q < 4) o[(rq + (q ^ 7)) * NC] = 0.0;
    }
  }
}

template <int DIM, int SP, int P, int QUAD>
__device__ __forceinline__ bool compute_cell(const double *__restrict__ X, int cx, int cy, int cz, double alpha,
                                             double beta, double *__restrict__ out, int NC, int ci,
                                             const double *ca = nullptr, const double *cb = nullptr) {
  constexpr int NP1 = P + 1;
  // variable coefficients (NEXT-3): the cell's corner values from the element's coefficient E-vectors
  double a8[8], b8[8];
  const double *pa = nullptr, *pb = nullptr;
  if (ca) {
#pragma unroll
    for (int q = 0; q < (DIM == 3 ? 8 : 4); ++q) {
      const int l = DIM == 3 ? (cx + (q & 1)) + NP1 * ((cy + ((q >> 1) & 1)) + NP1 * (cz + ((q >> 2) & 1)))
                             : (cx + (q & 1)) + NP1 * (cy + ((q >> 1) & 1));
      a8[q] = __ldg(ca + l);
      b8[q] = __ldg(cb + l);
    }
    pa = a8;
    pb = b8;
  }
  if (DIM == 3 && SP == SP_ND && QUAD == 0) {  // vertex rule: straight into the packed slots
    auto XF = [&](int v, int k) -> double {
      return X[k * ipow_c(NP1, 3) + (cx + (v & 1)) + NP1 * ((cy + ((v >> 1) & 1)) + NP1 * (cz + ((v >> 2) & 1)))];
    };
    return cell_nd_vertex_to(XF, alpha, beta, out + ci, NC, pa, pb);
  }
  if (DIM == 3) {
    double C[8][3];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int l = (cx + (q & 1)) + NP1 * ((cy + ((q >> 1) & 1)) + NP1 * (cz + ((q >> 2) & 1)));
#pragma unroll
      for (int d = 0; d < 3; ++d) C[q][d] = X[d * ipow_c(NP1, 3) + l];
    }
    if (SP == SP_H1) {
      double A[36];
      bool ok = cell_h1_3d<QUAD>(C, alpha, beta, A, pa, pb);
#pragma unroll
      for (int i = 0; i < 36; ++i) out[i * NC + ci] = A[i];
      return ok;
    } else if (SP == SP_ND) {
      double A[78];
      bool ok = cell_nd<QUAD>(C, alpha, beta, A, pa, pb);
#pragma unroll
      for (int i = 0; i < 78; ++i) out[i * NC + ci] = A[i];
      return ok;
    } else {
      double A[21];
      bool ok = cell_rt<QUAD>(C, alpha, beta, A, pa, pb);
#pragma unroll
      for (int i = 0; i < 21; ++i) out[i * NC + ci] = A[i];
      return ok;
    }
  } else {
    double C[4][2];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int l = (cx + (q & 1)) + NP1 * (cy + ((q >> 1) & 1));
#pragma unroll
      for (int d = 0; d < 2; ++d) C[q][d] = X[d * NP1 * NP1 + l];
    }
    double A[10];
    bool ok = cell_h1_2d<QUAD>(C, alpha, beta, A, pa, pb);
#pragma unroll
    for (int i = 0; i < 10; ++i) out[i * NC + ci] = A[i];
    return ok;
  }
}

// ---------------------------------------------------------------------- shared-row merge
// CTA-cooperative merge of the partial rows of one owned shared entity into final CSR rows.
// Row g has k contributing elements (element order); list m = that element's partial row, sorted,
// made of runs of equal block base (a block = the dofs of one coarse entity in one sub-lattice,
// a contiguous range of global ids, identical in every element that holds it).  Phase A (one
// thread per row) merges the k block-run lists by base: union blocks in ascending order, their
// offsets P0 in the final row and the start of each block in every list holding it.  Phase B (one
// thread per list entry) writes the final entry for the first list holding its block:
// position P0(u) + offset in block, value = sum over the lists holding the block in element order
// (deterministic, no atomics).
struct FinScratch {
  int maxl, kmax, nu;  // per-row capacities
};

static __device__ __noinline__ void finalize_ose(const Ose O, const int32_t *__restrict__ ose_slots, const RecEntry *scratch,
                                                 int rstride, int maxl, int maxu, int64_t row_begin,
                                                 const int64_t *__restrict__ row_ptr, int32_t *__restrict__ col,
                                                 double *__restrict__ val, unsigned char *smem, int smem_bytes) {
  const int k = O.k;
  // per row: len[k] int, rec[k] int64 (entry offset), bb[k][maxl] int, uidx[k][maxl] uint8,
  //          U: nu int, p0u[maxu] int16, first[maxu] uint8, start[maxu][k] int8
  const int per_row = k * 4 + k * 8 + k * maxl * 4 + k * maxl + 4 + maxu * 3 + maxu * k + 16;
  int rp = smem_bytes / per_row;
  if (rp > O.nrows) rp = O.nrows;
  if (rp < 1) rp = 1;
  int64_t *s_rec = reinterpret_cast<int64_t *>(smem);             // [rp][k]
  int *s_len = reinterpret_cast<int *>(s_rec + rp * k);            // [rp][k]
  int *s_bb = s_len + rp * k;                                      // [rp][k][maxl]
  int *s_nu = s_bb + rp * k * maxl;                                // [rp]
  int16_t *s_p0u = reinterpret_cast<int16_t *>(s_nu + rp);         // [rp][maxu]
  uint8_t *s_first = reinterpret_cast<uint8_t *>(s_p0u + rp * maxu);  // [rp][maxu]
  int8_t *s_start = reinterpret_cast<int8_t *>(s_first + rp * maxu);   // [rp][maxu][k]
  uint8_t *s_uidx = reinterpret_cast<uint8_t *>(s_start + rp * maxu * k);  // [rp][k][maxl]
  for (int r0 = 0; r0 < O.nrows; r0 += rp) {
    const int nr = (O.nrows - r0 < rp) ? O.nrows - r0 : rp;
    const int nl = nr * k;
    for (int li = threadIdx.x; li < nl; li += blockDim.x) {
      const int row = li / k, m = li - row * k;
      const int64_t rec = ((int64_t)ose_slots[O.slot_off + m] + r0 + row) * rstride;
      s_rec[li] = rec;
      s_len[li] = __ldcg(&scratch[rec + rstride - 1].col);
    }
    __syncthreads();
    for (int it = threadIdx.x; it < nl * maxl; it += blockDim.x) {
      const int li = it / maxl, e = it - li * maxl;
      if (e < s_len[li]) s_bb[it] = __ldcg(&scratch[s_rec[li] + e].bbase);
    }
    __syncthreads();
    // phase A: k-way merge of block runs (one thread per row)
    for (int row = threadIdx.x; row < nr; row += blockDim.x) {
      int ptr[MAX_VALENCE];
      for (int m = 0; m < k; ++m) ptr[m] = 0;
      int u = 0, P = 0;
      while (true) {
        int minb = 0x7fffffff;
        for (int m = 0; m < k; ++m) {
          const int li = row * k + m;
          if (ptr[m] < s_len[li]) {
            const int b = s_bb[li * maxl + ptr[m]];
            minb = b < minb ? b : minb;
          }
        }
        if (minb == 0x7fffffff || u >= maxu) break;
        int size = 0, first = -1;
        for (int m = 0; m < k; ++m) {
          const int li = row * k + m;
          int8_t st = -1;
          if (ptr[m] < s_len[li] && s_bb[li * maxl + ptr[m]] == minb) {
            int e = ptr[m];
            while (e < s_len[li] && s_bb[li * maxl + e] == minb) {
              s_uidx[li * maxl + e] = (uint8_t)u;
              ++e;
            }
            size = e - ptr[m];
            st = (int8_t)ptr[m];
            if (first < 0) first = m;
            ptr[m] = e;
          }
          s_start[(row * maxu + u) * k + m] = st;
        }
        s_p0u[row * maxu + u] = (int16_t)P;
        s_first[row * maxu + u] = (uint8_t)first;
        P += size;
        ++u;
      }
      s_nu[row] = u;
    }
    __syncthreads();
    // phase B: one thread per list entry; the first list holding the block writes
    for (int it = threadIdx.x; it < nl * maxl; it += blockDim.x) {
      const int li = it / maxl, e = it - li * maxl;
      if (e >= s_len[li]) continue;
      const int row = li / k, m = li - row * k;
      const int u = s_uidx[it];
      if (s_first[row * maxu + u] != m) continue;
      const int o = e - s_start[(row * maxu + u) * k + m];
      double sum = 0.0;
      for (int mm = 0; mm < k; ++mm) {
        const int st = s_start[(row * maxu + u) * k + mm];
        if (st >= 0) sum += __ldcg(&scratch[s_rec[row * k + mm] + st + o].val);
      }
      const int c = __ldcg(&scratch[s_rec[li] + e].col);
      const int64_t out = row_ptr[(int64_t)O.gid_base + r0 + row - row_begin] + s_p0u[row * maxu + u] + o;
      col[out] = c;
      val[out] = sum;
    }
    __syncthreads();
  }
}

template <int DIM, int SP, int P, int QUAD, int KZ, int MINB>
__global__ void __launch_bounds__(128, MINB) k_assemble(AsmArgs A) {
  using CF = AsmCfg<DIM, SP, P, KZ>;
  constexpr int S = CF::S, W = CF::W, NB = CF::NB, NC = CF::NCP;
  extern __shared__ __align__(16) unsigned char smem[];
  Blk *blk = reinterpret_cast<Blk *>(smem + CF::OFF_BLK);
  uint16_t *ordsig = reinterpret_cast<uint16_t *>(smem + CF::OFF_OS);
  uint8_t *blist = smem + CF::OFF_BL;
  int32_t *gmap = reinterpret_cast<int32_t *>(smem + CF::OFF_GM);
  uint8_t *bsg = smem + CF::OFF_BS;
  double *X = reinterpret_cast<double *>(smem + CF::OFF_X);
  double *cm = reinterpret_cast<double *>(smem + CF::OFF_CM);
  __shared__ ElemTopo T;
  __shared__ ElemSpace E;
  __shared__ int s_nb, s_fin_n, s_bad, s_ownacc;
  __shared__ int s_fin[27];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int16_t *dlt = reinterpret_cast<int16_t *>(smem + CF::OFF_DL);
  if ((int64_t)blockIdx.x >= A.nel_local) return;
  const int64_t el = A.order ? A.order[blockIdx.x] : blockIdx.x;  // local element (locality-preserving order)
  // L2 prefetch for the CTA that takes this CTA's place one residency later: its element id now,
  // its topology/space records, E-vector and element restriction after the prologue
  const int64_t pfb = (int64_t)blockIdx.x + A.pf_dist;
  const bool pf = A.pf_dist > 0 && pfb < A.nel_local && A.plan_mode == 0;
  int64_t pf_el = -1;
  if (pf && tid == 0) pf_el = A.order ? __ldg(A.order + pfb) : pfb;
  LOR_STAMP(0);
  if (A.tstamp && tid == 0) A.tstamp[(int64_t)blockIdx.x * 16 + 6] = gtimer();
  {
    const int4 *src = reinterpret_cast<const int4 *>(A.topo + el);
    int4 *dst = reinterpret_cast<int4 *>(&T);
    for (int i = tid; i < (int)(sizeof(ElemTopo) / 16); i += blockDim.x) dst[i] = src[i];
    const int4 *src2 = reinterpret_cast<const int4 *>(A.esp + el);
    int4 *dst2 = reinterpret_cast<int4 *>(&E);
    for (int i = tid; i < (int)(sizeof(ElemSpace) / 16); i += blockDim.x) dst2[i] = src2[i];
    const double2 *xs = reinterpret_cast<const double2 *>(A.X + el * A.xstride);
    double2 *xd = reinterpret_cast<double2 *>(X);
    constexpr int NX2 = (DIM * CF::NPTS) / 2;
    const uint64_t pfx = l2_policy_first();
    for (int i = tid; i < NX2; i += blockDim.x) xd[i] = ld_stream(xs + i, pfx);
    if ((DIM * CF::NPTS) & 1) {
      if (tid == 0) X[DIM * CF::NPTS - 1] = __ldg(A.X + el * A.xstride + DIM * CF::NPTS - 1);
    }
    if (tid == 0) { s_fin_n = 0; s_bad = 0; s_ownacc = 0; s_nb = 0; }
  }
  // one-rank assembly: the element restriction comes from setup and the block table (used only by
  // sorted records, i.e. multi-rank interface rows, and the setup passes) is skipped
  const bool fast = A.emap != nullptr && A.plan_mode == 0;
  if (fast) {
    for (int l = tid; l < CF::NDPE; l += blockDim.x) {
      gmap[l] = __ldg(A.emap + el * CF::NDPE + l);
      bsg[l] = __ldg(A.esgn + el * CF::NDPE + l) < 0 ? 128 : 0;
    }
  }
  __syncthreads();
  // ---- element block table, canonical axis order/directions, ascending-base order
  if (!fast) {
  if (tid < NB) {
    const int s = tid / 27, tau = tid - 27 * s;
    Blk B;
    if (DIM == 2 && tau >= 9) {
      B.size = 0; B.g0 = 0; B.base = 0; B.sigma = 1; B.ord = 0; B.str[0] = B.str[1] = B.str[2] = 0;
    } else {
      block_affine_eb<DIM, SP>(P, s, tau, T, E.ebase[tau], B);
    }
    blk[tid] = B;
    ordsig[tid] = (uint16_t)(B.ord | ((B.str[0] < 0) << 6) | ((B.str[1] < 0) << 7) | ((B.str[2] < 0) << 8));
  }
  __syncthreads();
  {
    __shared__ int s_wcnt[4];
    __shared__ uint8_t s_cl[NB];
    const bool ne = tid < NB && blk[tid].size > 0;
    const unsigned bal = __ballot_sync(0xffffffffu, ne);
    if (lane == 0) s_wcnt[warp] = __popc(bal);
    __syncthreads();
    int off = 0;
    for (int w2 = 0; w2 < warp; ++w2) off += s_wcnt[w2];
    if (ne) s_cl[off + __popc(bal & ((1u << lane) - 1u))] = (uint8_t)tid;
    if (tid == 0) s_nb = s_wcnt[0] + s_wcnt[1] + s_wcnt[2] + s_wcnt[3];
    __syncthreads();
    const int ncomp = s_nb;
    if (tid < ncomp) {
      const int b = s_cl[tid];
      const int mb = blk[b].base;
      int r = 0;
      for (int j = 0; j < ncomp; ++j) r += blk[s_cl[j]].base < mb;
      blist[r] = (uint8_t)b;
    }
  }
  }  // !fast
  // ---- slot -> local index offset relative to the row position in the column sub-lattice layout
  for (int i = tid; i < S * W; i += blockDim.x) {
    const int s = i / W, j = i - s * W;
    int jj = j, s2 = 0;
    while (s2 < S - 1 && jj >= st_n<DIM, SP>(s, s2)) { jj -= st_n<DIM, SP>(s, s2); ++s2; }
    const int nx = st_hi<SP>(s, s2, 0) - st_lo<SP>(s, s2, 0) + 1, ny = st_hi<SP>(s, s2, 1) - st_lo<SP>(s, s2, 1) + 1;
    const int dx = st_lo<SP>(s, s2, 0) + jj % nx, dy = st_lo<SP>(s, s2, 1) + (jj / nx) % ny;
    const int dz = (DIM == 3) ? st_lo<SP>(s, s2, 2) + jj / (nx * ny) : 0;
    dlt[i] = (int16_t)((uint8_t)(int8_t)(dx + ext_of<SP>(P, s2, 0) * (dy + ext_of<SP>(P, s2, 1) * dz)) | (s2 << 8));
  }
  // ---- element restriction in shared memory: global id and block/sign of every local dof
  if (!fast)
  for (int l = tid; l < CF::NDPE; l += blockDim.x) {
    int s, x[3];
    decode_local<DIM, SP>(P, l, s, x);
    const int b = s * 27 + row_tau<DIM, SP>(P, s, x);
    const Blk &B = blk[b];
    gmap[l] = B.g0 + B.str[0] * x[0] + B.str[1] * x[1] + B.str[2] * x[2];
    bsg[l] = (uint8_t)(b | (B.sigma < 0 ? 128 : 0));
  }
  __syncthreads();
  const int nb = s_nb;
  LOR_STAMP(1);
  if (pf) {
    const int64_t pe = __shfl_sync(0xffffffffu, pf_el, 0);
    if (warp == 0 && pe >= 0) {
      auto pfl = [](const void *a) { asm volatile("prefetch.global.L2 [%0];" ::"l"(a)); };
      constexpr int LT = (int)((sizeof(ElemTopo) + 127) / 128), LE = (int)((sizeof(ElemSpace) + 127) / 128);
      constexpr int LX = (DIM * CF::NPTS * 8 + 127) / 128;
      if (lane < LT) pfl(reinterpret_cast<const char *>(A.topo + pe) + 128 * lane);
      if (lane < LE) pfl(reinterpret_cast<const char *>(A.esp + pe) + 128 * lane);
      for (int l = lane; l < LX; l += 32) pfl(reinterpret_cast<const char *>(A.X + pe * A.xstride) + 128 * l);
      if (A.emap) {
        constexpr int LM = (CF::NDPE * 4 + 127) / 128 + 1, LS = (CF::NDPE + 127) / 128 + 1;
        for (int l = lane; l < LM; l += 32) pfl(reinterpret_cast<const char *>(A.emap + pe * CF::NDPE) + 128 * l);
        if (lane < LS) pfl(reinterpret_cast<const char *>(A.esgn + pe * CF::NDPE) + 128 * lane);
      }
    }
  }

  // variable coefficients (NEXT-3): this element's coefficient E-vectors, or null (constants)
  const double *eca = A.ca ? A.ca + el * CF::NPTS : nullptr, *ecb = A.ca ? A.cb + el * CF::NPTS : nullptr;
  // ---- z-chunks of cell layers
  constexpr int NCHUNK = (DIM == 3) ? (P + KZ - 1) / KZ : 1;
  for (int ch = 0; ch < NCHUNK; ++ch) {
    const int k0 = (DIM == 3) ? ch * KZ : 0;
    const int k1 = (DIM == 3) ? ((k0 + KZ < P) ? k0 + KZ : P) : P;
    const int ncell = (DIM == 3) ? (k1 - k0) * P * P : P * P;
    if (ch > 0) __syncthreads();  // previous chunk's rows done before its ring slots are reused
    if (DIM == 3 && SP == SP_H1 && QUAD == 0) {
      int bad = 0;
      cells_h1_corner<P, NC, CF::NRING>(X, cm, k0, ncell, A.alpha, A.beta, bad, eca, ecb);
      if (bad) s_bad = bad;
    } else {
      for (int c = tid; c < ncell; c += blockDim.x) {
        const int cx = c % P, cy = (c / P) % P, cz = (DIM == 3) ? k0 + c / (P * P) : 0;
        const int ci = (DIM == 3) ? (((cz % CF::NRING) * P) + cy) * P + cx : cy * P + cx;
        if (!compute_cell<DIM, SP, P, QUAD>(X, cx, cy, cz, A.alpha, A.beta, cm, NC, ci, eca, ecb))
          s_bad = 1 + cx + P * (cy + P * cz);
      }
    }
    __syncthreads();
    if (s_bad && tid == 0) report_error(A.err, 2, A.elem_begin + el, s_bad - 1);
    if (ch == 0) LOR_STAMP(2);
    // rows of this chunk: per sub-lattice s the z range [k0, kend(s))
    int nrows = 0, nrow_s0 = 0, nrow_s1 = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int ex = ext_of<SP>(P, s, 0), ey = ext_of<SP>(P, s, 1);
      int zl = 0, zh = 1;
      if (DIM == 3) {
        zl = k0;
        zh = k1 + ((vkind<SP>(s, 2) && k1 == P) ? 1 : 0);
      }
      const int n = ex * ey * (zh - zl);
      if (s == 0) nrow_s0 = n;
      if (s == 1) nrow_s1 = n;
      nrows += n;
    }
    // one thread per row: values from the cell matrices in shared memory; a shared row goes out
    // as a natural-order partial row (record), an own row straight into its CSR row at the
    // positions P0(block) + rank in the block's sub-box (ascending global column order)
    // per-thread row scratch, transposed ([byte][thread]) so lanes never share a bank:
    // bytes [0, TZS) block sizes, then slot positions; [TZS, TSB) P0 per block
    unsigned char *ts = smem + CF::OFF_TS + tid;
    auto decode_row = [&](int r, int &s, int *x) {
      s = 0;
      int rq = r;
      if (S > 1 && rq >= nrow_s0) { rq -= nrow_s0; s = 1; if (rq >= nrow_s1) { rq -= nrow_s1; s = 2; } }
      const int ex = ext_of<SP>(P, s, 0), ey = ext_of<SP>(P, s, 1);
      x[0] = rq % ex;
      x[1] = (rq / ex) % ey;
      x[2] = (DIM == 3) ? k0 + rq / (ex * ey) : 0;
      return row_tau<DIM, SP>(P, s, x);
    };
    // row order: partial rows first, own rows (the heavier path: positions + CSR stores) last, so
    // they fill as few warps as possible instead of diverging inside every warp
    // Own rows are listed in row order (block-wide ballot scan), so an own row's ordinal in its
    // element (the index of its setup position-table row) is deterministic.
    __shared__ int s_nsh, s_nown, s_wc[CF::NW];
    uint16_t *rlist = reinterpret_cast<uint16_t *>(smem + CF::OFF_RL);
    if (tid == 0) { s_nsh = 0; s_nown = 0; }
    __syncthreads();
    for (int r0 = 0; r0 < nrows; r0 += CF::NT) {
      const int r = r0 + tid;
      bool own = false;
      if (r < nrows) {
        int s, x[3];
        const int tr = decode_row(r, s, x);
        const bool owned = T.flags[tr] & TF_OWNED;
        const uint8_t sf = E.sflags[tr];
        const bool shared = sf & SF_SHARED;
        own = owned && !shared;
        if (!own && shared && (owned || (sf & SF_SEND)) && A.plan_mode != 2) rlist[atomicAdd(&s_nsh, 1)] = (uint16_t)r;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, own);
      if (lane == 0) s_wc[warp] = __popc(bal);
      __syncthreads();
      int wb = s_nown;
      for (int w2 = 0; w2 < warp; ++w2) wb += s_wc[w2];
      if (own) rlist[CF::MAXR - 1 - (wb + __popc(bal & ((1u << lane) - 1u)))] = (uint16_t)r;
      __syncthreads();
      if (tid == 0) {
        int t = 0;
        for (int w2 = 0; w2 < CF::NW; ++w2) t += s_wc[w2];
        s_nown += t;
      }
      __syncthreads();
    }
    const int nown = s_nown;
    const int nsh = s_nsh, nact = s_nsh + (A.plan_mode == 1 ? 0 : nown);
    const int own0 = s_ownacc;  // own rows of earlier chunks of this element
    for (int ii = tid; ii < nact; ii += CF::NT) {
      const int r = ii < nsh ? rlist[ii] : rlist[CF::MAXR - 1 - (ii - nsh)];
      int s, x[3];
      const int tr = decode_row(r, s, x);
      const uint8_t fl = T.flags[tr], sf = E.sflags[tr];
      const bool owned = fl & TF_OWNED;
      const bool shared = sf & SF_SHARED;
      const bool natural = shared && owned && !(sf & SF_DEFER) && !A.plan_mode;   // merged in-kernel
      const bool rec = shared && (owned || (sf & SF_SEND)) && !natural;           // sorted record
      const int rk = row_key<DIM, SP>(P, s, x);
      int lb[3];
#pragma unroll
      for (int s2 = 0; s2 < S; ++s2) {
        const int OFFS = (SP == SP_H1) ? 0 : s2 * (SP == SP_ND ? P * (P + 1) * (P + 1) : (P + 1) * P * P);
        lb[s2] = OFFS + x[0] + ext_of<SP>(P, s2, 0) * (x[1] + ext_of<SP>(P, s2, 1) * x[2]);
      }
      const int lr = lb[s];
      const int gid = gmap[lr];
      const double sig_row = (bsg[lr] & 128) ? -1.0 : 1.0;
      int64_t out = 0;
      int rowlen = 0;
      uint32_t posw[(W + 3) / 4];  // final position of every stencil slot in the CSR row, 4 per word (255: none)
      auto pos_of = [&](int j) -> int { return (int)((posw[j >> 2] >> (8 * (j & 3))) & 255u); };
      const int64_t own_ord = ii >= nsh ? A.ownbase[el] + own0 + (ii - nsh) : 0;
      if (!natural && !rec && A.plan_mode == 0) {
        // own row: its slot positions are topological and come from the setup position table
        out = ld_stream(A.row_ptr + (gid - A.row_begin), l2_policy_first());
        const uint4 *op = reinterpret_cast<const uint4 *>(A.ownpos + own_ord * own_w(W));
#pragma unroll
        for (int q = 0; q < own_w(W) / 16; ++q) {
          const uint4 t = ld_stream(op + q, l2_policy_first());
          const uint32_t w4[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (4 * q + c < (W + 3) / 4) posw[4 * q + c] = w4[c];
        }
      } else if (!natural) {
        if (rec) {
          const int c0 = cls_of(tr, 0), c1 = cls_of(tr, 1), c2 = DIM == 3 ? cls_of(tr, 2) : 1;
          const int nI = (c0 == 1) + (c1 == 1) + (DIM == 3 ? (c2 == 1) : 0);
          const int type = (nI == 0) ? 0 : (nI == DIM ? 3 : (DIM == 3 ? nI : 1));
          out = ((int64_t)E.rec[tr] + (gid - A.base[type][T.ent[tr]])) * A.rstride;
        }
        LOR_TSTAMP(ii == nsh, 11);
        // P0 of every block of the row (ascending block base order), then the final position of
        // every stencil slot: P0 of its block + rank in the block's sub-box (per orientation code)
        const int64_t key = (int64_t)s * NROWKEY + rk;
        const uint4 *tz4 = reinterpret_cast<const uint4 *>(A.tabs.size + key * CF::TZS);
        uint32_t wv[SP == SP_H1 ? 1 : W];  // slot words (H1: validity and offsets are closed-form)
        if constexpr (SP != SP_H1) {
#pragma unroll
          for (int j = 0; j < W; ++j) wv[j] = __ldg(A.tabs.slot + key * W + j);
        }
#pragma unroll
        for (int q = 0; q < CF::TZS / 16; ++q) {
          const uint4 t = __ldg(tz4 + q);
          const uint32_t w4[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
          for (int c = 0; c < 16; ++c) ts[(16 * q + c) * CF::NT] = (unsigned char)(w4[c >> 2] >> (8 * (c & 3)));
        }
        unsigned char *p0 = ts + CF::TZS * CF::NT;
        if (NB <= 32) {  // all block sizes read before the first P0 store (no load-after-store chain)
          unsigned char sz[NB <= 32 ? NB : 1];
#pragma unroll
          for (int i = 0; i < (NB <= 32 ? NB : 1); ++i) sz[i] = i < nb ? ts[blist[i] * CF::NT] : 0;
#pragma unroll
          for (int i = 0; i < (NB <= 32 ? NB : 1); ++i)
            if (i < nb) {
              p0[blist[i] * CF::NT] = (unsigned char)rowlen;
              rowlen += sz[i];
            }
        } else {
          for (int i = 0; i < nb; ++i) {
            const int b = blist[i];
            p0[b * CF::NT] = (unsigned char)rowlen;
            rowlen += ts[b * CF::NT];
          }
        }
        // every slot's P0 and rank-table load issued before any position is stored
        unsigned char pz[W];
        unsigned char lx[W];
#pragma unroll
        for (int j = 0; j < W; ++j) {
          pz[j] = 255;
          lx[j] = 0;
          bool valid;
          int s2 = 0, l;
          if constexpr (SP == SP_H1) {
            valid = true;
#pragma unroll
            for (int a = 0; a < DIM; ++a) valid = valid && (unsigned)(x[a] + h1_off<DIM>(j, a)) <= (unsigned)P;
            l = lb[0] + h1_dl<DIM, P>(j);
          } else {
            valid = (wv[j] & 127) != 127;
            s2 = (wv[j] >> 24) & 3;
            l = (s2 == 0 ? lb[0] : (s2 == 1 ? lb[S > 1 ? 1 : 0] : lb[S > 2 ? 2 : 0])) + (int)(int8_t)(dlt[s * W + j] & 255);
          }
          if (valid) {
            const int b = bsg[l] & 127;
            pz[j] = p0[b * CF::NT];
            lx[j] = __ldg(A.tabs.lex + ((key * W + j) << 3) + T.orient[b - 27 * s2]);
          }
        }
#pragma unroll
        for (int i = 0; i < (W + 3) / 4; ++i) {
          uint32_t v = 0;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int j = 4 * i + c;
            const uint32_t b = j < W ? (pz[j] == 255 ? 255u : (uint32_t)(unsigned char)(pz[j] + lx[j])) : 255u;
            v |= b << (8 * c);
          }
          posw[i] = v;
        }
        if (A.plan_mode == 2) {  // setup own-row position pass: store the row's positions, no values
          uint32_t w[own_w(W) / 4];
#pragma unroll
          for (int i = 0; i < own_w(W) / 4; ++i) w[i] = i < (W + 3) / 4 ? posw[i] : 0xffffffffu;
          uint4 *op = reinterpret_cast<uint4 *>(A.ownpos + own_ord * own_w(W));
#pragma unroll
          for (int q = 0; q < own_w(W) / 16; ++q) op[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
          continue;
        }
        LOR_TSTAMP(ii == nsh, 12);
      }
      double acc[W];
      switch (s) {
        case 0: row_values<DIM, SP, P, 0, NC>(cm, x, CF::NRING, acc); break;
        case 1: if (S > 1) row_values<DIM, SP, P, (S > 1 ? 1 : 0), NC>(cm, x, CF::NRING, acc); break;
        default: if (S > 2) row_values<DIM, SP, P, (S > 2 ? 2 : 0), NC>(cm, x, CF::NRING, acc); break;
      }
      LOR_TSTAMP(ii == nsh, 13);
      if (natural) {  // natural-order partial row (slot order), column signs applied by the merge
        double2 *dst = reinterpret_cast<double2 *>(A.nval + (el * CF::NDPE + lr) * rec_w8(W));
#pragma unroll
        for (int j = 0; j + 1 < W; j += 2) dst[j / 2] = make_double2(acc[j] * sig_row, acc[j + 1] * sig_row);
        if (W & 1) A.nval[(el * CF::NDPE + lr) * rec_w8(W) + W - 1] = acc[W - 1] * sig_row;
      } else if (!rec) {
        const uint64_t pf = l2_policy_first();
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const int ps = pos_of(j);
          if (ps != 255) {
            int l;
            if constexpr (SP == SP_H1) {
              l = lb[0] + h1_dl<DIM, P>(j);
            } else {
              const int dd = dlt[s * W + j], s2 = (dd >> 8) & 3;
              l = (s2 == 0 ? lb[0] : (s2 == 1 ? lb[S > 1 ? 1 : 0] : lb[S > 2 ? 2 : 0])) + (int)(int8_t)(dd & 255);
            }
            const double v = acc[j] * ((bsg[l] & 128) ? -sig_row : sig_row);
            st_hint(A.col + out + ps, gmap[l], pf);
            st_hint(A.val + out + ps, v, pf);
          }
        }
      } else {  // sorted record {column | block base << 32, value (plan pass: slot | 64 if flipped)}
        double2 *dst = reinterpret_cast<double2 *>(A.scratch) + out;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const int ps = pos_of(j);
          if (ps != 255) {
            int l;
            if constexpr (SP == SP_H1) {
              l = lb[0] + h1_dl<DIM, P>(j);
            } else {
              const int dd = dlt[s * W + j], s2 = (dd >> 8) & 3;
              l = (s2 == 0 ? lb[0] : (s2 == 1 ? lb[S > 1 ? 1 : 0] : lb[S > 2 ? 2 : 0])) + (int)(int8_t)(dd & 255);
            }
            const int bs = bsg[l];
            const double v = acc[j] * ((bs & 128) ? -sig_row : sig_row);
            dst[ps] = make_double2(__longlong_as_double(((long long)(unsigned)blk[bs & 127].base << 32) | (unsigned)gmap[l]),
                                   A.plan_mode ? (double)(j | ((bs & 128) ? 64 : 0)) : v);
          }
        }
        dst[A.rstride - 1] = make_double2(__longlong_as_double(((long long)(unsigned)lr << 32) | (long long)(unsigned)rowlen), 0.0);
      }
    }
    __syncthreads();  // every thread has read s_ownacc
    if (tid == 0) s_ownacc += nown;
  }
  // shared rows are merged by the separate pass k_merge_rows (lor_kernels.cu)
  if (A.tstamp) {
    LOR_STAMP(3);  // thread 0 done
    __syncthreads();
    LOR_STAMP(4);  // CTA done
  }
}

template <int DIM, int SP, int P, int KZ>
cudaError_t launch_asm_p(const AsmArgs &a, int quad, cudaStream_t st, int *smem_out) {
  using CF = AsmCfg<DIM, SP, P, KZ>;
  const int smem = CF::SMEM;
  if (smem_out) { *smem_out = smem; return cudaSuccess; }
  if (a.nel_local <= 0) return cudaSuccess;
  // 3D H1 vertex rule: 5 CTAs/SM (96 registers) measured fastest at C2; LOR_MINB=4/6/8 for experiments
  static const int minb = getenv("LOR_MINB") ? atoi(getenv("LOR_MINB")) : 5;
  // dev experiment: LOR_SMEM_PAD inflates the dynamic shared memory to cap CTAs per SM
  static const int pad = getenv("LOR_SMEM_PAD") ? atoi(getenv("LOR_SMEM_PAD")) : 0;
  auto run = [&](auto k) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem + pad);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    // L2 prefetch distance = resident CTAs of the grid (LOR_APF=0: off)
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 128, smem + pad);
    static const bool apf = !(getenv("LOR_APF") && !atoi(getenv("LOR_APF")));
    AsmArgs b = a;
    b.pf_dist = apf ? (int64_t)nsm * occ : 0;
    k<<<(unsigned)a.nel_local, 128, smem + pad, st>>>(b);
  };
  if (quad == 0) {
    if (DIM == 3 && SP == SP_H1 && minb == 8) run(k_assemble<DIM, SP, P, 0, KZ, (DIM == 3 && SP == SP_H1) ? 8 : 4>);
    else if (DIM == 3 && SP == SP_H1 && minb == 6) run(k_assemble<DIM, SP, P, 0, KZ, (DIM == 3 && SP == SP_H1) ? 6 : 4>);
    else if (DIM == 3 && SP == SP_H1 && minb == 4) run(k_assemble<DIM, SP, P, 0, KZ, 4>);
    else run(k_assemble<DIM, SP, P, 0, KZ, CF::MINB_SMEM>);
  } else {
    run(k_assemble<DIM, SP, P, 1, KZ, 4>);
  }
  return cudaGetLastError();
}

template <int DIM, int SP, int P>
cudaError_t launch_asm_kz(const AsmArgs &a, int quad, cudaStream_t st, int *smem_out) {
  constexpr int NENT = Tr<DIM, SP>::NENT;
  constexpr int full = NENT * ipow_c(P, DIM) * 8;
  constexpr int KZ = (DIM == 2 || full <= 48 * 1024) ? P : ((NENT * P * P * 8 * 3 <= 64 * 1024) ? 2 : 1);
  return launch_asm_p<DIM, SP, P, KZ>(a, quad, st, smem_out);
}

}  // namespace lorb
