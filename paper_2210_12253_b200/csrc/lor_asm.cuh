// lor_asm.cuh -- templates of the fused element assembly kernel (k_assemble) and the shared-row
// merge (finalize_ose).  Instantiated per (dim, space, p) in generated translation units
// (build.py) so the sm_100a build runs in parallel.  See lor_kernels.cu for the pipeline.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lor_cells.cuh"
#include "lor_device.cuh"
#include "lor_kernels.h"

namespace lorb {

__host__ __device__ constexpr int ipow_c(int b, int e) { return e == 0 ? 1 : b * ipow_c(b, e - 1); }

// ------------------------------------------------------------------------ small helpers
// L2 eviction priorities: the CSR output is written once and never re-read by this kernel
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
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(double *a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
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
// natural-order partial-row records: row strides padded to whole 32-byte sectors and written
// completely (invalid slots as 0 / -1), so a record sector is never partially valid in L2
__host__ __device__ constexpr int rec_w8(int W) { return (W + 3) / 4 * 4; }   // doubles per row
__host__ __device__ constexpr int rec_w4(int W) { return (W + 7) / 8 * 8; }   // int32 per row

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
  static constexpr int NW = 4;                                    // warps per CTA
  static constexpr int RG = 16;                                   // rows per warp group
  static constexpr int NBP = (NB + 7) / 8 * 8;                    // P0 entries per row (uint16)
  // shared memory layout (bytes)
  static constexpr int OFF_BLK = 0;
  static constexpr int OFF_OS = OFF_BLK + NB * (int)sizeof(Blk);            // ordsig[NB] uint16
  static constexpr int OFF_BL = OFF_OS + NB * 2;                           // blist[NB] uint8
  static constexpr int OFF_GM = (OFF_BL + NB + 15) / 16 * 16;              // gmap[NDPE] int32
  static constexpr int OFF_BS = OFF_GM + NDPE * 4;                         // bsg[NDPE] uint8
  static constexpr int OFF_X = (OFF_BS + NDPE + 15) / 16 * 16;
  static constexpr int OFF_CM = (OFF_X + DIM * NPTS * 8 + 15) / 16 * 16;
  static constexpr int OFF_VB = (OFF_CM + NENT * NCELL * 8 + 15) / 16 * 16;  // per warp: RG rows x W values
  static constexpr int OFF_RM = (OFF_VB + NW * RG * W * 8 + 15) / 16 * 16;   // per warp: RG row records
  static constexpr int OFF_P0 = OFF_RM + NW * RG * 32;                     // per warp: RG x P0[NBP] uint16
  static constexpr int RMS = (MAXL + 7) / 8 * 8;                  // merge-plan row (uint16 entries)
  static constexpr int TMPB = tab_tzs(NB) + RMS * 2;              // per-row staging of table rows
  static constexpr int OFF_TMP = (OFF_P0 + NW * RG * NBP * 2 + 15) / 16 * 16;
  static constexpr int OFF_DL = OFF_TMP + NW * RG * TMPB;                  // dl[S][W] int8 (slot -> local offset)
  static constexpr int SMEM = (OFF_DL + S * W + 15) / 16 * 16;
};

// per-row record kept by the row's thread for the warp-wide emission
struct __align__(16) RowRec {
  int64_t out;     // mode 1, 3: CSR offset of the row; mode 2: scratch entry offset of the record
  int64_t recid;   // mode 4: natural record row; mode 2: record length (header)
  int32_t lb[3];   // local index of the row position in each column sub-lattice's layout
  uint16_t rk;     // row key
  uint8_t mode;    // 0 skip, 1 own row, 2 partial-row record (sorted, merged at run time), 4 natural-order partial row
  uint8_t s;       // sub-lattice
};
static_assert(sizeof(RowRec) == 32, "RowRec");

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
template <int P, int NC>
__device__ __forceinline__ void cells_h1_corner(const double *__restrict__ X, double *__restrict__ cm, int k0, int ncell,
                                                double alpha, double beta, int &bad) {
  constexpr int NP1 = P + 1, NPT = NP1 * NP1 * NP1;
  constexpr int NRING_ = P;  // only used with KZ == P for H1 (whole element)
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
    const double sa = 0.125 * alpha / det;
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
    double diag = sg[0] * Qs[0] + sg[1] * Qs[1] + sg[2] * Qs[2] + 0.125 * beta * det;
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
      o[tri(8, q, q) * NC] = diag;
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (!((q >> d) & 1)) o[tri(8, q, q ^ (1 << d)) * NC] = edge[d];
      // face diagonal of (d,d') is written by the lower of its two corners q, q^d^d'
      if (q < (q ^ 3)) o[tri(8, q ^ 1, q ^ 2) * NC] = fdg[0];
      if (q < (q ^ 5)) o[tri(8, q ^ 1, q ^ 4) * NC] = fdg[1];
      if (q < (q ^ 6)) o[tri(8, q ^ 2, q ^ 4) * NC] = fdg[2];
      if (q < 4) o[tri(8, q, q ^ 7) * NC] = 0.0;
    }
  }
}

template <int DIM, int SP, int P, int QUAD>
__device__ __forceinline__ bool compute_cell(const double *__restrict__ X, int cx, int cy, int cz, double alpha,
                                             double beta, double *__restrict__ out, int NC, int ci) {
  constexpr int NP1 = P + 1;
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
      bool ok = cell_h1_3d<QUAD>(C, alpha, beta, A);
#pragma unroll
      for (int i = 0; i < 36; ++i) out[i * NC + ci] = A[i];
      return ok;
    } else if (SP == SP_ND) {
      double A[78];
      bool ok = cell_nd<QUAD>(C, alpha, beta, A);
#pragma unroll
      for (int i = 0; i < 78; ++i) out[i * NC + ci] = A[i];
      return ok;
    } else {
      double A[21];
      bool ok = cell_rt<QUAD>(C, alpha, beta, A);
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
    bool ok = cell_h1_2d<QUAD>(C, alpha, beta, A);
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

// Warp-wide emission of one row (lanes = stencil slots): each lane places its column at
// P0(block) + rank inside the block's sub-box (setup table per orientation code of the block's
// entity), so the row comes out in ascending global column order and the warp's stores cover a
// contiguous range (coalesced).  P0 per block was prepared by the row's thread (p0r).
template <int DIM, int SP, int P>
__device__ __forceinline__ void emit_row(const AsmArgs &A, const RowRec &R, const uint32_t *wpre,
                                         const double *__restrict__ vrow,
                                         const uint16_t *__restrict__ p0r, const Blk *__restrict__ blk,
                                         const ElemTopo &T, const int32_t *__restrict__ gmap,
                                         const uint8_t *__restrict__ bsg, const int8_t *__restrict__ dlt, int lane) {
  using C = Tr<DIM, SP>;
  constexpr int W = C::W;
  const int64_t key = (int64_t)R.s * NROWKEY + R.rk;
  int32_t *colr = A.col + R.out;
  double *valr = A.val + R.out;
  if (R.mode == 4) {  // natural-order partial row: no position work, dense sector-aligned record
    constexpr int W8 = rec_w8(W), W4 = rec_w4(W);
    const uint64_t pl = l2_policy_last();
#pragma unroll
    for (int j0 = 0; j0 < W4; j0 += 32) {
      const int j = j0 + lane;
      double v = 0.0;
      int gid = -1;
      if (j < W) {
        const uint32_t w = wpre[j0 / 32];
        if ((w & 127) != 127) {
          const int s2 = (w >> 24) & 3;
          const int l = R.lb[s2] + dlt[R.s * W + j];
          gid = gmap[l];
          v = (bsg[l] & 128) ? -vrow[j] : vrow[j];
        }
      }
      if (j < W8) st_hint(A.nval + R.recid * W8 + j, v, pl);
      if (j < W4) st_hint(A.ngid + R.recid * W4 + j, gid, pl);
    }
    return;
  }
#pragma unroll
  for (int j0 = 0; j0 < W; j0 += 32) {
    const int j = j0 + lane;
    if (j < W) {
      const uint32_t w = wpre[j0 / 32];
      const int bw = w & 127;
      if (bw != 127) {
        const int s2 = (w >> 24) & 3;
        const int l = R.lb[s2] + dlt[R.s * W + j];
        const int gid = gmap[l];
        const int bs = bsg[l];
        const int b = bs & 127;
        {
          const int lex = __ldg(A.tabs.lex + ((key * W + j) << 3) + T.orient[b - 27 * s2]);
          const int pos = (int)(p0r[b] & 255u) + lex;
          const double v = (bs & 128) ? -vrow[j] : vrow[j];
          if (R.mode == 1) {
            const uint64_t pf = l2_policy_first();
            st_hint(colr + pos, gid, pf);
            st_hint(valr + pos, v, pf);
          } else {
            double2 *dst = reinterpret_cast<double2 *>(A.scratch) + R.out;
            dst[pos] = make_double2(__longlong_as_double(((long long)(unsigned)blk[b].base << 32) | (unsigned)gid),
                                    A.plan_mode ? (double)j : v);
          }
        }
      }
    }
  }
  if (R.mode == 2 && lane == 0)  // record header: length, local row
    reinterpret_cast<double2 *>(A.scratch)[R.out + A.rstride - 1] = make_double2(
        __longlong_as_double(((long long)(unsigned)R.lb[R.s] << 32) | (long long)(unsigned)R.recid), 0.0);
}

template <int DIM, int SP, int P, int QUAD, int KZ>
__global__ void __launch_bounds__(128, 4) k_assemble(AsmArgs A) {
  using CF = AsmCfg<DIM, SP, P, KZ>;
  constexpr int S = CF::S, W = CF::W, NB = CF::NB, NC = CF::NCELL;
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
  __shared__ int s_nb, s_fin_n, s_bad;
  __shared__ int s_fin[27];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int RG = CF::RG, NBP = CF::NBP;
  double *vb = reinterpret_cast<double *>(smem + CF::OFF_VB) + warp * RG * W;
  RowRec *rr = reinterpret_cast<RowRec *>(smem + CF::OFF_RM) + warp * RG;
  uint16_t *p0r = reinterpret_cast<uint16_t *>(smem + CF::OFF_P0) + warp * RG * NBP;
  int8_t *dlt = reinterpret_cast<int8_t *>(smem + CF::OFF_DL);
  if ((int64_t)blockIdx.x >= A.nel_local) return;
  const int64_t el = A.order ? A.order[blockIdx.x] : blockIdx.x;  // local element (locality-preserving order)
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
    for (int i = tid; i < NX2; i += blockDim.x) xd[i] = __ldg(xs + i);
    if ((DIM * CF::NPTS) & 1) {
      if (tid == 0) X[DIM * CF::NPTS - 1] = __ldg(A.X + el * A.xstride + DIM * CF::NPTS - 1);
    }
    if (tid == 0) { s_fin_n = 0; s_bad = 0; }
  }
  __syncthreads();
  // ---- element block table, canonical axis order/directions, ascending-base order
  if (tid < NB) {
    const int s = tid / 27, tau = tid - 27 * s;
    Blk B;
    if (DIM == 2 && tau >= 9) {
      B.size = 0; B.g0 = 0; B.base = 0; B.sigma = 1; B.ord = 0; B.str[0] = B.str[1] = B.str[2] = 0;
    } else {
      block_affine<DIM, SP>(P, s, tau, T, A.base, B);
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
  // ---- slot -> local index offset relative to the row position in the column sub-lattice layout
  for (int i = tid; i < S * W; i += blockDim.x) {
    const int s = i / W, j = i - s * W;
    int jj = j, s2 = 0;
    while (s2 < S - 1 && jj >= st_n<DIM, SP>(s, s2)) { jj -= st_n<DIM, SP>(s, s2); ++s2; }
    const int nx = st_hi<SP>(s, s2, 0) - st_lo<SP>(s, s2, 0) + 1, ny = st_hi<SP>(s, s2, 1) - st_lo<SP>(s, s2, 1) + 1;
    const int dx = st_lo<SP>(s, s2, 0) + jj % nx, dy = st_lo<SP>(s, s2, 1) + (jj / nx) % ny;
    const int dz = (DIM == 3) ? st_lo<SP>(s, s2, 2) + jj / (nx * ny) : 0;
    dlt[i] = (int8_t)(dx + ext_of<SP>(P, s2, 0) * (dy + ext_of<SP>(P, s2, 1) * dz));
  }
  // ---- element restriction in shared memory: global id and block/sign of every local dof
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

  // ---- z-chunks of cell layers
  constexpr int NCHUNK = (DIM == 3) ? (P + KZ - 1) / KZ : 1;
  for (int ch = 0; ch < NCHUNK; ++ch) {
    const int k0 = (DIM == 3) ? ch * KZ : 0;
    const int k1 = (DIM == 3) ? ((k0 + KZ < P) ? k0 + KZ : P) : P;
    const int ncell = (DIM == 3) ? (k1 - k0) * P * P : P * P;
    if (ch > 0) __syncthreads();  // previous chunk's rows done before its ring slots are reused
    if (DIM == 3 && SP == SP_H1 && QUAD == 0 && KZ == P) {
      int bad = 0;
      cells_h1_corner<P, NC>(X, cm, k0, ncell, A.alpha, A.beta, bad);
      if (bad) s_bad = bad;
    } else {
      for (int c = tid; c < ncell; c += blockDim.x) {
        const int cx = c % P, cy = (c / P) % P, cz = (DIM == 3) ? k0 + c / (P * P) : 0;
        const int ci = (DIM == 3) ? (((cz % CF::NRING) * P) + cy) * P + cx : cy * P + cx;
        if (!compute_cell<DIM, SP, P, QUAD>(X, cx, cy, cz, A.alpha, A.beta, cm, NC, ci)) s_bad = 1 + cx + P * (cy + P * cz);
      }
    }
    __syncthreads();
    if (s_bad && tid == 0) report_error(A.err, 2, A.elem_begin + el, s_bad - 1);
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
    // groups of RG rows per warp: the row's thread accumulates its values and prepares P0 of its
    // blocks (all global loads of the row issued here, in parallel across rows), then the warp
    // emits the rows one at a time, lanes = stencil slots
    for (int g0 = warp * RG; g0 < nrows; g0 += CF::NW * RG) {
      const int r = g0 + lane;
      if (lane < RG) {
        RowRec R;
        R.mode = 0;
        R.out = 0;
        R.recid = 0;
        R.rk = 0;
        R.s = 0;
        R.lb[0] = R.lb[1] = R.lb[2] = 0;
        if (r < nrows) {
          int s = 0, rq = r;
          if (S > 1 && rq >= nrow_s0) { rq -= nrow_s0; s = 1; if (rq >= nrow_s1) { rq -= nrow_s1; s = 2; } }
          const int ex = ext_of<SP>(P, s, 0), ey = ext_of<SP>(P, s, 1);
          int x[3];
          x[0] = rq % ex;
          x[1] = (rq / ex) % ey;
          x[2] = (DIM == 3) ? k0 + rq / (ex * ey) : 0;
          const int tr = row_tau<DIM, SP>(P, s, x);
          const uint8_t fl = T.flags[tr], sf = E.sflags[tr];
          const bool owned = fl & TF_OWNED;
          const bool shared = sf & SF_SHARED;
          const bool local_plan = shared && owned && !(sf & SF_DEFER) && !A.plan_mode;  // mode 3
          const bool rec = shared && (owned || (sf & SF_SEND)) && !local_plan;      // mode 2
          if ((owned && !A.plan_mode) || rec || local_plan) {
            R.s = (uint8_t)s;
            const int rk = row_key<DIM, SP>(P, s, x);
            R.rk = (uint16_t)rk;
#pragma unroll
            for (int s2 = 0; s2 < S; ++s2) {
              const int OFFS = (SP == SP_H1) ? 0 : s2 * (SP == SP_ND ? P * (P + 1) * (P + 1) : (P + 1) * P * P);
              R.lb[s2] = OFFS + x[0] + ext_of<SP>(P, s2, 0) * (x[1] + ext_of<SP>(P, s2, 1) * x[2]);
            }
            const int lr = R.lb[s];
            const int gid = gmap[lr];
            const double sig_row = (bsg[lr] & 128) ? -1.0 : 1.0;
            int t_in = 0;
            if (shared) {
              const int c0 = cls_of(tr, 0), c1 = cls_of(tr, 1), c2 = DIM == 3 ? cls_of(tr, 2) : 1;
              const int nI = (c0 == 1) + (c1 == 1) + (DIM == 3 ? (c2 == 1) : 0);
              const int type = (nI == 0) ? 0 : (nI == DIM ? 3 : (DIM == 3 ? nI : 1));
              t_in = gid - A.base[type][T.ent[tr]];
            }
            const int64_t recid = shared ? (int64_t)E.rec[tr] + t_in : 0;
            // P0 of the row's blocks: the row's block-size table row (and for planned shared rows
            // its merge-plan row) are fetched with 16-byte loads into the (still free) value row
            uint16_t *pr = p0r + lane * NBP;
            if (local_plan) {
              R.mode = 4;
              R.recid = el * CF::NDPE + lr;
            } else {
              constexpr int TZS = tab_tzs(NB);
              const uint4 *tz4 = reinterpret_cast<const uint4 *>(A.tabs.size + ((int64_t)s * NROWKEY + rk) * TZS);
              uint4 *tmp4 = reinterpret_cast<uint4 *>(smem + CF::OFF_TMP + (warp * RG + lane) * CF::TMPB);
              const uint8_t *tzs = reinterpret_cast<const uint8_t *>(tmp4);
#pragma unroll
              for (int q = 0; q < TZS / 16; ++q) tmp4[q] = __ldg(tz4 + q);
              int run = 0;
              for (int i = 0; i < nb; ++i) {
                const int b = blist[i];
                pr[b] = (uint16_t)(run | 0xff00);
                run += tzs[b];
              }
              if (!rec) {
                R.mode = 1;
                R.out = A.row_ptr[gid - A.row_begin];
              } else {
                R.mode = 2;
                R.out = recid * A.rstride;
                R.recid = run;
              }
            }
            double acc[W];
            switch (s) {
              case 0: row_values<DIM, SP, P, 0, NC>(cm, x, CF::NRING, acc); break;
              case 1: if (S > 1) row_values<DIM, SP, P, (S > 1 ? 1 : 0), NC>(cm, x, CF::NRING, acc); break;
              default: if (S > 2) row_values<DIM, SP, P, (S > 2 ? 2 : 0), NC>(cm, x, CF::NRING, acc); break;
            }
#pragma unroll
            for (int j = 0; j < W; ++j) vb[lane * W + j] = acc[j] * sig_row;
          }
        }
        rr[lane] = R;
      }
      __syncwarp();
      const int nr = (nrows - g0 < RG) ? nrows - g0 : RG;
      // slot words of the next row are fetched while the current row is emitted
      uint32_t wcur[(W + 31) / 32], wnext[(W + 31) / 32];
      {
        const RowRec &R0 = rr[0];
        const int64_t key0 = (int64_t)R0.s * NROWKEY + R0.rk;
#pragma unroll
        for (int h = 0; h < (W + 31) / 32; ++h) {
          const int j = h * 32 + lane;
          wcur[h] = (j < W) ? __ldg(A.tabs.slot + key0 * W + j) : 127u;
        }
      }
      for (int i = 0; i < nr; ++i) {
        if (i + 1 < nr) {
          const RowRec &Rn = rr[i + 1];
          const int64_t keyn = (int64_t)Rn.s * NROWKEY + Rn.rk;
#pragma unroll
          for (int h = 0; h < (W + 31) / 32; ++h) {
            const int j = h * 32 + lane;
            wnext[h] = (j < W) ? __ldg(A.tabs.slot + keyn * W + j) : 127u;
          }
        }
        const RowRec &Ri = rr[i];
        if (Ri.mode) emit_row<DIM, SP, P>(A, Ri, wcur, vb + i * W, p0r + i * NBP, blk, T, gmap, bsg, dlt, lane);
#pragma unroll
        for (int h = 0; h < (W + 31) / 32; ++h) wcur[h] = wnext[h];
      }
      __syncwarp();
    }
  }
  if (A.plan_mode) return;
  // ---- arrival on shared owned entities; the last element to arrive adds up their shared values
  __threadfence();
  __syncthreads();
  if (tid < CF::NSLOT) {
    const int tau = tid;
    const uint8_t sf = E.sflags[tau];
    if ((sf & SF_SHARED) && !(sf & (SF_DEFER | SF_SEND)) && E.ose[tau] >= 0) {
      const int oi = E.ose[tau];
      const int kk = A.ose[oi].k;
      const int old = atomicAdd(A.counters + oi, 1);
      if (old == kk - 1) {
        A.counters[oi] = 0;
        const int pos = atomicAdd(&s_fin_n, 1);
        s_fin[pos] = oi;
      }
    }
  }
  __syncthreads();
  const int nfin = s_fin_n;
  if (nfin > 0) {
    __threadfence();
    // Emit every row of the entities whose last contributor is this element: final position q of
    // row r takes its column from the first contributor holding it and its value from the sum over
    // all contributors holding it, in element order (setup merge plan: contributor m's stencil slot
    // at q, or 255).
    __shared__ int s_fk[27], s_fnr[27], s_fpre[28];
    __shared__ int64_t s_fpb[27];
    __shared__ int s_felem[27 * MAX_VALENCE];
    constexpr int MAXFR = 256;  // rows whose offsets are staged (value rows hold >= 256 * 12 B)
    int64_t *s_rowoff = reinterpret_cast<int64_t *>(smem + CF::OFF_VB);  // value rows are free now
    int *s_rowlen = reinterpret_cast<int *>(s_rowoff + MAXFR);
    __shared__ int s_rpre[28];
    for (int i = tid; i < nfin; i += blockDim.x) {
      const Ose O = A.ose[s_fin[i]];
      s_fk[i] = O.k;
      s_fnr[i] = O.nrows;
      s_fpb[i] = A.pbase[s_fin[i]];
      for (int m = 0; m < O.k; ++m) s_felem[i * MAX_VALENCE + m] = A.ose_elem[O.slot_off + m];
    }
    __syncthreads();
    if (tid == 0) {
      int accr = 0;
      for (int i = 0; i < nfin; ++i) { s_rpre[i] = accr; s_fpre[i] = accr * W; accr += s_fnr[i]; }
      s_rpre[nfin] = accr;
      s_fpre[nfin] = accr * W;
    }
    __syncthreads();
    const int nfr = s_rpre[nfin];
    {
      int i = 0;
      for (int rr2 = tid; rr2 < nfr && rr2 < MAXFR; rr2 += blockDim.x) {
        while (rr2 >= s_rpre[i + 1]) ++i;
        const int64_t g = (int64_t)A.ose[s_fin[i]].gid_base + (rr2 - s_rpre[i]) - A.row_begin;
        const int64_t a = A.row_ptr[g];
        s_rowoff[rr2] = a;
        s_rowlen[rr2] = (int)(A.row_ptr[g + 1] - a);
      }
    }
    __syncthreads();
    const int total = s_fpre[nfin];
    int i = 0;
    for (int it = tid; it < total; it += blockDim.x) {
      while (it >= s_fpre[i + 1]) ++i;  // items ascend per thread: amortised O(1)
      const int rem = it - s_fpre[i];
      const int r = rem / W, q = rem - r * W;
      const int rg2 = s_rpre[i] + r;
      int64_t ro;
      int len;
      if (rg2 < MAXFR) { ro = s_rowoff[rg2]; len = s_rowlen[rg2]; }
      else {
        const int64_t g = (int64_t)A.ose[s_fin[i]].gid_base + r - A.row_begin;
        ro = A.row_ptr[g];
        len = (int)(A.row_ptr[g + 1] - ro);
      }
      if (q >= len) continue;
      const int k = s_fk[i];
      const int rstr = ((2 * k + W * k) + 1) & ~1;
      const uint8_t *pr = A.plan + s_fpb[i] + (int64_t)r * rstr;
      const uint16_t *lrow = reinterpret_cast<const uint16_t *>(pr);
      const uint8_t *js = pr + 2 * k + q * k;
      int gid = 0;
      bool have = false;
      double sum = 0.0;
      for (int m = 0; m < k; ++m) {
        const int jm = __ldg(js + m);
        if (jm == 255) continue;
        const int64_t rr3 = (int64_t)s_felem[i * MAX_VALENCE + m] * CF::NDPE + __ldg(lrow + m);
        if (!have) { gid = __ldcg(A.ngid + rr3 * rec_w4(W) + jm); have = true; }
        sum += __ldcg(A.nval + rr3 * rec_w8(W) + jm);
      }
      const uint64_t pf = l2_policy_first();
      st_hint(A.col + ro + q, gid, pf);
      st_hint(A.val + ro + q, sum, pf);
    }
  }
}

template <int DIM, int SP, int P, int KZ>
cudaError_t launch_asm_p(const AsmArgs &a, int quad, cudaStream_t st, int *smem_out) {
  using CF = AsmCfg<DIM, SP, P, KZ>;
  const int smem = CF::SMEM;
  if (smem_out) { *smem_out = smem; return cudaSuccess; }
  if (a.nel_local <= 0) return cudaSuccess;
  if (quad == 0) {
    auto k = k_assemble<DIM, SP, P, 0, KZ>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<(unsigned)a.nel_local, 128, smem, st>>>(a);
  } else {
    auto k = k_assemble<DIM, SP, P, 1, KZ>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<(unsigned)a.nel_local, 128, smem, st>>>(a);
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
