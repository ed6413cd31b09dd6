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
__device__ __forceinline__ void report_error(int *err, int code, int64_t e, int cell) {
  if (atomicCAS(err, 0, code) == 0) {
    err[1] = (int)e;
    err[2] = cell;
  }
}

// length of the class-c segment of the clipped stencil range of column sub-lattice s2 along axis a
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
  int ext[3];
  for (int a = 0; a < 3; ++a) ext[a] = vkind<SP>(s, a) ? p + 1 : p;
  x[0] = r % ext[0];
  r /= ext[0];
  x[1] = r % ext[1];
  x[2] = r / ext[1];
}

template <int DIM, int SP>
__device__ __forceinline__ int row_tau(int p, int s, const int x[3]) {
  int t = coord_cls(vkind<SP>(s, 0), x[0], p) + 3 * coord_cls(vkind<SP>(s, 1), x[1], p);
  if (DIM == 3) t += 9 * coord_cls(vkind<SP>(s, 2), x[2], p);
  return t;
}

// join entity of a row (classes cr) and a column (classes cc): fixed where both sit on the same side
__device__ __forceinline__ int join_cls(int cr, int cc) { return (cr == cc && cr != 1) ? cr : 1; }

// ================================================================================ k_assemble
template <int DIM, int SP, int P, int KZ>
struct AsmCfg {
  using T_ = Tr<DIM, SP>;
  static constexpr int S = T_::S, W = T_::W, NENT = T_::NENT, NSLOT = T_::NSLOT;
  static constexpr int NB = S * 27;                               // block table entries
  static constexpr int NPTS = ipow_c(P + 1, DIM);                 // lattice points (coords)
  static constexpr int CPL = DIM == 3 ? P * P : P * P;            // cells per layer (2D: all)
  static constexpr int NRING = DIM == 3 ? (KZ == P ? P : KZ + 1) : 1;
  static constexpr int NCELL = NRING * CPL;                       // cells resident in smem
  static constexpr int BATCH = 128;                               // rows per batch (= threads)
  // shared memory layout (bytes)
  static constexpr int OFF_BLK = 0;
  static constexpr int OFF_BL = OFF_BLK + NB * (int)sizeof(Blk);
  static constexpr int OFF_X = (OFF_BL + NB + 15) / 16 * 16;
  static constexpr int OFF_CM = OFF_X + DIM * NPTS * 8;
  static constexpr int OFF_RG = OFF_CM + NENT * NCELL * 8;                 // row gids [BATCH][W]
  static constexpr int OFF_RV = OFF_RG + BATCH * W * 4;                    // row vals [BATCH][W]
  static constexpr int OFF_RM = OFF_RV + BATCH * W * 8;                    // row mults [BATCH][W]
  static constexpr int OFF_P0 = (OFF_RM + BATCH * W + 15) / 16 * 16;       // P0 [NB][BATCH] int16
  static constexpr int OFF_META = OFF_P0 + NB * BATCH * 2;                 // per row: out (int64), len, mode
  static constexpr int SMEM = OFF_META + BATCH * 16;
};

struct RowMeta {
  int64_t out;  // DIRECT: CSR offset; RECORD: scratch entry offset
  int32_t len;
  int32_t mode;  // 0 skip, 1 direct, 2 record
};

// per-row value accumulation: acc[slot] = sum over cells containing the row of the cell matrix row
template <int DIM, int SP, int P, int RS, int NC>
__device__ __forceinline__ void row_values(const double *__restrict__ cm, const int x[3], int lay0, int nring,
                                           double *acc) {
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

// positions, global ids and merge multiplicities of the row's stencil slots -> row buffers
template <int DIM, int SP, int P, int RS>
__device__ __forceinline__ int row_emit(const Blk *__restrict__ blk, const uint8_t *__restrict__ blist, int nb,
                                        const ElemTopo &T, const int x[3], int sig_row, const double *acc,
                                        int16_t *__restrict__ p0, int32_t *__restrict__ rg, double *__restrict__ rv,
                                        uint8_t *__restrict__ rm) {
  using C = Tr<DIM, SP>;
  constexpr int S = C::S;
  constexpr int BATCH = 128;
  // P0 of every block present in the row: prefix of sub-box sizes in ascending block-base order
  int run = 0;
  for (int i = 0; i < nb; ++i) {
    const int b = blist[i];
    const int s2 = b / 27, t2 = b - 27 * s2;
    int n = 1;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      int lo, hi;
      seg_bounds<SP>(P, RS, s2, a, x[a], cls_of(t2, a), lo, hi);
      n *= hi >= lo ? hi - lo + 1 : 0;
    }
    p0[b * BATCH] = (int16_t)run;
    run += n;
  }
  int cr[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) cr[a] = (a < DIM) ? coord_cls(vkind<SP>(RS, a), x[a], P) : 1;
  // slots
#pragma unroll
  for (int s2 = 0; s2 < S; ++s2) {
#pragma unroll
    for (int dz = (DIM == 3 ? st_lo<SP>(RS, s2, 2) : 0); dz <= (DIM == 3 ? st_hi<SP>(RS, s2, 2) : 0); ++dz)
#pragma unroll
      for (int dy = st_lo<SP>(RS, s2, 1); dy <= st_hi<SP>(RS, s2, 1); ++dy)
#pragma unroll
        for (int dx = st_lo<SP>(RS, s2, 0); dx <= st_hi<SP>(RS, s2, 0); ++dx) {
          const int y[3] = {x[0] + dx, x[1] + dy, DIM == 3 ? x[2] + dz : 0};
          bool in = true;
#pragma unroll
          for (int a = 0; a < DIM; ++a) in &= (y[a] >= 0) && (y[a] <= (vkind<SP>(s2, a) ? P : P - 1));
          if (!in) continue;
          int cc[3] = {1, 1, 1};
#pragma unroll
          for (int a = 0; a < DIM; ++a) cc[a] = coord_cls(vkind<SP>(s2, a), y[a], P);
          const int t2 = cc[0] + 3 * cc[1] + (DIM == 3 ? 9 * cc[2] : 0);
          const int b = s2 * 27 + t2;
          const Blk &B = blk[b];
          // lexicographic rank inside the sub-box, axes ordered by |stride|
          int off[3], len[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            off[a] = 0;
            len[a] = 1;
          }
#pragma unroll
          for (int a = 0; a < DIM; ++a) {
            int lo, hi;
            seg_bounds<SP>(P, RS, s2, a, x[a], cc[a], lo, hi);
            len[a] = hi - lo + 1;
            off[a] = B.str[a] >= 0 ? y[a] - lo : hi - y[a];
          }
          const int f = B.ord & 3, m = (B.ord >> 2) & 3, sl = (B.ord >> 4) & 3;
          const int pos = p0[b * BATCH] + off[f] + len[f] * (off[m] + len[m] * off[sl]);
          const int gid = B.g0 + B.str[0] * y[0] + B.str[1] * y[1] + B.str[2] * y[2];
          int tj = join_cls(cr[0], cc[0]) + 3 * join_cls(cr[1], cc[1]);
          if (DIM == 3) tj += 9 * join_cls(cr[2], cc[2]);
          const int slot = st_slot<DIM, SP>(RS, s2, dx, dy, dz);
          rg[pos * BATCH] = gid;
          rv[pos * BATCH] = acc[slot] * (double)(sig_row * B.sigma);
          rm[pos * BATCH] = T.val[tj];
        }
  }
  return run;
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

// CTA-cooperative merge of the partial rows of one owned shared entity into final CSR rows.
// For row g with contributing elements i = 0..k-1 (element order) each holding a sorted partial
// list L_i with per-entry multiplicity m (number of lists holding that column), the final
// position of column v is  sum_i sum_{u in L_i, u < v} 1/m(u)  (exact, integer weights), and its
// value is the sum over the lists holding v in element order (deterministic).
static __device__ __noinline__ void finalize_ose(const Ose O, const int32_t *__restrict__ ose_slots, const RecEntry *scratch, int rstride,
                             int64_t row_begin, const int64_t *__restrict__ row_ptr, int32_t *__restrict__ col,
                             double *__restrict__ val, unsigned char *smem, int smem_bytes) {
  const int k = O.k, maxl = rstride;
  // per list: len, weights prefix (maxl+1), cols, vals
  const int per_list = 4 + (maxl + 1) * 4 + maxl * 4 + maxl * 8;
  int rp = smem_bytes / (k * per_list);
  if (rp > O.nrows) rp = O.nrows;
  if (rp < 1) rp = 1;  // smem too small is prevented on the host
  int *s_len = reinterpret_cast<int *>(smem);
  int *s_w = s_len + rp * k;
  int *s_col = s_w + rp * k * (maxl + 1);
  const int ints_before = rp * k * (2 * maxl + 2);  // even: s_val stays 8-byte aligned
  double *s_val = reinterpret_cast<double *>(s_len + ints_before);
  for (int r0 = 0; r0 < O.nrows; r0 += rp) {
    const int nr = (O.nrows - r0 < rp) ? O.nrows - r0 : rp;
    const int nl = nr * k;
    for (int li = threadIdx.x; li < nl; li += blockDim.x) {
      const int row = li / k, slot = li - row * k;
      const int64_t rec = (int64_t)ose_slots[O.slot_off + slot] + r0 + row;
      const int meta = __ldcg(&scratch[rec * rstride].meta);
      s_len[li] = meta >> 8;
    }
    __syncthreads();
    for (int it = threadIdx.x; it < nl * maxl; it += blockDim.x) {
      const int li = it / maxl, e = it - li * maxl;
      if (e >= s_len[li]) continue;
      const int row = li / k, slot = li - row * k;
      const int64_t rec = (int64_t)ose_slots[O.slot_off + slot] + r0 + row;
      const RecEntry *src = scratch + rec * rstride + e;
      const int c = __ldcg(&src->col);
      const int meta = __ldcg(&src->meta);
      const double v = __ldcg(&src->val);
      s_col[li * maxl + e] = c;
      s_val[li * maxl + e] = v;
      s_w[li * (maxl + 1) + e + 1] = WEIGHT_L / (meta & 255);
    }
    __syncthreads();
    for (int li = threadIdx.x; li < nl; li += blockDim.x) {  // exclusive prefix of weights
      int *w = s_w + li * (maxl + 1);
      w[0] = 0;
      for (int e = 0; e < s_len[li]; ++e) w[e + 1] += w[e];
    }
    __syncthreads();
    for (int it = threadIdx.x; it < nl * maxl; it += blockDim.x) {
      const int li = it / maxl, e = it - li * maxl;
      if (e >= s_len[li]) continue;
      const int row = li / k, slot = li - row * k;
      const int v = s_col[li * maxl + e];
      int64_t wsum = 0;
      bool first = true;
      double sum = 0.0;
      for (int j = 0; j < k; ++j) {
        const int lj = row * k + j;
        if (j == slot) {
          wsum += s_w[lj * (maxl + 1) + e];
          sum += s_val[lj * maxl + e];
          continue;
        }
        // lower bound of v in list j
        int lo = 0, hi = s_len[lj];
        const int *cj = s_col + lj * maxl;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (cj[mid] < v) lo = mid + 1;
          else hi = mid;
        }
        wsum += s_w[lj * (maxl + 1) + lo];
        if (lo < s_len[lj] && cj[lo] == v) {
          if (j < slot) first = false;
          sum += s_val[lj * maxl + lo];
        }
      }
      if (first) {
        const int64_t out = row_ptr[(int64_t)O.gid_base + r0 + row - row_begin] + wsum / WEIGHT_L;
        col[out] = v;
        val[out] = sum;
      }
    }
    __syncthreads();
  }
}

template <int DIM, int SP, int P, int QUAD, int KZ>
__global__ void __launch_bounds__(128) k_assemble(AsmArgs A) {
  using CF = AsmCfg<DIM, SP, P, KZ>;
  constexpr int S = CF::S, W = CF::W, NB = CF::NB, BATCH = CF::BATCH, NC = CF::NCELL;
  extern __shared__ __align__(16) unsigned char smem[];
  Blk *blk = reinterpret_cast<Blk *>(smem + CF::OFF_BLK);
  uint8_t *blist = smem + CF::OFF_BL;
  double *X = reinterpret_cast<double *>(smem + CF::OFF_X);
  double *cm = reinterpret_cast<double *>(smem + CF::OFF_CM);
  int32_t *rg = reinterpret_cast<int32_t *>(smem + CF::OFF_RG);
  double *rv = reinterpret_cast<double *>(smem + CF::OFF_RV);
  uint8_t *rm = smem + CF::OFF_RM;
  int16_t *p0 = reinterpret_cast<int16_t *>(smem + CF::OFF_P0);
  RowMeta *meta = reinterpret_cast<RowMeta *>(smem + CF::OFF_META);
  __shared__ ElemTopo T;
  __shared__ ElemSpace E;
  __shared__ int s_nb, s_fin_n, s_bad;
  __shared__ int s_fin[27];

  const int tid = threadIdx.x;
  const int64_t el = blockIdx.x;  // local element index
  if (el >= A.nel_local) return;
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
  // ---- element block table + ascending-base order
  if (tid < NB) {
    const int s = tid / 27, tau = tid - 27 * s;
    Blk B;
    if (DIM == 2 && tau >= 9) { B.size = 0; B.g0 = 0; B.base = 0; B.sigma = 1; B.ord = 0; B.str[0] = B.str[1] = B.str[2] = 0; }
    else block_affine<DIM, SP>(P, s, tau, T, A.base, B);
    blk[tid] = B;
  }
  __syncthreads();
  if (tid < NB) {
    const Blk &B = blk[tid];
    if (B.size > 0) {
      int r = 0;
      for (int b = 0; b < NB; ++b) r += (blk[b].size > 0 && blk[b].base < B.base);
      blist[r] = (uint8_t)tid;
    }
  }
  if (tid == 0) {
    int n = 0;
    for (int b = 0; b < NB; ++b) n += blk[b].size > 0;
    s_nb = n;
  }
  __syncthreads();
  const int nb = s_nb;

  // ---- z-chunks of cell layers
  constexpr int NCHUNK = (DIM == 3) ? (P + KZ - 1) / KZ : 1;
  for (int ch = 0; ch < NCHUNK; ++ch) {
    const int k0 = (DIM == 3) ? ch * KZ : 0;
    const int k1 = (DIM == 3) ? ((k0 + KZ < P) ? k0 + KZ : P) : P;
    // cells of layers [k0, k1)
    const int ncell = (DIM == 3) ? (k1 - k0) * P * P : P * P;
    for (int c = tid; c < ncell; c += blockDim.x) {
      const int cx = c % P, cy = (c / P) % P, cz = (DIM == 3) ? k0 + c / (P * P) : 0;
      const int ci = (DIM == 3) ? (((cz % CF::NRING) * P) + cy) * P + cx : cy * P + cx;
      if (!compute_cell<DIM, SP, P, QUAD>(X, cx, cy, cz, A.alpha, A.beta, cm, NC, ci)) s_bad = 1 + cx + P * (cy + P * cz);
    }
    __syncthreads();
    if (s_bad && tid == 0) report_error(A.err, 2, A.elem_begin + el, s_bad - 1);
    // rows of this chunk: per sub-lattice s the z range [k0, kend(s))
    int nrow_s[S], zlo[S];
    int nrows = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int ex = vkind<SP>(s, 0) ? P + 1 : P, ey = vkind<SP>(s, 1) ? P + 1 : P;
      int zl = 0, zh = 1;
      if (DIM == 3) {
        const bool vz = vkind<SP>(s, 2);
        zl = k0;
        zh = k1 + ((vz && k1 == P) ? 1 : 0);
      }
      zlo[s] = zl;
      nrow_s[s] = ex * ey * (zh - zl);
      nrows += nrow_s[s];
    }
    for (int r0 = 0; r0 < nrows; r0 += BATCH) {
      const int r = r0 + tid;
      if (r < nrows) {
        int s = 0, rr = r;
        while (rr >= nrow_s[s]) { rr -= nrow_s[s]; ++s; }
        const int ex = vkind<SP>(s, 0) ? P + 1 : P, ey = vkind<SP>(s, 1) ? P + 1 : P;
        int x[3];
        x[0] = rr % ex;
        x[1] = (rr / ex) % ey;
        x[2] = (DIM == 3) ? zlo[s] + rr / (ex * ey) : 0;
        const int tr = row_tau<DIM, SP>(P, s, x);
        const uint8_t fl = T.flags[tr], sf = E.sflags[tr];
        RowMeta M;
        M.len = 0;
        M.mode = 0;
        M.out = 0;
        const bool owned = fl & TF_OWNED;
        const bool rec = (sf & SF_SHARED) && (owned || (sf & SF_SEND));
        if (owned || rec) {
          const Blk &Br = blk[s * 27 + tr];
          const int gid = Br.g0 + Br.str[0] * x[0] + Br.str[1] * x[1] + Br.str[2] * x[2];
          double acc[W];
          int len = 0;
          const int lay0 = k0;
          switch (s) {
            case 0:
              row_values<DIM, SP, P, 0, NC>(cm, x, lay0, CF::NRING, acc);
              len = row_emit<DIM, SP, P, 0>(blk, blist, nb, T, x, Br.sigma, acc, p0 + tid, rg + tid, rv + tid, rm + tid);
              break;
            case 1:
              if (S > 1) {
                row_values<DIM, SP, P, (S > 1 ? 1 : 0), NC>(cm, x, lay0, CF::NRING, acc);
                len = row_emit<DIM, SP, P, (S > 1 ? 1 : 0)>(blk, blist, nb, T, x, Br.sigma, acc, p0 + tid, rg + tid,
                                                             rv + tid, rm + tid);
              }
              break;
            default:
              if (S > 2) {
                row_values<DIM, SP, P, (S > 2 ? 2 : 0), NC>(cm, x, lay0, CF::NRING, acc);
                len = row_emit<DIM, SP, P, (S > 2 ? 2 : 0)>(blk, blist, nb, T, x, Br.sigma, acc, p0 + tid, rg + tid,
                                                             rv + tid, rm + tid);
              }
              break;
          }
          M.len = len;
          if (!rec) {
            M.mode = 1;
            M.out = A.row_ptr[gid - A.row_begin];
          } else {
            M.mode = 2;
            int type, li;
            {
              const int c0 = cls_of(tr, 0), c1 = cls_of(tr, 1), c2 = DIM == 3 ? cls_of(tr, 2) : 1;
              const int nI = (c0 == 1) + (c1 == 1) + (DIM == 3 ? (c2 == 1) : 0);
              type = (nI == 0) ? 0 : (nI == DIM ? 3 : (DIM == 3 ? nI : 1));
              (void)li;
            }
            const int t_in = gid - A.base[type][T.ent[tr]];
            M.out = ((int64_t)E.rec[tr] + t_in) * A.rstride;
          }
        }
        meta[tid] = M;
      } else {
        RowMeta M;
        M.len = 0;
        M.mode = 0;
        M.out = 0;
        meta[tid] = M;
      }
      __syncthreads();
      // coalesced write-out: consecutive threads -> consecutive entries of consecutive rows
      for (int it = tid; it < BATCH * W; it += blockDim.x) {
        const int row = it / W, e = it - row * W;
        const RowMeta &M = meta[row];
        if (e >= M.len) continue;
        const int g = rg[e * BATCH + row];
        const double v = rv[e * BATCH + row];
        if (M.mode == 1) {
          A.col[M.out + e] = g;
          A.val[M.out + e] = v;
        } else if (M.mode == 2) {
          RecEntry R;
          R.col = g;
          R.meta = (int)rm[e * BATCH + row] | (M.len << 8);
          R.val = v;
          reinterpret_cast<double2 *>(A.scratch)[M.out + e] =
              make_double2(__longlong_as_double(((long long)(unsigned)R.meta << 32) | (unsigned)R.col), R.val);
        }
      }
      __syncthreads();
    }
  }
  // ---- arrival on shared owned entities; the last element to arrive merges their rows
  __threadfence();
  __syncthreads();
  if (tid < CF::NSLOT) {
    const int tau = tid;
    const uint8_t sf = E.sflags[tau];
    if ((sf & SF_SHARED) && !(sf & (SF_DEFER | SF_SEND)) && E.ose[tau] >= 0) {
      const int oi = E.ose[tau];
      const Ose O = A.ose[oi];
      const int old = atomicAdd(A.counters + oi, 1);
      if (old == O.k - 1) {
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
    for (int i = 0; i < nfin; ++i) {
      const Ose O = A.ose[s_fin[i]];
      finalize_ose(O, A.ose_slots, A.scratch, A.rstride, A.row_begin, A.row_ptr, A.col, A.val, smem + CF::OFF_CM,
                   CF::SMEM - CF::OFF_CM);
      __syncthreads();
    }
  }
}


// finalize_ose is defined (non-template) in lor_kernels.cu
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
