// lor_legacy.cu -- the fully unstructured ("legacy") LOR assembly the paper compares the macro-element
// method against: the LOR mesh is treated as an arbitrary
// low-order hex mesh -- explicit LOR element restriction (8 global H1 ids per LOR cell), LOR
// coordinate E-vector in broken (per-cell, duplicated) format, dof -> (cell, corner) transpose -- and
// every call "constructs small dense matrices for each element of the low-order-refined mesh, and
// then directly assembles the global sparse matrix" (l.597-598) with no use of the macro-element
// structure:
//   k_leg_mesh   setup: LOR element restriction + broken LOR coordinates from the HO E-vector and the
//                H1 element restriction (the overhead l.604-606 says "can dominate").
//   k_leg_ea     per call: one thread per LOR cell, the dense 8x8 Q1 matrix (vertex rule, the same
//                sub-cell math as the macro path) staged in shared memory, written coalesced.
//   k_leg_rows   per call, twice (count, then fill): one warp per row gathers the 8 x 8 candidate
//                (column, value) pairs of the <= 8 cells containing the row through the transpose,
//                ranks them by (column, candidate index) in shared memory, and counts / writes the
//                distinct columns in ascending order with the duplicates summed in candidate order.
// H1, 3D, vertex rule.  The comparator of lor_legacy_*; at p = 1 (a macro-element is one LOR cell)
// also the product path of lor_assemble_h1 on one rank (lor_fill_path 2).
#include <cuda_runtime.h>
#include <stdint.h>

#include "lor_cells.cuh"
#include "lor_legacy.h"

namespace lorb {

namespace {

__global__ void k_leg_mesh(int p, int64_t nel, const int32_t *__restrict__ emap, const double *__restrict__ X,
                           int64_t xstride, int32_t *__restrict__ lmap, double *__restrict__ lx) {
  const int np1 = p + 1, npts = np1 * np1 * np1, ncpe = p * p * p;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nel * ncpe * 8) return;
  const int q = (int)(t & 7);
  const int64_t cell = t >> 3, e = cell / ncpe;
  const int c = (int)(cell - e * ncpe);
  const int cx = c % p, cy = (c / p) % p, cz = c / (p * p);
  const int l = (cx + (q & 1)) + np1 * ((cy + ((q >> 1) & 1)) + np1 * (cz + ((q >> 2) & 1)));
  lmap[t] = emap[e * npts + l];
#pragma unroll
  for (int d = 0; d < 3; ++d) lx[cell * 24 + d * 8 + q] = X[e * xstride + d * npts + l];
}

constexpr int EA_T = 64;  // cells per block of k_leg_ea

__global__ void __launch_bounds__(EA_T) k_leg_ea(int64_t ncell, int ncpe, const double *__restrict__ lx, double alpha,
                                                  double beta, double *__restrict__ ea, int *err) {
  __shared__ double s[EA_T * 64];
  const int64_t c0 = (int64_t)blockIdx.x * EA_T;
  const int64_t cell = c0 + threadIdx.x;
  if (cell < ncell) {
    double C[8][3];
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int d = 0; d < 3; ++d) C[q][d] = lx[cell * 24 + d * 8 + q];
    double A[36];
    if (!cell_h1_3d<0>(C, alpha, beta, A) && atomicCAS(err, 0, 1) == 0) {  // (element, cell) as lor_sync reports
      err[1] = (int)(cell / ncpe);
      err[2] = (int)(cell % ncpe);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) s[threadIdx.x * 64 + i * 8 + j] = A[i <= j ? tri(8, i, j) : tri(8, j, i)];
  }
  __syncthreads();
  const int64_t nv = (ncell - c0 < EA_T ? ncell - c0 : EA_T) * 64;
  for (int64_t k = threadIdx.x; k < nv; k += EA_T) ea[c0 * 64 + k] = s[k];
}

// one warp per row; FILL = false: row lengths, true: columns + values
template <bool FILL>
__global__ void __launch_bounds__(256) k_leg_rows(LegArgs a) {
  __shared__ int64_t s_key[8][64];
  __shared__ double s_val[8][64];
  __shared__ int s_pos[8][64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * 8 + w);
  if (r >= a.n) return;
  const int64_t e0 = a.off[r], ne = a.off[r + 1] - e0;
  const int nc = (int)(ne * 8);  // candidates (<= 64: a hex vertex lies in <= 8 cells)
  int64_t key[2];
  double val[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int t = lane + 32 * h;
    key[h] = INT64_MAX;
    val[h] = 0.0;
    if (t < nc) {
      const int32_t en = a.ent[e0 + t / 8];
      const int64_t cell = en >> 3;
      const int i = en & 7, j = t & 7;
      key[h] = ((int64_t)a.lmap[cell * 8 + j] << 6) | t;  // (column, candidate index): a strict order
      if (FILL) val[h] = a.ea[cell * 64 + i * 8 + j];
    }
    s_key[w][t] = key[h];
  }
  __syncwarp();
  // rank of each candidate in the sorted order, scatter to it
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    int rk = 0;
    for (int u = 0; u < nc; ++u) rk += s_key[w][u] < key[h];
    const int t = lane + 32 * h;
    if (t < nc) s_pos[w][t] = rk;
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int t = lane + 32 * h;
    if (t < nc) {
      s_key[w][s_pos[w][t]] = key[h];  // every rank is written once (keys are distinct)
      if (FILL) s_val[w][s_pos[w][t]] = val[h];
    }
  }
  __syncwarp();
  // run heads of equal columns in sorted order
  bool head[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int t = lane + 32 * h;
    head[h] = t < nc && (t == 0 || (s_key[w][t] >> 6) != (s_key[w][t - 1] >> 6));
  }
  const unsigned b0 = __ballot_sync(0xffffffffu, head[0]), b1 = __ballot_sync(0xffffffffu, head[1]);
  if (!FILL) {
    if (lane == 0) a.cnt[r] = __popc(b0) + __popc(b1);
    return;
  }
  const int64_t o = a.row_ptr[r];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (!head[h]) continue;
    const int t = lane + 32 * h;
    const int k = h == 0 ? __popc(b0 & ((1u << lane) - 1u)) : __popc(b0) + __popc(b1 & ((1u << lane) - 1u));
    const int64_t col = s_key[w][t] >> 6;
    double v = s_val[w][t];
    for (int u = t + 1; u < nc && (s_key[w][u] >> 6) == col; ++u) v += s_val[w][u];
    a.col[o + k] = (int32_t)col;
    a.val[o + k] = v;
  }
}

// ---- p = 1 vector spaces (fill path 2 of lor_assemble_nd / _rt): the element is the LOR cell, its
// element-local dofs are the cell-local ones (ND edge eps = 4a + b1 + 2 b2, RT face 2a + side: the
// App. A.3 family-major lattice order at p = 1), the element restriction and orientation signs are
// the space's own (emap / esgn).
template <int SP>
struct RvK {
  static constexpr int K = SP == 1 ? 12 : 6;  // dofs per cell
  static constexpr int KP = K * (K + 1) / 2;   // packed triangle
  static constexpr int T = SP == 1 ? 32 : 64;  // cells per block of k_rv_ea (staging <= 20 KB)
};

template <int SP>
__global__ void __launch_bounds__(RvK<SP>::T) k_rv_ea(int64_t ncell, const double *__restrict__ X, int64_t xstride,
                                                     double alpha, double beta, double *__restrict__ ea, int *err) {
  constexpr int KP = RvK<SP>::KP, T = RvK<SP>::T;
  __shared__ double s[T * KP];
  const int64_t c0 = (int64_t)blockIdx.x * T;
  const int64_t cell = c0 + threadIdx.x;
  if (cell < ncell) {
    double C[8][3];
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int d = 0; d < 3; ++d) C[q][d] = X[cell * xstride + d * 8 + q];  // p = 1: lattice point = corner q
    double A[KP];
    bool ok;
    if (SP == 1) ok = cell_nd<0>(C, alpha, beta, A);
    else ok = cell_rt<0>(C, alpha, beta, A);
    if (!ok && atomicCAS(err, 0, 1) == 0) {
      err[1] = (int)cell;
      err[2] = 0;
    }
#pragma unroll
    for (int k = 0; k < KP; ++k) s[threadIdx.x * KP + k] = A[k];
  }
  __syncthreads();
  const int64_t nv = (ncell - c0 < T ? ncell - c0 : T) * KP;
  for (int64_t k = threadIdx.x; k < nv; k += T) ea[c0 * KP + k] = s[k];
}

// one warp per row over its <= 4 (ND) / 2 (RT) cells: candidates (column, candidate index) ranked
// as in k_leg_rows, values s_i s_j A_ij
template <int SP, bool FILL>
__global__ void __launch_bounds__(256) k_rv_rows(RvArgs a) {
  constexpr int K = RvK<SP>::K, KP = RvK<SP>::KP;
  __shared__ int64_t s_key[8][64];
  __shared__ double s_val[8][64];
  __shared__ int s_pos[8][64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * 8 + w);
  if (r >= a.n) return;
  const int64_t e0 = a.off[r], ne = a.off[r + 1] - e0;
  const int nc = (int)(ne * K);
  if (nc > 64) {  // not a conforming hex mesh (an edge in more than 5 cells)
    if (lane == 0) atomicCAS(a.err, 0, 3);
    return;
  }
  int64_t key[2];
  double val[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int t = lane + 32 * h;
    key[h] = INT64_MAX;
    val[h] = 0.0;
    if (t < nc) {
      const int32_t en = a.ent[e0 + t / K];
      const int64_t cell = en / K;
      const int i = en - (int)cell * K, j = t % K;
      key[h] = ((int64_t)a.map[cell * K + j] << 6) | t;
      if (FILL) {
        const double v = a.ea[cell * KP + (i <= j ? tri(K, i, j) : tri(K, j, i))];
        val[h] = (a.sgn[cell * K + i] * a.sgn[cell * K + j]) > 0 ? v : -v;
      }
    }
    s_key[w][t] = key[h];
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    int rk = 0;
    for (int u = 0; u < nc; ++u) rk += s_key[w][u] < key[h];
    const int t = lane + 32 * h;
    if (t < nc) s_pos[w][t] = rk;
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int t = lane + 32 * h;
    if (t < nc) {
      s_key[w][s_pos[w][t]] = key[h];
      if (FILL) s_val[w][s_pos[w][t]] = val[h];
    }
  }
  __syncwarp();
  bool head[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int t = lane + 32 * h;
    head[h] = t < nc && (t == 0 || (s_key[w][t] >> 6) != (s_key[w][t - 1] >> 6));
  }
  const unsigned b0 = __ballot_sync(0xffffffffu, head[0]), b1 = __ballot_sync(0xffffffffu, head[1]);
  if (!FILL) {
    if (lane == 0) a.cnt[r] = __popc(b0) + __popc(b1);
    return;
  }
  const int64_t o = a.row_ptr[r];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (!head[h]) continue;
    const int t = lane + 32 * h;
    const int k = h == 0 ? __popc(b0 & ((1u << lane) - 1u)) : __popc(b0) + __popc(b1 & ((1u << lane) - 1u));
    const int64_t col = s_key[w][t] >> 6;
    double v = s_val[w][t];
    for (int u = t + 1; u < nc && (s_key[w][u] >> 6) == col; ++u) v += s_val[w][u];
    a.col[o + k] = (int32_t)col;
    a.val[o + k] = v;
  }
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t > 0 ? (n + t - 1) / t : 1); }

}  // namespace

cudaError_t launch_leg_mesh(int p, int64_t nel, const int32_t *emap, const double *X, int64_t xstride, int32_t *lmap,
                            double *lx, cudaStream_t st) {
  const int64_t n = nel * (int64_t)p * p * p * 8;
  if (n > 0) k_leg_mesh<<<nblk(n, 256), 256, 0, st>>>(p, nel, emap, X, xstride, lmap, lx);
  return cudaGetLastError();
}
cudaError_t launch_leg_ea(int64_t ncell, int ncpe, const double *lx, double alpha, double beta, double *ea, int *err,
                          cudaStream_t st) {
  if (ncell > 0) k_leg_ea<<<nblk(ncell, EA_T), EA_T, 0, st>>>(ncell, ncpe, lx, alpha, beta, ea, err);
  return cudaGetLastError();
}
cudaError_t launch_leg_rows(const LegArgs &a, bool fill, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  if (fill) k_leg_rows<true><<<nblk(a.n, 8), 256, 0, st>>>(a);
  else k_leg_rows<false><<<nblk(a.n, 8), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_rv_ea(int sp, int64_t ncell, const double *X, int64_t xstride, double alpha, double beta, double *ea,
                         int *err, cudaStream_t st) {
  if (ncell <= 0) return cudaSuccess;
  if (sp == 1) k_rv_ea<1><<<nblk(ncell, RvK<1>::T), RvK<1>::T, 0, st>>>(ncell, X, xstride, alpha, beta, ea, err);
  else k_rv_ea<2><<<nblk(ncell, RvK<2>::T), RvK<2>::T, 0, st>>>(ncell, X, xstride, alpha, beta, ea, err);
  return cudaGetLastError();
}
cudaError_t launch_rv_rows(int sp, const RvArgs &a, bool fill, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  const unsigned g = nblk(a.n, 8);
  if (sp == 1) {
    if (fill) k_rv_rows<1, true><<<g, 256, 0, st>>>(a);
    else k_rv_rows<1, false><<<g, 256, 0, st>>>(a);
  } else {
    if (fill) k_rv_rows<2, true><<<g, 256, 0, st>>>(a);
    else k_rv_rows<2, false><<<g, 256, 0, st>>>(a);
  }
  return cudaGetLastError();
}
int rv_dofs_per_cell(int sp) { return sp == 1 ? 12 : 6; }
int64_t rv_ea_words(int sp) { return sp == 1 ? 78 : 21; }

}  // namespace lorb
