// lor_vec2d.cu -- 2D H(curl) Nedelec and H(div) Raviart-Thomas LOR matrices and the 2D discrete /
// rotated gradient ("grad-div problems in 2D ... rotated gradient", SURVEY 8(f)
// NEXT-2; numbering and signs: DESIGN.md reading P-29).  A 2D LOR cell carries 4 lattice-edge dofs,
// so the assembly uses the unstructured machinery of lor_legacy.cu generalised to signed 4-dof
// cells: per call the 4x4 cell matrices (vertex rule or Gauss-2, covariant / contravariant Piola,
// signs applied), then one warp per row ranks the <= 8 candidates of its <= 2 cells (count, scan,
// fill).  Setup: the LOR cells' signed dof lists and the dof -> (cell, local dof) transpose.
#include <cuda_runtime.h>
#include <stdint.h>

#include "lor_cells.cuh"
#include "lor_vec2d.h"

namespace lorb {

namespace {

// the cells' signed dof lists from the element restriction (local order: ND x-edges (b) -> b,
// y-edges (a) -> 2 + a; RT faces 2d + side, normal +e_d)
__global__ void k_v2_cells(int sp, int p, int64_t nel, const int32_t *__restrict__ emap, const int8_t *__restrict__ esgn,
                           int32_t *__restrict__ cmap, int8_t *__restrict__ csgn) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int ncpe = p * p, ndpe = 2 * p * (p + 1);
  if (t >= nel * ncpe * 4) return;
  const int i = (int)(t & 3);
  const int64_t cell = t >> 2, e = cell / ncpe;
  const int c = (int)(cell - e * ncpe), kx = c % p, ky = c / p;
  const int fam = i >> 1, off = i & 1;
  int x0 = kx, x1 = ky;
  if (sp == SP_ND) { if (fam == 0) x1 += off; else x0 += off; }
  else { if (fam == 0) x0 += off; else x1 += off; }
  const int ext0 = sp == SP_ND ? (fam == 0 ? p : p + 1) : (fam == 0 ? p + 1 : p);
  const int l = fam * p * (p + 1) + x0 + ext0 * x1;
  cmap[t] = emap[e * ndpe + l];
  csgn[t] = esgn[e * ndpe + l];
}

template <int SP, int QUAD>
__device__ __forceinline__ bool cell_vec2d(const double X[4][2], double alpha, double beta, const double *ca,
                                           const double *cb, double A[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) A[i] = 0.0;
  bool ok = true;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double t0 = QUAD == 0 ? (double)(q & 1) : gauss2_pt(q & 1), t1 = QUAD == 0 ? (double)(q >> 1) : gauss2_pt(q >> 1);
    // J[k][d] = d x_k / d t_d of the bilinear map
    double J[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int b0 = v & 1, b1 = v >> 1;
      const double f0 = b0 ? t0 : 1.0 - t0, f1 = b1 ? t1 : 1.0 - t1;
      const double g0 = (b0 ? 1.0 : -1.0) * f1, g1 = f0 * (b1 ? 1.0 : -1.0);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        J[k][0] += X[v][k] * g0;
        J[k][1] += X[v][k] * g1;
      }
    }
    const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    ok = ok && det > 0.0;
    const double w = 0.25, aq = alpha * coef_q<QUAD, 4>(ca, q), bq = beta * coef_q<QUAD, 4>(cb, q);
    double phi[4][2], s[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int fam = i >> 1, off = i & 1;
      double ph[2];
      double dv;
      if (SP == SP_ND) {  // (f(y), 0) / (0, f(x)); covariant Piola J^{-T}; curl = curl-hat / det
        const double tt = fam == 0 ? t1 : t0, f = off ? tt : 1.0 - tt, df = off ? 1.0 : -1.0;
        ph[fam] = f;
        ph[1 - fam] = 0.0;
        dv = fam == 0 ? -df : df;
        // J^{-T} = adj(J)^T / det: rows (J11, -J10), (-J01, J00)
        phi[i][0] = (J[1][1] * ph[0] - J[1][0] * ph[1]) / det;
        phi[i][1] = (-J[0][1] * ph[0] + J[0][0] * ph[1]) / det;
      } else {  // e_fam (off ? t_fam : 1 - t_fam); contravariant J phi-hat / det; div = div-hat / det
        const double tt = fam == 0 ? t0 : t1;
        ph[fam] = off ? tt : 1.0 - tt;
        ph[1 - fam] = 0.0;
        dv = off ? 1.0 : -1.0;
        phi[i][0] = (J[0][0] * ph[0] + J[0][1] * ph[1]) / det;
        phi[i][1] = (J[1][0] * ph[0] + J[1][1] * ph[1]) / det;
      }
      s[i] = dv / det;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        A[i * 4 + j] += w * (aq * s[i] * s[j] + bq * (phi[i][0] * phi[j][0] + phi[i][1] * phi[j][1])) * det;
  }
  return ok;
}

template <int SP, int QUAD>
__global__ void __launch_bounds__(128) k_v2_ea(V2Args a) {
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int ncpe = a.p * a.p, np1 = a.p + 1, npt = np1 * np1;
  if (cell >= a.ncell) return;
  const int64_t e = cell / ncpe;
  const int c = (int)(cell - e * ncpe), kx = c % a.p, ky = c / a.p;
  double X[4][2], ca8[4], cb8[4];
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const int l = (kx + (v & 1)) + np1 * (ky + (v >> 1));
    X[v][0] = a.X[e * a.xstride + l];
    X[v][1] = a.X[e * a.xstride + npt + l];
    if (a.ca) {
      ca8[v] = a.ca[e * npt + l];
      cb8[v] = a.cb[e * npt + l];
    }
  }
  double A[16];
  if (!cell_vec2d<SP, QUAD>(X, a.alpha, a.beta, a.ca ? ca8 : nullptr, a.ca ? cb8 : nullptr, A)) atomicExch(a.err, 1);
  double sg[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) sg[i] = (double)a.csgn[cell * 4 + i];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) a.ea[cell * 16 + i * 4 + j] = sg[i] * sg[j] * A[i * 4 + j];
}

// one warp per row: the (column, candidate) keys of its <= 2 cells ranked, count or fill
template <bool FILL>
__global__ void __launch_bounds__(256) k_v2_rows(V2Rows a) {
  __shared__ int64_t s_key[8][32];
  __shared__ double s_val[8][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + w;
  if (r >= a.n) return;
  const int64_t e0 = a.off[r];
  const int nc = (int)(a.off[r + 1] - e0) * 4;  // <= 32 candidates
  int64_t key = INT64_MAX;
  double val = 0.0;
  if (lane < nc) {
    const int32_t en = a.ent[e0 + lane / 4];
    const int64_t cell = en >> 2;
    const int i = en & 3, j = lane & 3;
    key = ((int64_t)a.cmap[cell * 4 + j] << 5) | lane;
    if (FILL) val = a.ea[cell * 16 + i * 4 + j];
  }
  s_key[w][lane] = key;
  __syncwarp();
  int rk = 0;
  for (int u = 0; u < nc; ++u) rk += s_key[w][u] < key;
  __syncwarp();
  if (lane < nc) {
    s_key[w][rk] = key;
    if (FILL) s_val[w][rk] = val;
  }
  __syncwarp();
  const bool head = lane < nc && (lane == 0 || (s_key[w][lane] >> 5) != (s_key[w][lane - 1] >> 5));
  const unsigned b = __ballot_sync(0xffffffffu, head);
  if (!FILL) {
    if (lane == 0) a.cnt[r] = __popc(b);
    return;
  }
  if (!head) return;
  const int k = __popc(b & ((1u << lane) - 1u));
  const int64_t col = s_key[w][lane] >> 5;
  double v = s_val[w][lane];
  for (int u = lane + 1; u < nc && (s_key[w][u] >> 5) == col; ++u) v += s_val[w][u];
  a.col[a.row_ptr[r] + k] = (int32_t)col;
  a.val[a.row_ptr[r] + k] = v;
}

// 2D discrete gradient (ND rows) / rotated gradient (RT rows): thread per (element, local dof),
// written by the element the setup marks as the row's writer (the minimal element containing it)
__global__ void k_v2_disc(V2Disc a) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int p = a.p, np1 = p + 1, ndpe = 2 * p * np1;
  if (t >= a.nel * ndpe || !a.writer[t]) return;
  const int64_t e = t / ndpe;
  const int l = (int)(t - e * ndpe), fam = l / (p * np1), rl = l - fam * p * np1;
  const int ext0 = a.sp == SP_ND ? (fam == 0 ? p : np1) : (fam == 0 ? np1 : p);
  const int x0 = rl % ext0, x1 = rl / ext0;
  int tx = x0, ty = x1, hx = x0, hy = x1;  // tail / head lattice points
  if (a.sp == SP_ND) { if (fam == 0) hx += 1; else hy += 1; }        // edge along fam, +axis
  else if (fam == 1) { hx += 1; }                                      // RT normal y: tau = +e_x
  else { ty += 1; }                                                    // RT normal x: tau = -e_y
  const int32_t row = a.rmap[t];
  const double sr = (double)a.rsgn[t];
  int32_t c0 = a.hmap[e * np1 * np1 + tx + np1 * ty], c1 = a.hmap[e * np1 * np1 + hx + np1 * hy];
  double v0 = -sr, v1 = sr;
  if (c1 < c0) {
    const int32_t tc = c0; c0 = c1; c1 = tc;
    const double tv = v0; v0 = v1; v1 = tv;
  }
  const int64_t o = 2 * (int64_t)(row - a.row_begin);
  a.col[o] = c0;
  a.col[o + 1] = c1;
  a.val[o] = v0;
  a.val[o + 1] = v1;
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t > 0 ? (n + t - 1) / t : 1); }

}  // namespace

cudaError_t launch_v2_cells(int sp, int p, int64_t nel, const int32_t *emap, const int8_t *esgn, int32_t *cmap,
                            int8_t *csgn, cudaStream_t st) {
  const int64_t n = nel * p * p * 4;
  if (n > 0) k_v2_cells<<<nblk(n, 256), 256, 0, st>>>(sp, p, nel, emap, esgn, cmap, csgn);
  return cudaGetLastError();
}
cudaError_t launch_v2_ea(int sp, int quad, const V2Args &a, cudaStream_t st) {
  if (a.ncell <= 0) return cudaSuccess;
  const unsigned g = nblk(a.ncell, 128);
  if (sp == SP_ND) {
    if (quad == 0) k_v2_ea<SP_ND, 0><<<g, 128, 0, st>>>(a);
    else k_v2_ea<SP_ND, 1><<<g, 128, 0, st>>>(a);
  } else {
    if (quad == 0) k_v2_ea<SP_RT, 0><<<g, 128, 0, st>>>(a);
    else k_v2_ea<SP_RT, 1><<<g, 128, 0, st>>>(a);
  }
  return cudaGetLastError();
}
cudaError_t launch_v2_rows(const V2Rows &a, bool fill, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  if (fill) k_v2_rows<true><<<nblk(a.n, 8), 256, 0, st>>>(a);
  else k_v2_rows<false><<<nblk(a.n, 8), 256, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_v2_disc(const V2Disc &a, cudaStream_t st) {
  const int64_t n = a.nel * 2 * a.p * (a.p + 1);
  if (n > 0) k_v2_disc<<<nblk(n, 256), 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace lorb
