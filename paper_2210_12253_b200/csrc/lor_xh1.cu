// lor_xh1.cu -- extended-frame H1 fill (3D, vertex rule): one CTA per macro element writes the
// complete CSR rows of every dof the element owns (the minimal macro element
// containing a nonzero writes it), shared rows included, in one pass.  See lor_xframe.h.
//
//   prologue  element record, extended box table, coordinates of the element (its E-vector,
//             PAPER.md l.342-345) and of the neighbour points one lattice layer around it, read in
//             the element's own frame; global id of every extended lattice point (affine per box);
//   cells     per z-chunk, the packed 8x8 vertex-rule cell matrices (36 doubles, corner-parallel:
//             eight lanes per cell) of every LOR cell of the cell box -- the element's
//             own p^3 cells plus the neighbour cells touching its owned rows;
//   rows      one thread per owned row: values from the <= 8 cells containing the row (registers),
//             columns = global ids of the 27 stencil points, each stored at its final position in
//             the row (setup position table: ascending global column order, reading P-5).
#include <cuda_runtime.h>
#include <stdint.h>

#include "lor_device.cuh"
#include "lor_xframe.h"

namespace lorb {

namespace {

__device__ __forceinline__ int ycls(int y, int p) { return y < 0 ? 0 : (y == 0 ? 1 : (y < p ? 2 : (y == p ? 3 : 4))); }
__device__ __forceinline__ int ydelta(int y, int p) { return y < 0 ? -1 : (y > p ? 1 : 0); }
__device__ __forceinline__ int lcls(int l, int p) { return l == 0 ? 0 : (l == p ? 2 : 1); }

// neighbour-local lattice coordinates of extended-frame point y (lor_xframe.h XNbr::code)
__device__ __forceinline__ void x_to_local(int p, uint32_t code, const int y[3], int L[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int k = (code >> (2 * a)) & 3;
    const int ok = (int)((code >> (9 + 2 * k)) & 3) - 1;
    const int v = y[k] - p * ok;
    L[a] = ((code >> (6 + a)) & 1) ? -v : v;
  }
}

__device__ __forceinline__ void xreport(int *err, int code, int64_t e, int cell) {
  if (atomicCAS(err, 0, code) == 0) {
    err[1] = (int)e;
    err[2] = cell;
  }
}

__device__ __forceinline__ void cross3x(const double *a, const double *b, double *c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}
__device__ __forceinline__ double dot3x(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

}  // namespace

// ============================================================================== setup kernel
// Box table of every element (125 boxes of the extended frame) and the position table of every
// owned row: final position of each of the 27 stencil slots in the ascending-column CSR row.
template <int P>
__global__ void __launch_bounds__(128) k_xh1_setup(XSetupArgs A) {
  const int64_t e = blockIdx.x;
  if (e >= A.nel_local) return;
  __shared__ XElem H;
  __shared__ XBox B[125];
  {
    const int4 *src = reinterpret_cast<const int4 *>(A.xe + e);
    int4 *dst = reinterpret_cast<int4 *>(&H);
    for (int i = threadIdx.x; i < (int)(sizeof(XElem) / 16); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 125; b += blockDim.x) {
    const int cb[3] = {b % 5, (b / 5) % 5, b / 25};
    XBox bx;
    bx.g0 = 0;
    bx.s[0] = bx.s[1] = bx.s[2] = 0;
    bx.valid = 0;
    bool ok = true;
    int y[3];
    for (int a = 0; a < 3; ++a) {
      y[a] = cb[a] == 0 ? -1 : (cb[a] == 1 ? 0 : (cb[a] == 2 ? 1 : (cb[a] == 3 ? P : P + 1)));
      if (cb[a] == 2 && P < 2) ok = false;
    }
    const int ni = (ydelta(y[0], P) + 1) + 3 * (ydelta(y[1], P) + 1) + 9 * (ydelta(y[2], P) + 1);
    int64_t f = e;
    uint32_t code = 0 | (1u << 2) | (2u << 4) | (1u << 9) | (1u << 11) | (1u << 13);  // identity
    if (ni != 13) {
      f = H.nbr[ni].el;
      code = H.nbr[ni].code;
      if (f < 0) ok = false;
    }
    if (ok) {
      int L[3];
      x_to_local(P, code, y, L);
      const int tau = lcls(L[0], P) + 3 * lcls(L[1], P) + 9 * lcls(L[2], P);
      Blk Bk;
      block_affine<3, SP_H1>(P, 0, tau, A.topo[f], A.base, Bk);
      if (Bk.size > 0) {
        // gid = g0 + sum_a str_a L_a,  L_a = sn_a (y[ax_a] - P o[ax_a])
        int g0 = Bk.g0;
        int s[3] = {0, 0, 0};
        for (int a = 0; a < 3; ++a) {
          const int k = (code >> (2 * a)) & 3;
          const int ok2 = (int)((code >> (9 + 2 * k)) & 3) - 1;
          const int sn = ((code >> (6 + a)) & 1) ? -1 : 1;
          s[k] = Bk.str[a] * sn;
          g0 -= Bk.str[a] * sn * P * ok2;
        }
        bx.g0 = g0;
        for (int k = 0; k < 3; ++k) bx.s[k] = (int8_t)s[k];
        bx.valid = 1;
      }
    }
    B[b] = bx;
    A.box[e * 125 + b] = bx;
  }
  __syncthreads();
  auto gid = [&](const int y[3], bool &okg) -> int {
    const XBox &bx = B[ycls(y[0], P) + 5 * ycls(y[1], P) + 25 * ycls(y[2], P)];
    okg = okg && bx.valid;
    return bx.g0 + bx.s[0] * y[0] + bx.s[1] * y[1] + bx.s[2] * y[2];
  };
  constexpr int NP1 = P + 1;
  for (int l = threadIdx.x; l < NP1 * NP1 * NP1; l += blockDim.x) {
    const int x[3] = {l % NP1, (l / NP1) % NP1, l / (NP1 * NP1)};
    const int tau = lcls(x[0], P) + 3 * lcls(x[1], P) + 9 * lcls(x[2], P);
    if (!((H.own >> tau) & 1)) continue;
    bool okg = true;
    const int g = gid(x, okg);
    int ids[27];
    int nvalid = 0;
    for (int j = 0; j < 27; ++j) {
      const int y[3] = {x[0] + j % 3 - 1, x[1] + (j / 3) % 3 - 1, x[2] + j / 9 - 1};
      bool v = true;
      for (int a = 0; a < 3; ++a) {
        int lo = (x[a] > y[a] ? x[a] : y[a]) - 1, hi = x[a] < y[a] ? x[a] : y[a];
        lo = lo < H.clo[a] ? H.clo[a] : lo;
        hi = hi > H.chi[a] ? H.chi[a] : hi;
        v = v && lo <= hi;
      }
      ids[j] = v ? gid(y, okg) : -1;
      nvalid += v;
    }
    const int64_t r = (int64_t)g - A.row_begin;
    if (!okg || r < 0 || A.cnt[r] != nvalid) {
      atomicExch(A.err, 1);
      continue;
    }
    uint32_t w[XPOS_W / 4];
    for (int i = 0; i < XPOS_W / 4; ++i) w[i] = 0xffffffffu;
    for (int j = 0; j < 27; ++j) {
      if (ids[j] < 0) continue;
      int rk = 0;
      for (int k = 0; k < 27; ++k) {
        if (ids[k] >= 0 && ids[k] < ids[j]) ++rk;
        if (k != j && ids[k] == ids[j]) atomicExch(A.err, 1);
      }
      w[j >> 2] = (w[j >> 2] & ~(0xffu << (8 * (j & 3)))) | ((uint32_t)rk << (8 * (j & 3)));
    }
    uint4 *dst = reinterpret_cast<uint4 *>(A.pos + r * XPOS_W);
    dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
    dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
}

// ============================================================================== fill kernel
struct XLayout {
  int npb;   // points in the (max) point box
  int ncp;   // cell-matrix pitch (odd)
  int nr;    // ring layers
  int off_xg, off_cm, bytes;
};

__host__ __device__ inline XLayout xh1_layout(int ncx, int ncy, int ncz, int kz) {
  XLayout L;
  L.npb = (ncx + 1) * (ncy + 1) * (ncz + 1);
  L.nr = kz + 1 < ncz ? kz + 1 : ncz;
  L.ncp = (L.nr * ncx * ncy) | 1;
  L.off_xg = 3 * L.npb * 8;
  L.off_cm = (L.off_xg + L.npb * 4 + 15) / 16 * 16;
  L.bytes = L.off_cm + 36 * L.ncp * 8;
  return L;
}

template <int P>
__global__ void __launch_bounds__(128, 3) k_xh1_fill(XFillArgs A, int kz) {
  constexpr int NP1 = P + 1, NPT = NP1 * NP1 * NP1;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ XElem H;
  __shared__ XBox B[125];
  __shared__ int s_bad;
  const XLayout LY = xh1_layout(A.ncx, A.ncy, A.ncz, kz);
  double *XE = reinterpret_cast<double *>(smem);
  int32_t *XG = reinterpret_cast<int32_t *>(smem + LY.off_xg);
  double *cm = reinterpret_cast<double *>(smem + LY.off_cm);
  const int tid = threadIdx.x;
  if ((int64_t)blockIdx.x >= A.nel_local) return;
  const int64_t el = A.order ? A.order[blockIdx.x] : blockIdx.x;
  {
    const int4 *src = reinterpret_cast<const int4 *>(A.xe + el);
    int4 *dst = reinterpret_cast<int4 *>(&H);
    for (int i = tid; i < (int)(sizeof(XElem) / 16); i += blockDim.x) dst[i] = __ldg(src + i);
    const uint2 *bs = reinterpret_cast<const uint2 *>(A.box + el * 125);
    uint2 *bd = reinterpret_cast<uint2 *>(B);
    for (int i = tid; i < 125; i += blockDim.x) bd[i] = __ldg(bs + i);
    if (tid == 0) s_bad = 0;
  }
  __syncthreads();
  const int clo0 = H.clo[0], clo1 = H.clo[1], clo2 = H.clo[2];
  const int nx = H.chi[0] - clo0 + 1, ny = H.chi[1] - clo1 + 1, nz = H.chi[2] - clo2 + 1;
  const int npx = nx + 1, npy = ny + 1, npz = nz + 1;
  const int npb = npx * npy * npz;
  // point box origin = clo; index of point y: (y0-clo0) + npx ((y1-clo1) + npy (y2-clo2))
  {
    // own E-vector (contiguous, 16-byte vector loads) scattered into the point box
    const double2 *xs = reinterpret_cast<const double2 *>(A.X + el * A.xstride);
    constexpr int NX2 = (3 * NPT + 1) / 2;
    for (int i = tid; i < NX2; i += blockDim.x) {
      const double2 v = __ldg(xs + i);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int q = 2 * i + h;
        if (q < 3 * NPT) {
          const int d = q / NPT, l = q - d * NPT;
          const int x0 = l % NP1, x1 = (l / NP1) % NP1, x2 = l / (NP1 * NP1);
          XE[d * LY.npb + (x0 - clo0) + npx * ((x1 - clo1) + npy * (x2 - clo2))] = h ? v.y : v.x;
        }
      }
    }
    // neighbour points of the point box (read in the element's frame) and every point's gid
    for (int i = tid; i < npb; i += blockDim.x) {
      const int y[3] = {clo0 + i % npx, clo1 + (i / npx) % npy, clo2 + i / (npx * npy)};
      const XBox bx = B[ycls(y[0], P) + 5 * ycls(y[1], P) + 25 * ycls(y[2], P)];
      XG[i] = bx.g0 + bx.s[0] * y[0] + bx.s[1] * y[1] + bx.s[2] * y[2];
      const int ni = (ydelta(y[0], P) + 1) + 3 * (ydelta(y[1], P) + 1) + 9 * (ydelta(y[2], P) + 1);
      if (ni == 13) continue;
      const XNbr nb = H.nbr[ni];
      int L[3];
      x_to_local(P, nb.code, y, L);
      const double *src = A.X + (int64_t)nb.el * A.xstride + L[0] + NP1 * (L[1] + NP1 * L[2]);
      XE[i] = __ldg(src);
      XE[LY.npb + i] = __ldg(src + NPT);
      XE[2 * LY.npb + i] = __ldg(src + 2 * NPT);
    }
  }
  __syncthreads();
  // owned-row box
  int olo[3], ohi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    bool c0 = false, c1 = false, c2 = false;
    for (int tau = 0; tau < 27; ++tau) {
      if (!((H.own >> tau) & 1)) continue;
      const int c = a == 0 ? tau % 3 : (a == 1 ? (tau / 3) % 3 : tau / 9);
      c0 |= c == 0;
      c1 |= c == 1;
      c2 |= c == 2;
    }
    olo[a] = c0 ? 0 : (c1 ? 1 : P);
    ohi[a] = c2 ? P : (c1 ? P - 1 : 0);
  }
  const int NR = LY.nr, NCP = LY.ncp, lay = nx * ny;
  const double alpha = A.alpha, beta = A.beta;
  const int nchunk = (nz + kz - 1) / kz;
  for (int ch = 0; ch < nchunk; ++ch) {
    const int cz0 = clo2 + ch * kz;
    const int cz1 = (cz0 + kz - 1 < H.chi[2]) ? cz0 + kz - 1 : H.chi[2];
    if (ch > 0) __syncthreads();  // rows of the previous chunk done with the ring slots
    // ---- cells of layers [cz0, cz1]: eight lanes per cell, one corner each
    {
      const int ncell = (cz1 - cz0 + 1) * lay;
      const int items = ncell * 8;
      const int ceil32 = (items + 31) / 32 * 32;
      int bad = 0;
      for (int it = tid; it < ceil32; it += blockDim.x) {
        const bool act = it < items;
        const int c = act ? it >> 3 : 0, q = it & 7;
        const int ux = c % nx, uy = (c / nx) % ny, uz = c / lay;  // cell offsets in the box / chunk
        const int cz = cz0 + uz;
        const int pb = ux + npx * (uy + npy * (cz - clo2));
        auto pt = [&](int v, int d) -> double {
          return XE[d * LY.npb + pb + (v & 1) + npx * (((v >> 1) & 1) + npy * ((v >> 2) & 1))];
        };
        double j[3][3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const int hi = q | (1 << d), lo = q & ~(1 << d);
#pragma unroll
          for (int k = 0; k < 3; ++k) j[d][k] = pt(hi, k) - pt(lo, k);
        }
        double r[3][3];
        cross3x(j[1], j[2], r[0]);
        cross3x(j[2], j[0], r[1]);
        cross3x(j[0], j[1], r[2]);
        const double det = dot3x(j[0], r[0]);
        const int cx = clo0 + ux, cy = clo1 + uy;
        if (act && !(det > 0.0) && cx >= 0 && cx < P && cy >= 0 && cy < P && cz >= 0 && cz < P)
          bad = 1 + cx + P * (cy + P * cz);
        const double sa = 0.125 * alpha / det;
        double Q[3][3];
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int e2 = d; e2 < 3; ++e2) Q[d][e2] = Q[e2][d] = sa * dot3x(r[d], r[e2]);
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
          const double ev = -sg[d] * Qs[d];
          edge[d] = ev + __shfl_xor_sync(0xffffffffu, ev, 1 << d);
        }
        {
          const double f01 = sg[0] * sg[1] * Q[0][1], f02 = sg[0] * sg[2] * Q[0][2], f12 = sg[1] * sg[2] * Q[1][2];
          fdg[0] = f01 + __shfl_xor_sync(0xffffffffu, f01, 3);
          fdg[1] = f02 + __shfl_xor_sync(0xffffffffu, f02, 5);
          fdg[2] = f12 + __shfl_xor_sync(0xffffffffu, f12, 6);
        }
        if (act) {
          const int ci = ((cz - clo2) % NR) * lay + uy * nx + ux;
          double *o = cm + ci;
          const int rq = (q * (15 - q)) >> 1;
          o[(rq + q) * NCP] = diag;
#pragma unroll
          for (int d = 0; d < 3; ++d)
            if (!((q >> d) & 1)) o[(rq + (q | (1 << d))) * NCP] = edge[d];
          auto tp = [](int a, int b) { const int i = a < b ? a : b, jj = a < b ? b : a; return ((i * (15 - i)) >> 1) + jj; };
          if (q < (q ^ 3)) o[tp(q ^ 1, q ^ 2) * NCP] = fdg[0];
          if (q < (q ^ 5)) o[tp(q ^ 1, q ^ 4) * NCP] = fdg[1];
          if (q < (q ^ 6)) o[tp(q ^ 2, q ^ 4) * NCP] = fdg[2];
          if (q < 4) o[(rq + (q ^ 7)) * NCP] = 0.0;
        }
      }
      if (bad) s_bad = bad;
    }
    __syncthreads();
    if (s_bad && tid == 0) xreport(A.err, 2, A.elem_begin + el, s_bad - 1);
    // ---- rows of layers [cz0, cz1] (+ cz1 + 1 after the last cell layer), owned only
    int rz0 = cz0, rz1 = (ch == nchunk - 1) ? cz1 + 1 : cz1;
    rz0 = rz0 < olo[2] ? olo[2] : rz0;
    rz1 = rz1 > ohi[2] ? ohi[2] : rz1;
    const int rnx = ohi[0] - olo[0] + 1, rny = ohi[1] - olo[1] + 1;
    const int nrow = (rz1 >= rz0) ? rnx * rny * (rz1 - rz0 + 1) : 0;
    for (int ri = tid; ri < nrow; ri += blockDim.x) {
      const int x[3] = {olo[0] + ri % rnx, olo[1] + (ri / rnx) % rny, rz0 + ri / (rnx * rny)};
      const int tau = lcls(x[0], P) + 3 * lcls(x[1], P) + 9 * lcls(x[2], P);
      if (!((H.own >> tau) & 1)) continue;
      const int px = (x[0] - clo0) + npx * ((x[1] - clo1) + npy * (x[2] - clo2));
      const int g = XG[px];
      const int64_t r = (int64_t)g - A.row_begin;
      const int64_t out = __ldg(A.row_ptr + r);
      const uint4 *pp = reinterpret_cast<const uint4 *>(A.pos + r * XPOS_W);
      const uint4 pa = __ldcs(pp), pbv = __ldcs(pp + 1);
      const uint32_t pw[8] = {pa.x, pa.y, pa.z, pa.w, pbv.x, pbv.y, pbv.z, pbv.w};
      double acc[27];
#pragma unroll
      for (int j = 0; j < 27; ++j) acc[j] = 0.0;
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        const int ox = o & 1, oy = (o >> 1) & 1, oz = (o >> 2) & 1;
        const int cx = x[0] - ox, cy = x[1] - oy, cz = x[2] - oz;
        if (cx < clo0 || cx > H.chi[0] || cy < clo1 || cy > H.chi[1] || cz < clo2 || cz > H.chi[2]) continue;
        const int ci = ((cz - clo2) % NR) * lay + (cy - clo1) * nx + (cx - clo0);
#pragma unroll
        for (int jc = 0; jc < 8; ++jc) {
          const int dx = (jc & 1) - ox, dy = ((jc >> 1) & 1) - oy, dz = ((jc >> 2) & 1) - oz;
          acc[(dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)] += cm[tri(8, o, jc) * NCP + ci];
        }
      }
#pragma unroll
      for (int j = 0; j < 27; ++j) {
        const int ps = (int)((pw[j >> 2] >> (8 * (j & 3))) & 255u);
        if (ps != 255) {
          const int dj = (j % 3 - 1) + npx * (((j / 3) % 3 - 1) + npy * (j / 9 - 1));
          __stcs(A.col + out + ps, XG[px + dj]);
          __stcs(A.val + out + ps, acc[j]);
        }
      }
    }
  }
}

// ============================================================================== launchers
template <int P>
static cudaError_t xh1_setup_p(const XSetupArgs &a, cudaStream_t st) {
  if (a.nel_local <= 0) return cudaSuccess;
  k_xh1_setup<P><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
  return cudaGetLastError();
}

template <int P>
static cudaError_t xh1_fill_p(const XFillArgs &a, cudaStream_t st, int *smem_out) {
  // largest z-chunk whose shared memory keeps >= 3 CTAs per SM (<= 72 KB dynamic)
  int kz = a.ncz;
  while (kz > 1 && xh1_layout(a.ncx, a.ncy, a.ncz, kz).bytes > 72 * 1024) --kz;
  const int smem = xh1_layout(a.ncx, a.ncy, a.ncz, kz).bytes;
  if (smem_out) { *smem_out = smem; return cudaSuccess; }
  if (a.nel_local <= 0) return cudaSuccess;
  cudaFuncSetAttribute(k_xh1_fill<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_xh1_fill<P>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  k_xh1_fill<P><<<(unsigned)a.nel_local, 128, smem, st>>>(a, kz);
  return cudaGetLastError();
}

cudaError_t launch_xh1_setup(int p, const XSetupArgs &a, cudaStream_t st) {
  switch (p) {
    case 1: return xh1_setup_p<1>(a, st);
    case 2: return xh1_setup_p<2>(a, st);
    case 3: return xh1_setup_p<3>(a, st);
    case 4: return xh1_setup_p<4>(a, st);
    case 5: return xh1_setup_p<5>(a, st);
    case 6: return xh1_setup_p<6>(a, st);
    case 7: return xh1_setup_p<7>(a, st);
    case 8: return xh1_setup_p<8>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_xh1_fill(int p, const XFillArgs &a, cudaStream_t st, int *smem_out) {
  switch (p) {
    case 1: return xh1_fill_p<1>(a, st, smem_out);
    case 2: return xh1_fill_p<2>(a, st, smem_out);
    case 3: return xh1_fill_p<3>(a, st, smem_out);
    case 4: return xh1_fill_p<4>(a, st, smem_out);
    case 5: return xh1_fill_p<5>(a, st, smem_out);
    case 6: return xh1_fill_p<6>(a, st, smem_out);
    case 7: return xh1_fill_p<7>(a, st, smem_out);
    case 8: return xh1_fill_p<8>(a, st, smem_out);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lorb
