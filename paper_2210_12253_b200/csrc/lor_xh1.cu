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
#include <cstdlib>
#include <cstring>
#include <stdint.h>

#include <utility>

#include "lor_device.cuh"
#include "lor_xdev.cuh"
#include "lor_xframe.h"

#ifndef XPFENCE
#define XPFENCE 2  // persistent fill: corners per fence in the cell phase
#endif
#ifndef XMINB
#define XMINB 5  // CTAs per SM of the one-chunk fill kernels (p <= 4): 96 registers
#endif

namespace lorb {

using namespace xdev;

namespace {

__device__ __forceinline__ void cross3x(const double *a, const double *b, double *c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}
__device__ __forceinline__ double dot3x(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

}  // namespace

// ============================================================================== fill kernel
// Compile-time geometry of the shared-memory boxes.  NB = cell-box extent per axis the kernel is
// built for: P+1 (every element of the mesh has a box of at most P+1 cells per axis: elements
// owning entities on one side per axis -- lexicographic and orientation-scrambled structured
// meshes) or P+2 (general).  All box-local index arithmetic then has constant strides.
template <int P, int NB, int NCOMP = 3>  // NCOMP = 5: + the coefficient boxes a, b (NEXT-3)
struct XCfg {
  static constexpr int PB = NB + 1;                 // points per axis of the point box
  static constexpr int NPB = PB * PB * PB;
  static constexpr int LAY = NB * NB;               // cells per layer
  static constexpr int CE = 32;                     // stored entries per cell (36 packed minus the
                                                    // four body diagonals, exactly 0 under the vertex rule)
  static constexpr int CP = 35;                     // cell pitch (doubles): 2*CP = 6 (mod 32), conflict-free
                                                    // cell writes and row gathers; 35 >= 27*10/8 holds a
                                                    // chunk's staged rows in one ring slot
  static constexpr bool ONE = NB * LAY * CP * 8 <= 36 * 1024;  // all cells resident: one chunk
  static constexpr int KZ = ONE ? P + 1 : 1;       // row layers per chunk
  static constexpr int NR = ONE ? NB : 2;          // resident cell layers (ring)
  static constexpr int NP1 = P + 1;
  static constexpr int MAXROW = KZ * NP1 * NP1;     // rows per chunk (<= 125 for P <= 4, (P+1)^2 else)
  // one chunk: E-vector box and cells are contiguous, and the staging of the element's rows (values
  // and int32 columns, 12 B per entry) is placed over both once the cells have been read; ring:
  // the restriction sits between them, staging uses one ring slot (values + uint16 box points)
  // E-vector box in shared memory: point (u0, u1, u2) at u0 + XR u1 + XS u2 per component (pitch
  // XN).  One chunk: odd pitches (P = 4: 7, 43) so that a thread->cell assignment exists in which
  // the 16 lanes of every half-warp read distinct banks (cell_perm); ring: dense
  static constexpr int XR = ONE ? (PB % 2 ? PB : PB + 1) : PB;
  static constexpr int XS = ONE ? PB * XR + 1 : PB * PB;
  static constexpr int XN = ONE ? XS * PB : NPB;
  static constexpr int XEB = NCOMP * XN * 8;
  static constexpr int STAGE1 = MAXROW * 27 * 12;
  static constexpr int OFF_CM_1 = XEB;
  static constexpr int NSL = ONE ? 128 : NR * LAY;  // cell storage slots (one chunk: slot = thread)
  static constexpr int CMB_1 = (XEB + NSL * CP * 8 >= STAGE1) ? NSL * CP * 8 : (STAGE1 - XEB + 15) / 16 * 16;
  static constexpr int OFF_XG = ONE ? OFF_CM_1 + CMB_1 : XEB;
  static constexpr int OFF_CM = ONE ? OFF_CM_1 : (OFF_XG + NPB * 4 + 15) / 16 * 16;
  static constexpr int NCHUNK = ONE ? 1 : P + 1;
  static constexpr int OFF_MT = ONE ? (OFF_XG + NPB * 4 + 15) / 16 * 16 : OFF_CM + NR * LAY * CP * 8;  // per chunk row: out int64
  static constexpr int OFF_SO = OFF_MT + 8 * MAXROW;                      // per chunk row: length
  static constexpr int OFF_INV = OFF_SO + 4 * MAXROW;                     // one chunk: cell -> storage slot
  static constexpr int SMEM = OFF_INV + (ONE ? 128 : 0);
  // staging of a chunk's rows for the write-out: the values of every row in final position order
  // in its thread's 27-entry segment, and the column (one chunk: int32) or its box point (ring:
  // uint16), placed over cell storage no longer needed (one chunk: all of it; ring: the slot the
  // next chunk overwrites first)
  static_assert(ONE ? STAGE1 <= XEB + CMB_1 : MAXROW * 27 * 10 <= LAY * CP * 8, "stage does not fit");
  static_assert(MAXROW <= 128, "one row per thread per chunk");
  static_assert(MAXROW * 27 <= 4096, "12-bit staging offsets");
};

// ============================================================================== setup kernel
// Box table of every element (125 boxes of the extended frame), the position table of every
// owned row (final position of each of the 27 stencil slots in the ascending-column CSR row, and
// the row's staging offset), and the write-out pieces of every chunk of the fill kernel.
template <int P, int NB>
__global__ void __launch_bounds__(128) k_xh1_setup(XSetupArgs A) {
  using CF = XCfg<P, NB>;
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
    int64_t f = H.el;
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
  {
    const int pb = A.nb + 1, npb = pb * pb * pb;
    for (int i = threadIdx.x; i < npb; i += blockDim.x) {
      const int u[3] = {i % pb, (i / pb) % pb, i / (pb * pb)};
      bool in = true;
      for (int a = 0; a < 3; ++a) in = in && u[a] <= H.chi[a] - H.clo[a] + 1;
      const int y[3] = {H.clo[0] + u[0], H.clo[1] + u[1], H.clo[2] + u[2]};
      bool okg = true;
      const int g = in ? gid(y, okg) : -1;
      if (!okg) atomicExch(A.err, 1);
      A.xmap[e * npb + i] = g;
    }
    // coordinate gather list of the box points that lie in neighbours (box lexicographic order)
    if (threadIdx.x == 0) {
      constexpr int NP1c = P + 1;
      const int hc = npb - NP1c * NP1c * NP1c;
      int k = 0;
      for (int i = 0; i < npb; ++i) {
        const int u[3] = {i % pb, (i / pb) % pb, i / (pb * pb)};
        const int y[3] = {H.clo[0] + u[0], H.clo[1] + u[1], H.clo[2] + u[2]};
        if (y[0] >= 0 && y[0] <= P && y[1] >= 0 && y[1] <= P && y[2] >= 0 && y[2] <= P) continue;
        int2 ent = make_int2(-1, i);
        bool in = true;
        for (int a = 0; a < 3; ++a) in = in && u[a] <= H.chi[a] - H.clo[a] + 1;
        if (in) {
          const int ni = (ydelta(y[0], P) + 1) + 3 * (ydelta(y[1], P) + 1) + 9 * (ydelta(y[2], P) + 1);
          const XNbr nb = H.nbr[ni];
          int L[3];
          x_to_local(P, nb.code, y, L);
          if (nb.el < 0) atomicExch(A.err, 1);
          ent.x = (int)((int64_t)nb.el * A.xstride + L[0] + NP1c * (L[1] + NP1c * L[2]));
        }
        if (k < hc) A.xhalo[e * hc + k] = ent;
        ++k;
      }
      if (k != hc) atomicExch(A.err, 1);
    }
  }
}

// Symbolic pass of the extended-frame path, per call (A2: the row lengths the
// scan turns into I, and where every column goes in its row).  For every owned row of the element
// (the minimal element containing its coarse entity):
//   * its length: the stencil points sharing a cell with it -- per axis the offsets d whose cells
//     [max(x, x+d) - 1, min(x, x+d)] meet the element's cell box, a product over the three axes;
//   * the final position of each stencil slot in the ascending-column row (reading P-5): the order
//     of the slot ids (extended element restriction, setup) -- a sorting network on packed keys
//     (ids < 2^26), else the 351 pairwise comparisons.
// One CTA (NT threads) per element.  Outputs cnt[row], pos[row][8 words] (bytes 0-26: position,
// 255 = not a column).
template <int P, int NB, int NT>
__global__ void __launch_bounds__(NT) k_xh1_sym(XFillArgs A) {
  constexpr int PB = NB + 1, NPB = PB * PB * PB;
  __shared__ int32_t XG[NPB];
  __shared__ __align__(16) uint8_t s_pos[NT * 28];  // per-thread position scatter
  __shared__ uint32_t s_cls[P >= 5 ? 125 * 7 : 1];   // p >= 5: positions per row class
  const int tid = threadIdx.x;
  const int64_t bs = blockIdx.x;
  if (bs >= A.nel_local) return;
  const int4 hw = __ldg(reinterpret_cast<const int4 *>(A.xe + bs));
  const int32_t *xm = A.xmap + bs * NPB;
  for (int i = tid; i < NPB; i += NT) XG[i] = __ldg(xm + i);
  const int clo[3] = {(int8_t)(hw.y & 255), (int8_t)((hw.y >> 8) & 255), (int8_t)((hw.y >> 16) & 255)};
  const int chi[3] = {(int8_t)((hw.y >> 24) & 255), (int8_t)(hw.z & 255), (int8_t)((hw.z >> 8) & 255)};
  const int olo[3] = {(int8_t)((hw.z >> 16) & 255), (int8_t)((hw.z >> 24) & 255), (int8_t)(hw.w & 255)};
  const int ohi[3] = {(int8_t)((hw.w >> 8) & 255), (int8_t)((hw.w >> 16) & 255), (int8_t)((hw.w >> 24) & 255)};
  const uint32_t own = (uint32_t)hw.x;
  const int rnx = ohi[0] - olo[0] + 1, rny = ohi[1] - olo[1] + 1, nrow = rnx * rny * (ohi[2] - olo[2] + 1);
  // positions of one row (lattice point x, per-axis valid-offset masks m)
  auto row_positions = [&](const int x[3], const int m[3], uint32_t (&pw)[7]) {
    const int px = (x[0] - clo[0]) + PB * ((x[1] - clo[1]) + PB * (x[2] - clo[2]));
    int key[27];
#pragma unroll
    for (int j = 0; j < 27; ++j) {
      const int dx = j % 3, dy = (j / 3) % 3, dz = j / 9;
      const bool v = (m[0] >> dx) & (m[1] >> dy) & (m[2] >> dz) & 1;
      key[j] = v ? XG[px + (dx - 1) + PB * (dy - 1) + PB * PB * (dz - 1)] - A.key_base : 0x7fffffff;
    }
    xdev::row_positions<27>(key, A.sort32 != 0, s_pos + tid * 28, pw);
  };
  auto masks = [&](const int x[3], int m[3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
      m[a] = ((x[a] - 1 >= clo[a] && x[a] - 1 <= chi[a]) ? 1 : 0) | ((x[a] - 1 <= chi[a] && x[a] >= clo[a]) ? 2 : 0) |
             ((x[a] >= clo[a] && x[a] <= chi[a]) ? 4 : 0);
  };
  // p >= 5: rows whose three per-axis classes (x = 0, 1, [2, p-2], p-1, p) agree have the same
  // coarse entities at the same stencil slots and the same affine order inside each -- hence the
  // same positions: computed once per class from a representative row (125 classes vs (p+1)^3 rows)
  constexpr bool CLS = P >= 5;
  auto acls = [](int x) { return x <= 1 ? x : (x <= P - 2 ? 2 : (x == P - 1 ? 3 : 4)); };
  __syncthreads();
  if (CLS) {
    for (int c = tid; c < 125; c += NT) {
      const int k[3] = {c % 5, (c / 5) % 5, c / 25};
      int x[3], m[3];
      bool in = true;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        x[a] = k[a] <= 2 ? k[a] : (k[a] == 3 ? P - 1 : P);
        in = in && x[a] >= olo[a] && x[a] <= ohi[a];
      }
      if (!in) continue;
      masks(x, m);
      uint32_t pw[7];
      row_positions(x, m, pw);
#pragma unroll
      for (int q2 = 0; q2 < 7; ++q2) s_cls[c * 7 + q2] = pw[q2];
    }
    __syncthreads();
  }
  for (int t = tid; t < nrow; t += NT) {
    const int q = t / rnx;
    const int x[3] = {olo[0] + t - q * rnx, olo[1] + q % rny, olo[2] + q / rny};
    if (!((own >> (lcls(x[0], P) + 3 * lcls(x[1], P) + 9 * lcls(x[2], P))) & 1)) continue;
    int m[3];
    masks(x, m);
    const int px = (x[0] - clo[0]) + PB * ((x[1] - clo[1]) + PB * (x[2] - clo[2]));
    const int64_t r = (int64_t)XG[px] - A.row_begin;
    A.cnt[r] = __popc(m[0]) * __popc(m[1]) * __popc(m[2]);
    uint32_t pw[7];
    if (CLS) {
      const int c = acls(x[0]) + 5 * acls(x[1]) + 25 * acls(x[2]);
#pragma unroll
      for (int q2 = 0; q2 < 7; ++q2) pw[q2] = s_cls[c * 7 + q2];
    } else {
      row_positions(x, m, pw);
    }
    uint4 *dst = reinterpret_cast<uint4 *>(A.pos + r * 8);
    dst[0] = make_uint4(pw[0], pw[1], pw[2], pw[3]);
    dst[1] = make_uint4(pw[4], pw[5], pw[6], 0xffffffffu);
  }
}

// packed index of the cell-matrix entry (a, b), a <= b, with the four body diagonals removed
__host__ __device__ constexpr int cidx(int a, int b) {
  const int i = a < b ? a : b, j = a < b ? b : a;
  const int t = i * 8 - i * (i - 1) / 2 + (j - i);  // tri(8, i, j)
  // body diagonals (q, q^7), q < 4, sit at tri indices 7, 13, 18, 22
  return t - (t > 7) - (t > 13) - (t > 18) - (t > 22);
}
__host__ __device__ constexpr bool body_diag(int a, int b) { return (a ^ b) == 7; }

// One LOR cell under the vertex rule (reading P-1), computed by one thread with the corner loop
// unrolled: at corner q the Jacobian columns are the cell edge vectors through q, Q = w a
// adj adj^T / det, and the corner adds (same terms as lor_cells.cuh)
//   (q,q) += s^T Q s + w b det,  (q^d,q^d) += Q_dd,  (q,q^d) += -s_d (Q s)_d,
//   (q^d,q^d') += s_d s_d' Q_dd'   (s = reference gradient signs of N_q, compile-time).
// 32 entries (cidx order) stored at o[0..31]; returns false if det J <= 0 at a corner.
// does corner q of a cell add to the entry (a, b) (see cell_h1v)?
__host__ __device__ constexpr bool corner_touches(int q, int a, int b) {
  if (a > b) { const int t = a; a = b; b = t; }
  if (a == b) return a == q || (a ^ q) == 1 || (a ^ q) == 2 || (a ^ q) == 4;       // diagonal
  const int x = a ^ b;
  if (x == 1 || x == 2 || x == 4) return q == a || q == b;                         // edge
  if (x == 7) return false;                                                        // body diagonal
  return (q ^ a) != 0 && (q ^ b) != 0 && ((q ^ a) | (q ^ b)) == x;                 // face diagonal
}
__host__ __device__ constexpr bool first_touch(int q, int a, int b) {
  for (int k = 0; k < q; ++k)
    if (corner_touches(k, a, b)) return false;
  return true;
}

// VC: variable coefficients -- the boxes XE[3 XN ...] (a) and XE[4 XN ...] (b) hold the coefficient
// E-vectors; corner q's contributions are scaled by a and b at its point (vertex rule, reading P-28)
template <int XN, int XR, int XS, int FENCE = 1, bool VC = false>
__device__ __forceinline__ bool cell_h1v(const double *__restrict__ XE, int pb, double a8, double b8, double *__restrict__ o) {
  auto X = [&](int v, int k) -> double { return XE[k * XN + pb + (v & 1) + XR * ((v >> 1) & 1) + XS * ((v >> 2) & 1)]; };
  // accumulate in the cell's (thread-private) shared-memory row: the first corner touching an
  // entry stores, later ones add (compile-time after unrolling)
  auto put = [&](int q, int ea, int eb, double v) {
    double &dst = o[cidx(ea, eb)];
    if (first_touch(q, ea, eb)) dst = v;
    else dst += v;
  };
  bool ok = true;
  double dg[8];  // the eight diagonal entries (four corners each) accumulate in registers
#pragma unroll
  for (int q = 0; q < 8; ++q) dg[q] = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    // corners are evaluated one after the other (the fence keeps the compiler from hoisting every
    // corner's loads and arithmetic at once: ~200 registers otherwise; caching the eight points in
    // registers instead spills at 128); the corner re-reads its four points from shared memory.
    // FENCE = 2: two corners in flight (more ILP where the register budget allows)
    if (q % FENCE == 0) asm volatile("" ::: "memory");
    double j[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int k = 0; k < 3; ++k)
        j[d][k] = X(q | (1 << d), k) - X(q & ~(1 << d), k);
    double r[3][3];
    cross3x(j[1], j[2], r[0]);
    cross3x(j[2], j[0], r[1]);
    cross3x(j[0], j[1], r[2]);
    const double det = dot3x(j[0], r[0]);
    ok = ok && det > 0.0;
    const double sa = (VC ? a8 * X(q, 3) : a8) * rcp_pos(det);
    double Q[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int e = d; e < 3; ++e) Q[d][e] = Q[e][d] = sa * dot3x(r[d], r[e]);
    const double s0 = (q & 1) ? 1.0 : -1.0, s1 = ((q >> 1) & 1) ? 1.0 : -1.0, s2 = ((q >> 2) & 1) ? 1.0 : -1.0;
    double Qs[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) Qs[d] = s0 * Q[d][0] + s1 * Q[d][1] + s2 * Q[d][2];
    dg[q] += s0 * Qs[0] + s1 * Qs[1] + s2 * Qs[2] + (VC ? b8 * X(q, 4) : b8) * det;
    dg[q ^ 1] += Q[0][0];
    dg[q ^ 2] += Q[1][1];
    dg[q ^ 4] += Q[2][2];
    put(q, q, q ^ 1, -s0 * Qs[0]);
    put(q, q, q ^ 2, -s1 * Qs[1]);
    put(q, q, q ^ 4, -s2 * Qs[2]);
    put(q, q ^ 1, q ^ 2, s0 * s1 * Q[0][1]);
    put(q, q ^ 1, q ^ 4, s0 * s2 * Q[0][2]);
    put(q, q ^ 2, q ^ 4, s1 * s2 * Q[1][2]);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) o[cidx(q, q)] = dg[q];
  return ok;
}

// WCOL = false: numeric-only re-assembly (pattern reuse): col keeps what the
// previous full call wrote, only val is stored.
template <int P, int NB, int MINB, bool WCOL, bool VC = false>
__global__ void __launch_bounds__(128, MINB) k_xh1_fill(XFillArgs A) {
  using CF = XCfg<P, NB, VC ? 5 : 3>;
  constexpr int NP1 = P + 1, NPT = NP1 * NP1 * NP1, PB = CF::PB, NPB = CF::NPB, LAY = CF::LAY, CP = CF::CP;
  constexpr int NR = CF::NR;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_bad;
  double *XE = reinterpret_cast<double *>(smem);  // one chunk: also the start of the staging area
  int32_t *XG = reinterpret_cast<int32_t *>(smem + CF::OFF_XG);
  double *cm = reinterpret_cast<double *>(smem + CF::OFF_CM);
  int64_t *m_out = reinterpret_cast<int64_t *>(smem + CF::OFF_MT);  // per chunk row: CSR offset (-1: none)
  int32_t *m_n = reinterpret_cast<int32_t *>(smem + CF::OFF_SO);     // per chunk row: length
  uint8_t *s_inv = smem + CF::OFF_INV;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if ((int64_t)blockIdx.x >= A.nel_local) return;
  const int64_t bs = blockIdx.x;  // processing slot: element record, restriction, gather list, pieces
#define XSTAMP(k) \
  do { if (A.tstamp && tid == 0) A.tstamp[(int64_t)blockIdx.x * 16 + (k)] = clock64(); } while (0)
  XSTAMP(0);
  // element header word {own, clo, chi, olo, ohi} read by every thread (broadcast); all loads of the
  // prologue (extended restriction, own E-vector, neighbour points) are independent of each other
  // and complete at one barrier
  const int4 hw = __ldg(reinterpret_cast<const int4 *>(A.xe + bs));
  const int64_t el = __ldg(&A.xe[bs].el);  // same round trip as the header
  // L2 prefetch for the CTA that takes this CTA's place about one CTA lifetime from now (slot +
  // resident CTAs): its record, restriction and gather list now; its E-vector (needs its element
  // id) after the cell phase; its neighbour points (need its gather list) before the write-out
  constexpr int HC = NPB - NPT;
  const int64_t nbs = bs + A.pf_dist;
  const bool pf = A.pf_dist > 0 && nbs < A.nel_local;
  int pf_el = -1;
  int2 pf_h = make_int2(-1, 0);
  if (pf) {
    constexpr int LX = (int)((sizeof(XElem) + 127) / 128), LM = (NPB * 4 + 127) / 128 + 1, LH = (HC * 8 + 127) / 128 + 1;
    if (tid < LX) pf_l2(reinterpret_cast<const char *>(A.xe + nbs) + 128 * tid);
    else if (tid < LX + LM) pf_l2(reinterpret_cast<const char *>(A.xmap + nbs * NPB) + 128 * (tid - LX));
    else if (tid < LX + LM + LH) pf_l2(reinterpret_cast<const char *>(A.xhalo + nbs * HC) + 128 * (tid - LX - LM));
    if (tid == 127) pf_el = __ldg(&A.xe[nbs].el);
  }
  const int clo0 = (int8_t)(hw.y & 255), clo1 = (int8_t)((hw.y >> 8) & 255), clo2 = (int8_t)((hw.y >> 16) & 255);
  const int ex0 = (int8_t)((hw.y >> 24) & 255) - clo0 + 1, ex1 = (int8_t)(hw.z & 255) - clo1 + 1,
            ex2 = (int8_t)((hw.z >> 8) & 255) - clo2 + 1;  // cell-box extents (<= NB)
  const int olo0 = (int8_t)((hw.z >> 16) & 255), olo1 = (int8_t)((hw.z >> 24) & 255), olo2 = (int8_t)(hw.w & 255);
  const int ohi0 = (int8_t)((hw.w >> 8) & 255), ohi1 = (int8_t)((hw.w >> 16) & 255), ohi2 = (int8_t)((hw.w >> 24) & 255);
  const uint32_t own = (uint32_t)hw.x;
  const int pbase = -(clo0 + PB * (clo1 + PB * clo2));  // box-local index of lattice point 0
  {
    if (tid == 0) s_bad = 0;
    if (CF::ONE && tid < NB * NB * NB) s_inv[tid] = A.cinv[tid];
    // extended element restriction (setup): global id of every point of the box
    const int32_t *xm = A.xmap + bs * NPB;
    for (int i = tid; i < NPB; i += blockDim.x) XG[i] = __ldg(xm + i);
    // own E-vector (and coefficient E-vectors), one lattice x-row per thread
    const double *xs = A.X + el * A.xstride;
    for (int rr = tid; rr < (VC ? 5 : 3) * NP1 * NP1; rr += blockDim.x) {
      const int d = rr / (NP1 * NP1), x12 = rr - d * NP1 * NP1, x1 = x12 % NP1, x2 = x12 / NP1;
      const double *src = d < 3 ? xs + d * NPT + x12 * NP1 : (d == 3 ? A.ca : A.cb) + el * NPT + x12 * NP1;
      double *dst = XE + d * CF::XN + (x1 - clo1) * CF::XR + (x2 - clo2) * CF::XS - clo0;
#pragma unroll
      for (int i = 0; i < NP1; ++i) dst[i] = __ldg(src + i);
    }
    // neighbour points of the box (setup gather list)
    const int2 *hl = A.xhalo + bs * HC;
    for (int h = tid; h < HC; h += blockDim.x) {
      const int2 hv = __ldg(hl + h);
      if (hv.x >= 0) {
        const int q = hv.y % PB + CF::XR * ((hv.y / PB) % PB) + CF::XS * (hv.y / (PB * PB));
        XE[q] = __ldg(A.X + hv.x);
        XE[CF::XN + q] = __ldg(A.X + hv.x + NPT);
        XE[2 * CF::XN + q] = __ldg(A.X + hv.x + 2 * NPT);
        if (VC) {  // the neighbour's coefficient at the same point (its element e', point l)
          const int64_t e2 = hv.x / A.xstride, l2 = hv.x - e2 * A.xstride;
          XE[3 * CF::XN + q] = __ldg(A.ca + e2 * NPT + l2);
          XE[4 * CF::XN + q] = __ldg(A.cb + e2 * NPT + l2);
        }
      }
    }
  }
  __syncthreads();
  XSTAMP(1);
  // rows: the owned-row bounding box [olo, ohi], z-layers in chunks of KZ
  const int zlo = olo2, zhi = ohi2;
  const int rnx = ohi0 - olo0 + 1, rny = ohi1 - olo1 + 1;
  const double alpha = A.alpha, beta = A.beta;
  double *stage_v = cm;  // overwritten per chunk, see below
  for (int z0 = zlo, ch = 0; z0 <= zhi; z0 += CF::KZ, ++ch) {
    const int z1 = (z0 + CF::KZ - 1 < zhi) ? z0 + CF::KZ - 1 : zhi;
    // cell layers to compute now (lattice coordinates): [z0-1 (first chunk only), z1] within the box
    int c0 = (z0 == zlo) ? z0 - 1 : z0;
    int c1 = z1;
    c0 = c0 < clo2 ? clo2 : c0;
    c1 = c1 > clo2 + ex2 - 1 ? clo2 + ex2 - 1 : c1;
    if (c1 >= c0) {
      const int ncell = (c1 - c0 + 1) * LAY;
      const double a8 = 0.125 * alpha, b8 = 0.125 * beta;
      for (int c = tid; c < (CF::ONE ? 128 : 128 * (c1 - c0 + 1)); c += blockDim.x) {
        // thread -> cell by the bank-conflict-free permutation (one chunk: the whole box, cell
        // stored at slot = thread; ring: one layer per 128 threads, natural slots)
        const int cc = CF::ONE ? (int)A.cperm[c] : ((int)A.cperm[c & 127] < LAY ? (int)A.cperm[c & 127] + LAY * (c >> 7) : ncell);
        if (cc >= ncell) continue;
        const int ux = cc % NB, uy = (cc / NB) % NB, uz = c0 - clo2 + cc / LAY;  // box-local cell
        if (ux >= ex0 || uy >= ex1) continue;
        double *dstc = cm + (CF::ONE ? c : ((uz % NR) * LAY + uy * NB + ux)) * CP;
        // det J <= 0 in any cell of the box -- own or a neighbour's, which may be computed by no
        // other CTA (an element owning no rows) -- is reported (extended-frame cell coordinates)
        if (!cell_h1v<CF::XN, CF::XR, CF::XS, 1, VC>(XE, ux + CF::XR * uy + CF::XS * uz, a8, b8, dstc))
          s_bad = 1 + (clo0 + ux + 1) + (P + 2) * ((clo1 + uy + 1) + (P + 2) * (clo2 + uz + 1));
      }
    }
    __syncthreads();
    if (ch == 0) XSTAMP(2);
    if (pf && ch == 0) {
      // next CTA's E-vector (3 x (p+1)^3 doubles, 128-byte aligned) and gather list entries
      const int pe = __shfl_sync(0xffffffffu, pf_el, 31);
      if (warp == 3 && pe >= 0) {
        const char *xp = reinterpret_cast<const char *>(A.X + (int64_t)pe * A.xstride);
        for (int l = lane; l < (3 * NPT * 8 + 127) / 128; l += 32) pf_l2(xp + 128 * l);
      }
      if (tid < HC) pf_h = __ldg(A.xhalo + nbs * HC + tid);
    }
    if (s_bad && tid == 0) {  // map the extended-frame cell to (element, cell) of the element it lies in
      const int b = s_bad - 1, q[3] = {b % (P + 2) - 1, (b / (P + 2)) % (P + 2) - 1, b / ((P + 2) * (P + 2)) - 1};
      const int ni = (q[0] < 0 ? 0 : (q[0] >= P ? 2 : 1)) + 3 * (q[1] < 0 ? 0 : (q[1] >= P ? 2 : 1)) +
                     9 * (q[2] < 0 ? 0 : (q[2] >= P ? 2 : 1));
      int64_t ee = el;
      int kc[3] = {q[0], q[1], q[2]};
      if (ni != 13) {
        const XNbr nb = A.xe[bs].nbr[ni];
        ee = nb.el;
        int y0[3] = {q[0], q[1], q[2]}, y1[3] = {q[0] + 1, q[1] + 1, q[2] + 1}, L0[3], L1[3];
        x_to_local(P, nb.code, y0, L0);
        x_to_local(P, nb.code, y1, L1);
        for (int a = 0; a < 3; ++a) kc[a] = L0[a] < L1[a] ? L0[a] : L1[a];
      }
      xreport(A.err, 2, A.elem_begin + ee, kc[0] + P * (kc[1] + P * kc[2]));
      s_bad = 0;
    }
    // the chunk's write-out pieces (setup), consumed after the staging barrier
    // ---- rows of layers [z0, z1]: one thread per owned row, values from the <= 8 cells
    const int nrow = rnx * rny * (z1 - z0 + 1);
    double acc[27];
    uint32_t pw[8];
    int px = 0, nrw = 0;
    int64_t out = 0;
    bool hasrow = false;
    int x0 = 0, x1 = 0, x2 = 0;
    if (tid < nrow) {
      const int t = tid / rnx;
      x0 = olo0 + tid - t * rnx;
      x1 = olo1 + t % rny;
      x2 = z0 + t / rny;
      hasrow = (own >> (lcls(x0, P) + 3 * lcls(x1, P) + 9 * lcls(x2, P))) & 1;
    }
    if (hasrow) {
      px = pbase + x0 + PB * (x1 + PB * x2);
      const int64_t r = (int64_t)XG[px] - A.row_begin;
      out = __ldg(A.row_ptr + r);
      nrw = (int)(__ldg(A.row_ptr + r + 1) - out);
      const uint4 *pp = reinterpret_cast<const uint4 *>(A.pos + r * 8);
      const uint4 pa = __ldcs(pp), pv = __ldcs(pp + 1);
      pw[0] = pa.x; pw[1] = pa.y; pw[2] = pa.z; pw[3] = pa.w;
      pw[4] = pv.x; pw[5] = pv.y; pw[6] = pv.z; pw[7] = pv.w;
#pragma unroll
      for (int jj = 0; jj < 27; ++jj) acc[jj] = 0.0;
      const int u0 = x0 - clo0, u1 = x1 - clo1, u2 = x2 - clo2;  // box-local lattice point
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        const int ox = o & 1, oy = (o >> 1) & 1, oz = (o >> 2) & 1;
        const int cx = u0 - ox, cy = u1 - oy, cz = u2 - oz;
        if (cx < 0 || cx >= ex0 || cy < 0 || cy >= ex1 || cz < 0 || cz >= ex2) continue;
        const double *ce = cm + (CF::ONE ? (int)s_inv[cz * LAY + cy * NB + cx] : ((cz % NR) * LAY + cy * NB + cx)) * CP;
#pragma unroll
        for (int jc = 0; jc < 8; ++jc) {
          if (body_diag(o, jc)) continue;
          const int dx = (jc & 1) - ox, dy = ((jc >> 1) & 1) - oy, dz = ((jc >> 2) & 1) - oz;
          acc[(dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)] += ce[cidx(o, jc)];
        }
        asm volatile("" ::: "memory");  // one cell's loads in flight at a time (register pressure)
      }
    }
    __syncthreads();  // every row has read the cells: stage over the cell storage
    if (ch == 0) XSTAMP(5);
    if (pf_h.x >= 0) {  // next CTA's neighbour points
      pf_l2(A.X + pf_h.x);
      pf_l2(A.X + pf_h.x + NPT);
      pf_l2(A.X + pf_h.x + 2 * NPT);
      pf_h.x = -1;
    }
    // stage: ONE chunk -> all cells; ring -> the slot of layer z0-1 (next chunk's first write)
    stage_v = CF::ONE ? XE : cm + (((z0 - 1 - clo2) % NR + NR) % NR) * LAY * CP;
    uint16_t *stage_p = reinterpret_cast<uint16_t *>(stage_v + CF::MAXROW * 27);  // ring: box point of the column
    int32_t *stage_c = reinterpret_cast<int32_t *>(stage_v + CF::MAXROW * 27);    // one chunk: the column
    if (hasrow) {  // the row's values and columns in final position order at its thread's segment
      const int so = tid * 27;
#pragma unroll
      for (int jj = 0; jj < 27; ++jj) {
        const int ps = (int)((pw[jj >> 2] >> (8 * (jj & 3))) & 255u);
        if (ps != 255) {
          stage_v[so + ps] = acc[jj];
          const int pt = px + (jj % 3 - 1) + PB * ((jj / 3) % 3 - 1) + PB * PB * (jj / 9 - 1);
          if constexpr (CF::ONE) stage_c[so + ps] = XG[pt];
          else stage_p[so + ps] = (uint16_t)pt;
        }
      }
    }
    if (tid < CF::MAXROW) {
      m_out[tid] = hasrow ? out : -1;
      m_n[tid] = hasrow ? nrw : 0;
    }
    __syncthreads();
    if (ch == 0) XSTAMP(3);
    // write-out: one warp per row, lane k stores entry k, two rows in flight per warp (consecutive
    // rows of a coarse entity are consecutive CSR ranges: the sectors a row leaves partial are
    // completed by its neighbour while both are in L2)
    for (int t = warp; t < nrow; t += 8) {
      const int t2 = t + 4;
      const int64_t o = m_out[t], o2 = t2 < nrow ? m_out[t2] : -1;
      const int n = m_n[t], n2 = t2 < nrow ? m_n[t2] : 0;
      const bool w1 = o >= 0 && lane < n, w2 = o2 >= 0 && lane < n2;
      int32_t c1 = 0, c2 = 0;
      double v1 = 0.0, v2 = 0.0;
      if (w1) { c1 = CF::ONE ? stage_c[t * 27 + lane] : XG[stage_p[t * 27 + lane]]; v1 = stage_v[t * 27 + lane]; }
      if (w2) { c2 = CF::ONE ? stage_c[t2 * 27 + lane] : XG[stage_p[t2 * 27 + lane]]; v2 = stage_v[t2 * 27 + lane]; }
      if (w1) {
        if (WCOL) __stcs(A.col + o + lane, c1);
        __stcs(A.val + o + lane, v1);
      }
      if (w2) {
        if (WCOL) __stcs(A.col + o2 + lane, c2);
        __stcs(A.val + o2 + lane, v2);
      }
    }
    __syncthreads();
  }
  XSTAMP(4);
#undef XSTAMP
}

// ============================================================================== persistent fill
// One-chunk configurations (p <= 4): a persistent CTA walks the elements bs = blockIdx.x + k gridDim.x
// and loads the NEXT element's prologue (extended restriction, gather list, own E-vector, neighbour
// points) with cp.async into a second shared-memory buffer while it computes the current one -- the
// prologue (a quarter of a CTA's lifetime as one-shot CTAs: 5.5 K of 21 K cycles, C2) leaves the
// critical path.  The staging of the rows sits in the cell storage (values + uint16 box points;
// the current buffer's restriction gives the column at write-out).  Same arithmetic and output
// as k_xh1_fill.
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int P, int NB>
struct XPCfg {
  using CF = XCfg<P, NB>;
  static constexpr int NPT = (P + 1) * (P + 1) * (P + 1);
  static constexpr int HC = CF::NPB - NPT;
  static constexpr int OFF_XG = (CF::XEB + 15) / 16 * 16, OFF_HL = (OFF_XG + CF::NPB * 4 + 15) / 16 * 16;
  static constexpr int BUF = (OFF_HL + HC * 8 + 15) / 16 * 16;  // XE | XG | gather list
  static constexpr int OFF_CM = 2 * BUF;
  static constexpr int CMB = CF::NSL * CF::CP * 8;
  static constexpr int OFF_MT = OFF_CM + CMB;
  static constexpr int OFF_SO = OFF_MT + 8 * CF::MAXROW;
  static constexpr int OFF_INV = OFF_SO + 4 * CF::MAXROW;
  static constexpr int SMEM = OFF_INV + 128;
  static_assert(CF::ONE, "persistent fill: one-chunk configurations");
  static_assert(CF::MAXROW * 27 * 10 <= CMB, "staging (values + uint16 points) must fit in the cell storage");
  static_assert(OFF_HL + HC * 8 <= BUF, "buffer layout");
};

template <int P, int NB, int MINB, bool WCOL>
__global__ void __launch_bounds__(128, MINB) k_xh1_fill_pers(XFillArgs A) {
  using CF = XCfg<P, NB>;
  using PC = XPCfg<P, NB>;
  constexpr int NP1 = P + 1, NPT = NP1 * NP1 * NP1, PB = CF::PB, NPB = CF::NPB, LAY = CF::LAY, CP = CF::CP;
  constexpr int HC = PC::HC;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_bad;
  double *cm = reinterpret_cast<double *>(smem + PC::OFF_CM);
  int64_t *m_out = reinterpret_cast<int64_t *>(smem + PC::OFF_MT);
  int32_t *m_n = reinterpret_cast<int32_t *>(smem + PC::OFF_SO);
  uint8_t *s_inv = smem + PC::OFF_INV;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto XEb = [&](int b) { return reinterpret_cast<double *>(smem + b * PC::BUF); };
  auto XGb = [&](int b) { return reinterpret_cast<int32_t *>(smem + b * PC::BUF + PC::OFF_XG); };
  auto HLb = [&](int b) { return reinterpret_cast<int2 *>(smem + b * PC::BUF + PC::OFF_HL); };
  // stage A of element e into buffer b: restriction and gather list (addresses from e alone)
  auto stage_a = [&](int64_t e, int b) {
    const int32_t *xm = A.xmap + e * NPB;
    int32_t *xg = XGb(b);
    if constexpr (NPB % 4 == 0) {  // element rows 16-byte aligned
      for (int i = tid; i < NPB / 4; i += 128) cp_async16(xg + 4 * i, xm + 4 * i);
    } else {
      for (int i = tid; i < NPB; i += 128) cp_async4(xg + i, xm + i);
    }
    const int2 *hl = A.xhalo + e * HC;
    int2 *hs = HLb(b);
    for (int h = tid; h < HC; h += 128) cp_async8(hs + h, hl + h);
    cp_commit();
  };
  // stage B of element e into buffer b: own E-vector and neighbour points (needs the element id, the
  // box corner and this thread's gather-list entries of stage A)
  auto stage_b = [&](int64_t e_el, int4 hwx, int b) {
    const int c0 = (int8_t)(hwx.y & 255), c1 = (int8_t)((hwx.y >> 8) & 255), c2 = (int8_t)((hwx.y >> 16) & 255);
    double *xe = XEb(b);
    const double *xs = A.X + e_el * A.xstride;
    for (int rr = tid; rr < 3 * NP1 * NP1; rr += 128) {
      const int d = rr / (NP1 * NP1), x12 = rr - d * NP1 * NP1, x1 = x12 % NP1, x2 = x12 / NP1;
      const double *src = xs + d * NPT + x12 * NP1;
      double *dst = xe + d * CF::XN + (x1 - c1) * CF::XR + (x2 - c2) * CF::XS - c0;
#pragma unroll
      for (int i = 0; i < NP1; ++i) cp_async8(dst + i, src + i);
    }
    const int2 *hs = HLb(b);
    for (int h = tid; h < HC; h += 128) {
      const int2 hv = hs[h];  // written by this thread's own stage-A copy (waited for by the caller)
      if (hv.x >= 0) {
        const int q = hv.y % PB + CF::XR * ((hv.y / PB) % PB) + CF::XS * (hv.y / (PB * PB));
        cp_async8(xe + q, A.X + hv.x);
        cp_async8(xe + CF::XN + q, A.X + hv.x + NPT);
        cp_async8(xe + 2 * CF::XN + q, A.X + hv.x + 2 * NPT);
      }
    }
    cp_commit();
  };
  const int64_t stride = gridDim.x;
  int64_t bs = blockIdx.x;
  if (bs >= A.nel_local) return;
  if (tid == 0) s_bad = 0;
  if (tid < NB * NB * NB) s_inv[tid] = A.cinv[tid];
  int4 hw = __ldg(reinterpret_cast<const int4 *>(A.xe + bs));
  int64_t el = __ldg(&A.xe[bs].el);
  stage_a(bs, 0);
  cp_wait_all();
  stage_b(el, hw, 0);
  const double alpha = A.alpha, beta = A.beta;
  for (int b = 0; bs < A.nel_local; bs += stride, b ^= 1) {
    cp_wait_all();
    __syncthreads();  // buffer b holds element bs; the previous element's write-out is done
    double *XE = XEb(b);
    const int32_t *XG = XGb(b);
    const int64_t nbs = bs + stride;
    int4 hwn = make_int4(0, 0, 0, 0);
    int64_t eln = 0;
    if (nbs < A.nel_local) {
      hwn = __ldg(reinterpret_cast<const int4 *>(A.xe + nbs));
      eln = __ldg(&A.xe[nbs].el);
      stage_a(nbs, b ^ 1);
    }
    const int clo0 = (int8_t)(hw.y & 255), clo1 = (int8_t)((hw.y >> 8) & 255), clo2 = (int8_t)((hw.y >> 16) & 255);
    const int ex0 = (int8_t)((hw.y >> 24) & 255) - clo0 + 1, ex1 = (int8_t)(hw.z & 255) - clo1 + 1,
              ex2 = (int8_t)((hw.z >> 8) & 255) - clo2 + 1;
    const int olo0 = (int8_t)((hw.z >> 16) & 255), olo1 = (int8_t)((hw.z >> 24) & 255), olo2 = (int8_t)(hw.w & 255);
    const int ohi0 = (int8_t)((hw.w >> 8) & 255), ohi1 = (int8_t)((hw.w >> 16) & 255), ohi2 = (int8_t)((hw.w >> 24) & 255);
    const uint32_t own = (uint32_t)hw.x;
    const int pbase = -(clo0 + PB * (clo1 + PB * clo2));
    // ---- cells: the whole box, thread -> cell by the bank-conflict-free permutation
    {
      const double a8 = 0.125 * alpha, b8 = 0.125 * beta;
      const int cc = (int)A.cperm[tid];
      if (cc < NB * LAY) {
        const int ux = cc % NB, uy = (cc / NB) % NB, uz = cc / LAY;
        if (ux < ex0 && uy < ex1 && uz < ex2) {
          if (!cell_h1v<CF::XN, CF::XR, CF::XS, XPFENCE>(XE, ux + CF::XR * uy + CF::XS * uz, a8, b8, cm + tid * CP))
            s_bad = 1 + (clo0 + ux + 1) + (P + 2) * ((clo1 + uy + 1) + (P + 2) * (clo2 + uz + 1));
        }
      }
    }
    __syncthreads();
    if (s_bad && tid == 0) {  // map the extended-frame cell to (element, cell) of the element it lies in
      const int bb = s_bad - 1, q[3] = {bb % (P + 2) - 1, (bb / (P + 2)) % (P + 2) - 1, bb / ((P + 2) * (P + 2)) - 1};
      const int ni = (q[0] < 0 ? 0 : (q[0] >= P ? 2 : 1)) + 3 * (q[1] < 0 ? 0 : (q[1] >= P ? 2 : 1)) +
                     9 * (q[2] < 0 ? 0 : (q[2] >= P ? 2 : 1));
      int64_t ee = el;
      int kc[3] = {q[0], q[1], q[2]};
      if (ni != 13) {
        const XNbr nb = A.xe[bs].nbr[ni];
        ee = nb.el;
        int y0[3] = {q[0], q[1], q[2]}, y1[3] = {q[0] + 1, q[1] + 1, q[2] + 1}, L0[3], L1[3];
        x_to_local(P, nb.code, y0, L0);
        x_to_local(P, nb.code, y1, L1);
        for (int a = 0; a < 3; ++a) kc[a] = L0[a] < L1[a] ? L0[a] : L1[a];
      }
      xreport(A.err, 2, A.elem_begin + ee, kc[0] + P * (kc[1] + P * kc[2]));
      s_bad = 0;
    }
    // next element, stage B (its gather-list entries are this thread's own stage-A copies)
    if (nbs < A.nel_local) {
      cp_wait_all();
      stage_b(eln, hwn, b ^ 1);
    }
    // ---- rows: one thread per owned row
    const int rnx = ohi0 - olo0 + 1, rny = ohi1 - olo1 + 1;
    const int nrow = rnx * rny * (ohi2 - olo2 + 1);
    double acc[27];
    uint32_t pw[8];
    int px = 0, nrw = 0;
    int64_t out = 0;
    bool hasrow = false;
    if (tid < nrow) {
      const int t = tid / rnx;
      const int x0 = olo0 + tid - t * rnx, x1 = olo1 + t % rny, x2 = olo2 + t / rny;
      hasrow = (own >> (lcls(x0, P) + 3 * lcls(x1, P) + 9 * lcls(x2, P))) & 1;
      if (hasrow) {
        px = pbase + x0 + PB * (x1 + PB * x2);
        const int64_t r = (int64_t)XG[px] - A.row_begin;
        out = __ldg(A.row_ptr + r);
        nrw = (int)(__ldg(A.row_ptr + r + 1) - out);
        const uint4 *pp = reinterpret_cast<const uint4 *>(A.pos + r * 8);
        const uint4 pa = __ldcs(pp), pv = __ldcs(pp + 1);
        pw[0] = pa.x; pw[1] = pa.y; pw[2] = pa.z; pw[3] = pa.w;
        pw[4] = pv.x; pw[5] = pv.y; pw[6] = pv.z; pw[7] = pv.w;
#pragma unroll
        for (int jj = 0; jj < 27; ++jj) acc[jj] = 0.0;
        const int u0 = x0 - clo0, u1 = x1 - clo1, u2 = x2 - clo2;
#pragma unroll
        for (int o = 0; o < 8; ++o) {
          const int ox = o & 1, oy = (o >> 1) & 1, oz = (o >> 2) & 1;
          const int cx = u0 - ox, cy = u1 - oy, cz = u2 - oz;
          if (cx < 0 || cx >= ex0 || cy < 0 || cy >= ex1 || cz < 0 || cz >= ex2) continue;
          const double *ce = cm + (int)s_inv[cz * LAY + cy * NB + cx] * CP;
#pragma unroll
          for (int jc = 0; jc < 8; ++jc) {
            if (body_diag(o, jc)) continue;
            const int dx = (jc & 1) - ox, dy = ((jc >> 1) & 1) - oy, dz = ((jc >> 2) & 1) - oz;
            acc[(dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)] += ce[cidx(o, jc)];
          }
          asm volatile("" ::: "memory");
        }
      }
    }
    __syncthreads();  // every row has read the cells: stage over the cell storage
    double *stage_v = cm;
    uint16_t *stage_p = reinterpret_cast<uint16_t *>(cm + CF::MAXROW * 27);
    if (hasrow) {
      const int so = tid * 27;
#pragma unroll
      for (int jj = 0; jj < 27; ++jj) {
        const int ps = (int)((pw[jj >> 2] >> (8 * (jj & 3))) & 255u);
        if (ps != 255) {
          stage_v[so + ps] = acc[jj];
          stage_p[so + ps] = (uint16_t)(px + (jj % 3 - 1) + PB * ((jj / 3) % 3 - 1) + PB * PB * (jj / 9 - 1));
        }
      }
    }
    if (tid < CF::MAXROW) {
      m_out[tid] = hasrow ? out : -1;
      m_n[tid] = hasrow ? nrw : 0;
    }
    __syncthreads();
    for (int t = warp; t < nrow; t += 8) {
      const int t2 = t + 4;
      const int64_t o = m_out[t], o2 = t2 < nrow ? m_out[t2] : -1;
      const int n = m_n[t], n2 = t2 < nrow ? m_n[t2] : 0;
      const bool w1 = o >= 0 && lane < n, w2 = o2 >= 0 && lane < n2;
      int32_t c1 = 0, c2 = 0;
      double v1 = 0.0, v2 = 0.0;
      if (w1) { c1 = XG[stage_p[t * 27 + lane]]; v1 = stage_v[t * 27 + lane]; }
      if (w2) { c2 = XG[stage_p[t2 * 27 + lane]]; v2 = stage_v[t2 * 27 + lane]; }
      if (w1) {
        if (WCOL) __stcs(A.col + o + lane, c1);
        __stcs(A.val + o + lane, v1);
      }
      if (w2) {
        if (WCOL) __stcs(A.col + o2 + lane, c2);
        __stcs(A.val + o2 + lane, v2);
      }
    }
    hw = hwn;
    el = eln;
  }
}

// ============================================================================== launchers
// Proper edge colouring of the bipartite multigraph (L[i], R[i]) (classes < 16) with `colors`
// colours (Koenig: possible when no class has more than `colors` edges), by alternating-path
// recolouring.  Used to give every half-warp (one colour) cells with distinct bank residues.
static bool konig16(int n, const int *L, const int *R, int colors, int *col) {
  int atL[16][8], atR[16][8];
  if (colors > 8) return false;
  for (int a = 0; a < 16; ++a)
    for (int k = 0; k < 8; ++k) atL[a][k] = atR[a][k] = -1;
  int path[256];
  for (int i = 0; i < n; ++i) {
    const int u = L[i], v = R[i];
    int a = -1, b = -1;
    for (int k = 0; k < colors && a < 0; ++k)
      if (atL[u][k] < 0) a = k;
    for (int k = 0; k < colors && b < 0; ++k)
      if (atR[v][k] < 0) b = k;
    if (a < 0 || b < 0) return false;
    if (a != b && atR[v][a] >= 0) {  // flip the a/b path that starts at v with its a-edge
      int np = 0, node = v, k = a;
      bool right = true;
      for (;;) {
        const int e = right ? atR[node][k] : atL[node][k];
        if (e < 0 || np >= 256) break;
        path[np++] = e;
        node = right ? L[e] : R[e];
        right = !right;
        k = (k == a) ? b : a;
      }
      for (int q = 0; q < np; ++q) { atL[L[path[q]]][col[path[q]]] = -1; atR[R[path[q]]][col[path[q]]] = -1; }
      for (int q = 0; q < np; ++q) {
        col[path[q]] = (col[path[q]] == a) ? b : a;
        atL[L[path[q]]][col[path[q]]] = path[q];
        atR[R[path[q]]][col[path[q]]] = path[q];
      }
    }
    col[i] = a;
    atL[u][a] = i;
    atR[v][a] = i;
  }
  return true;
}

template <int P>
static cudaError_t xh1_setup_p(const XSetupArgs &a, cudaStream_t st) {
  if (a.nel_local <= 0) return cudaSuccess;
  if (a.nb == P + 1) k_xh1_setup<P, P + 1><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
  else k_xh1_setup<P, P + 2><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
  return cudaGetLastError();
}

// thread -> cell permutation of the one-chunk / ring cell phases (cached per instantiation)
template <int P, int NB>
static void cell_perm(uint8_t *perm_out, uint8_t *inv_out) {
  using CF = XCfg<P, NB>;
  // one chunk: thread -> cell permutation.  The 64-bit E-vector loads of a half-warp are conflict
  // free when its 16 cells have distinct (ux + XR uy + XS uz) mod 16: the i-th cell of every residue
  // class goes to half-warp i.  Used when every class has NB^3/16 rounded down or up members, so
  // that the cells occupy threads (= storage slots) 0 .. NB^3-1; identity otherwise.
  static bool pinit = false;
  static uint8_t perm[128], inv[128];
  if (!pinit) {
    constexpr int N3 = NB * NB * NB;
    int cls[16][16], ncls[16] = {0};
    bool ok = CF::ONE && N3 <= 128;
    for (int c = 0; c < N3 && ok; ++c) {
      const int r = (c % NB + CF::XR * ((c / NB) % NB) + CF::XS * (c / (NB * NB))) % 16;
      if (ncls[r] >= 16) ok = false;
      else cls[r][ncls[r]++] = c;
    }
    int lo = 128, hi = 0;
    for (int r = 0; r < 16; ++r) { lo = ncls[r] < lo ? ncls[r] : lo; hi = ncls[r] > hi ? ncls[r] : hi; }
    ok = ok && hi - lo <= 1 && hi <= 8;
    for (int t = 0; t < 128; ++t) { perm[t] = (uint8_t)(t < N3 ? t : 255); inv[t] = (uint8_t)t; }
    // the 5^3 box of p = 4 (C2): the schedule of scripts/gen_cell_schedule.py, which also makes the
    // row gather of interior elements conflict free (4 x 4 cell windows on distinct banks)
    static const uint8_t k545[128] = {31, 6, 32, 33, 36, 40, 2, 23, 9, 10, 19, 26, 13, 16, 17, 39, 20, 45, 7, 8, 11, 44, 37, 3, 41, 14, 15, 12, 27, 28, 34, 18, 24, 82, 70, 75, 61, 85, 90, 52, 5, 55, 43, 65, 96, 66, 78, 35, 0, 49, 50, 79, 120, 21, 94, 38, 53, 59, 60, 69, 63, 77, 30, 68, 56, 25, 54, 58, 100, 1, 71, 72, 73, 103, 109, 46, 47, 116, 67, 255, 106, 107, 83, 99, 86, 62, 22, 101, 122, 91, 92, 93, 76, 97, 117, 84, 4, 57, 108, 95, 104, 112, 51, 121, 88, 123, 105, 114, 115, 48, 255, 80, 81, 29, 74, 111, 124, 89, 113, 87, 102, 42, 64, 110, 119, 255, 98, 118};
    if (!CF::ONE && NB * NB <= 128) {
      // ring: per layer, the cells of a half-warp read distinct E-vector banks (ux + XR uy) and
      // write distinct cell-storage banks (slot = uy NB + ux, pitch CP = 3 mod 16)
      constexpr int N2 = NB * NB;
      int Lc[128], Rc[128], col[128];
      for (int c = 0; c < N2; ++c) {
        Lc[c] = (c % NB + CF::XR * (c / NB)) % 16;
        Rc[c] = (c * (CF::CP % 16)) % 16;
      }
      for (int t = 0; t < 128; ++t) perm[t] = 255;
      if (konig16(N2, Lc, Rc, 8, col)) {
        int fill[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int c = 0; c < N2; ++c) perm[16 * col[c] + fill[col[c]]++] = (uint8_t)c;
      } else {
        for (int t = 0; t < 128; ++t) perm[t] = (uint8_t)(t < N2 ? t : 255);
      }
    } else if (P == 4 && NB == 5 && CF::XR == 7 && CF::XS == 43) {
      for (int q = 0; q < 128; ++q) perm[q] = k545[q];
      for (int q = 0; q < 128; ++q)
        if (perm[q] != 255) inv[perm[q]] = (uint8_t)q;
    } else if (ok) {
      int t = 0;
      for (int i = 0; i < hi; ++i)
        for (int r = 0; r < 16; ++r)
          if (i < ncls[r]) perm[t++] = (uint8_t)cls[r][i];
      for (int q = t; q < 128; ++q) perm[q] = 255;
      for (int q = 0; q < t; ++q) inv[perm[q]] = (uint8_t)q;
    }
    pinit = true;
  }
  memcpy(perm_out, perm, 128);
  memcpy(inv_out, inv, 128);
}

template <int P, int NB>
static cudaError_t xh1_fill_pers(const XFillArgs &a, cudaStream_t st) {
  using PC = XPCfg<P, NB>;
  constexpr int smem = PC::SMEM;
  constexpr int MINB = (smem + 1024) * 4 <= 228 * 1024 ? 4 : 3;
  static int grid = 0;
  if (!grid) {
    int dev = 0, nsm = 0, occ = 0;
    for (auto k : {k_xh1_fill_pers<P, NB, MINB, false>, k_xh1_fill_pers<P, NB, MINB, true>}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_xh1_fill_pers<P, NB, MINB, true>, 128, smem);
    grid = nsm * (occ > 0 ? occ : 1);
  }
  if (a.nel_local <= 0) return cudaSuccess;
  XFillArgs b = a;
  cell_perm<P, NB>(b.cperm, b.cinv);
  const unsigned g = (unsigned)std::min<int64_t>(a.nel_local, grid);
  if (a.values_only) k_xh1_fill_pers<P, NB, MINB, false><<<g, 128, smem, st>>>(b);
  else k_xh1_fill_pers<P, NB, MINB, true><<<g, 128, smem, st>>>(b);
  return cudaGetLastError();
}

// variable coefficients: the non-persistent kernel with the coefficient boxes (one rank)
template <int P, int NB>
static cudaError_t xh1_fill_vc(const XFillArgs &a, cudaStream_t st) {
  using CF = XCfg<P, NB, 5>;
  constexpr int smem = CF::SMEM;
  constexpr int MINB = ((smem + 1024) * 5 <= 228 * 1024) ? XMINB : ((smem + 1024) * 4 <= 228 * 1024 ? 4 : 3);
  auto k = a.values_only ? k_xh1_fill<P, NB, MINB, false, true> : k_xh1_fill<P, NB, MINB, true, true>;
  static bool attr = false;
  if (!attr) {
    for (auto kk : {k_xh1_fill<P, NB, MINB, false, true>, k_xh1_fill<P, NB, MINB, true, true>}) {
      cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(kk, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    attr = true;
  }
  XFillArgs b = a;
  b.pf_dist = 0;
  cell_perm<P, NB>(b.cperm, b.cinv);
  k<<<(unsigned)a.nel_local, 128, smem, st>>>(b);
  return cudaGetLastError();
}

template <int P, int NB>
static cudaError_t xh1_fill_nb(const XFillArgs &a, cudaStream_t st, int *smem_out) {
  using CF = XCfg<P, NB>;
  constexpr int smem = CF::SMEM;
  if (smem_out) { *smem_out = smem; return cudaSuccess; }
  if (a.nel_local <= 0) return cudaSuccess;
  if (a.ca) return xh1_fill_vc<P, NB>(a, st);
  constexpr int MINB = ((smem + 1024) * 5 <= 228 * 1024) ? XMINB : 3;  // 228 KB shared memory per SM
  if constexpr (CF::ONE) {
    static int pers = -1;
    if (pers < 0) {
      const char *e = getenv("LOR_XPERS");
      pers = (e && !atoi(e)) ? 0 : 1;
    }
    if (pers) return xh1_fill_pers<P, NB>(a, st);
  }
  auto k = a.values_only ? k_xh1_fill<P, NB, MINB, false> : k_xh1_fill<P, NB, MINB, true>;
  static bool attr = false;
  if (!attr) {
    for (auto kk : {k_xh1_fill<P, NB, MINB, false>, k_xh1_fill<P, NB, MINB, true>}) {
      cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(kk, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    attr = true;
  }
  // L2 prefetch distance = resident CTAs of the grid (cached per instantiation; LOR_XPF=0: off)
  static int64_t resident = -1;
  if (resident < 0) {
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 128, smem);
    const char *e = getenv("LOR_XPF");
    resident = (e && !atoi(e)) ? 0 : (int64_t)nsm * occ;
  }
  XFillArgs b = a;
  b.pf_dist = resident;
  cell_perm<P, NB>(b.cperm, b.cinv);
  k<<<(unsigned)a.nel_local, 128, smem, st>>>(b);
  return cudaGetLastError();
}

template <int P>
static cudaError_t xh1_fill_p(const XFillArgs &a, cudaStream_t st, int *smem_out) {
  if (a.ncx <= P + 1 && a.ncy <= P + 1 && a.ncz <= P + 1) return xh1_fill_nb<P, P + 1>(a, st, smem_out);
  return xh1_fill_nb<P, P + 2>(a, st, smem_out);
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

template <int P>
static cudaError_t xh1_count_p(const XFillArgs &a, cudaStream_t st) {
  if (a.nel_local <= 0) return cudaSuccess;
  // one thread per owned row (most elements own p^3: 64 threads for p <= 4, 128 above)
  constexpr int NT = P <= 4 ? 64 : 128;
  if (a.ncx <= P + 1 && a.ncy <= P + 1 && a.ncz <= P + 1) k_xh1_sym<P, P + 1, NT><<<(unsigned)a.nel_local, NT, 0, st>>>(a);
  else k_xh1_sym<P, P + 2, NT><<<(unsigned)a.nel_local, NT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_xh1_count(int p, const XFillArgs &a, cudaStream_t st) {
  switch (p) {
    case 1: return xh1_count_p<1>(a, st);
    case 2: return xh1_count_p<2>(a, st);
    case 3: return xh1_count_p<3>(a, st);
    case 4: return xh1_count_p<4>(a, st);
    case 5: return xh1_count_p<5>(a, st);
    case 6: return xh1_count_p<6>(a, st);
    case 7: return xh1_count_p<7>(a, st);
    case 8: return xh1_count_p<8>(a, st);
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
