// lor_xv.cuh -- extended-frame ("owner computes") assembly of the vector spaces: H(curl) Nedelec
// (SP_ND) and H(div) Raviart-Thomas (SP_RT) LOR matrices under the vertex rule, one pass, no
// partial rows and no merge pass (DESIGN.md §4 "k_xv").
//
// Every element writes the complete CSR rows of the dofs it owns (the minimal element containing
// the dof's coarse entity); the LOR cells of the neighbouring elements that
// touch those rows are recomputed in the owner's lattice frame extended by one cell layer (the
// frame, neighbourhood records and coordinate gather lists are those of the H1 path, lor_xframe.h).
// Per space three kernels:
//   k_xv_setup  once: the extended element restriction of the three dof families (global id and
//               orientation sign of every edge / face of the element's box, in the owner's frame);
//   k_xv_sym    per call (A2): length of every owned row and the final
//               position of each stencil slot in the ascending-column row (reading P-5);
//   k_xv_fill   per call (A1 + A2): per z-layer of rows the packed cell matrices of the cells the
//               layer needs (two resident cell layers), one thread per row summing the rows of the
//               <= 4 (ND) / 2 (RT) cells containing it, signs applied, staged in final order,
//               written out coalesced.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "lor_cells.cuh"
#include "lor_device.cuh"
#include "lor_xdev.cuh"
#include "lor_xframe.h"

#ifndef XV_PF_ROWS
#define XV_PF_ROWS 0  // k_xv_fill: L2 prefetch of the next-residency CTA's row pointers / positions
#endif
#ifndef XV_RT_GZ
#define XV_RT_GZ(P) ((P) + 1)  // RT with resident cells: row layers per group (all of them)
#endif
#ifndef XV_ND_ONE_KB
#define XV_ND_ONE_KB 80  // ND: all cell layers resident up to this size (p <= 4: 78 KB, 2 CTAs/SM)
#endif

namespace lorb {

using namespace xdev;

namespace {

template <int SP>
struct XvT;
template <>
struct XvT<SP_ND> {
  static constexpr int W = 33, NE = 78, PW = 12;  // stencil width, packed cell entries, position words stored
};
template <>
struct XvT<SP_RT> {
  static constexpr int W = 11, NE = 21, PW = 4;
};

template <int P, int NB, int SP, int NCOMP = 3>  // NCOMP = 5: + coefficient boxes a, b (NEXT-3)
struct XvCfg {
  static constexpr int PB = NB + 1, NPB = PB * PB * PB, LAY = NB * NB;
  static constexpr int NVF = SP == SP_ND ? NB * PB * PB : PB * NB * NB;  // box positions per family
  // rows of one z-layer: family 2 first, then families 0 and 1
  static constexpr int NRF2 = SP == SP_ND ? (P + 1) * (P + 1) : P * P;
  static constexpr int NRF0 = P * (P + 1);
  static constexpr int MAXR = NRF2 + 2 * NRF0;                    // rows of one z-layer
  static constexpr int W = XvT<SP>::W, NE = XvT<SP>::NE, PW = XvT<SP>::PW;
  static constexpr int NCP = LAY | 1;  // cells per entry plane (odd pitch)
  // all cell layers resident when they fit next to the rest (then every cell is computed in one
  // phase by all threads), else a ring of the two layers a row layer needs
  static constexpr bool ONE = NB * NE * NCP * 8 <= (SP == SP_ND ? XV_ND_ONE_KB : 40) * 1024;
  // rows processed per group of GZ z-layers: all of them at once for RT with resident cells (short
  // rows: per-layer barriers would dominate), one layer otherwise
  static constexpr int GZ = (ONE && SP == SP_RT) ? XV_RT_GZ(P) : 1;
  // rows of a group in family-major segments, each starting at a warp boundary (a warp then runs
  // one family's code: no divergence between the families' unrolled row kernels)
  static constexpr int NF2 = GZ * NRF2, NF0 = GZ * NRF0;
  static constexpr int B0 = (NF2 + 31) / 32 * 32, B1 = B0 + (NF0 + 31) / 32 * 32;
  static constexpr int MAXG = B1 + NF0;
  static constexpr int RPT = (MAXG + 127) / 128;
  static constexpr int NSLOT = ONE ? NB : 2;
  static constexpr int OFF_CM = NCOMP * NPB * 8;                   // E-vector box [3][NPB] (+ a, b)
  static constexpr int OFF_ST = OFF_CM + NSLOT * NE * NCP * 8;     // cell layers [NSLOT][NE][NCP]
  static constexpr int NROWS = NF2 + 2 * NF0;                      // rows of a group (staging capacity)
  static constexpr int OFF_SC = OFF_ST + NROWS * W * 8;            // staged values [NROWS][W]
  static constexpr int OFF_XV = OFF_SC + NROWS * W * 4;            // staged columns [NROWS][W]
  static constexpr int OFF_MO = (OFF_XV + 3 * NVF * 4 + 15) / 16 * 16;  // restriction [3][NVF]
  static constexpr int OFF_WE = (OFF_MO + 16 * RPT + 15) / 16 * 16;  // write-out: per warp 32 row ends
  static constexpr int OFF_WD = OFF_WE + 4 * 32 * 4;                 //   and 32 destination offsets
  static constexpr int SMEM = OFF_WD + 4 * 32 * 8;
};

// extent of family s along axis a in the box (cell-index axes: NB, point-index axes: NB + 1)
template <int SP>
__host__ __device__ constexpr bool ptk(int s, int a) { return vkind<SP>(s, a); }
template <int SP, int NB>
__host__ __device__ constexpr int fext(int s, int a) { return ptk<SP>(s, a) ? NB + 1 : NB; }
template <int SP, int NB>
__device__ __forceinline__ int fidx(int s, const int u[3]) {
  return u[0] + fext<SP, NB>(s, 0) * (u[1] + fext<SP, NB>(s, 1) * u[2]);
}

// natural stencil slot k of a row of family s (lor_device.cuh st_*): column family and offset
template <int SP>
__host__ __device__ constexpr int slot_s2(int s, int k) {
  int s2 = 0;
  while (k >= st_n<3, SP>(s, s2)) { k -= st_n<3, SP>(s, s2); ++s2; }
  return s2;
}
template <int SP>
__host__ __device__ constexpr int slot_d(int s, int k, int a) {
  int s2 = 0;
  while (k >= st_n<3, SP>(s, s2)) { k -= st_n<3, SP>(s, s2); ++s2; }
  const int nx = st_hi<SP>(s, s2, 0) - st_lo<SP>(s, s2, 0) + 1, ny = st_hi<SP>(s, s2, 1) - st_lo<SP>(s, s2, 1) + 1;
  const int i = a == 0 ? k % nx : (a == 1 ? (k / nx) % ny : k / (nx * ny));
  return i + st_lo<SP>(s, s2, a);
}

// row of layer z, flat index t -> family s and extended-frame (= element-local) position x; false if
// t is not a dof of this layer
template <int P, int SP>
__device__ __forceinline__ bool layer_row(int z, int t, int &s, int x[3]) {
  constexpr int NRF2 = SP == SP_ND ? (P + 1) * (P + 1) : P * P, NRF0 = P * (P + 1);
  if (t < NRF2) {
    s = 2;
    const int n = SP == SP_ND ? P + 1 : P;
    x[0] = t % n;
    x[1] = t / n;
    x[2] = z;
    return SP == SP_ND ? z < P : true;
  }
  t -= NRF2;
  if (t < NRF0) {
    s = 0;
    const int n0 = SP == SP_ND ? P : P + 1;
    x[0] = t % n0;
    x[1] = t / n0;
    x[2] = z;
    return SP == SP_ND ? true : z < P;
  }
  t -= NRF0;
  if (t >= NRF0) return false;
  s = 1;
  const int n0 = SP == SP_ND ? P + 1 : P;
  x[0] = t % n0;
  x[1] = t / n0;
  x[2] = z;
  return SP == SP_ND ? true : z < P;
}

// row t of the group of GZ layers starting at z0 (family-major warp-aligned segments, see XvCfg)
template <int P, int SP, int GZ, int B0, int B1, int NF2, int NF0>
__device__ __forceinline__ bool group_row(int z0, int t, int &s, int x[3]) {
  constexpr int NRF2 = SP == SP_ND ? (P + 1) * (P + 1) : P * P, NRF0 = P * (P + 1);
  int k, nr;
  if (t < B0) {
    if (t >= NF2) return false;
    k = t;
    nr = NRF2;
    s = 2;
  } else if (t < B1) {
    k = t - B0;
    if (k >= NF0) return false;
    nr = NRF0;
    s = 0;
  } else {
    k = t - B1;
    if (k >= NF0) return false;
    nr = NRF0;
    s = 1;
  }
  const int z = z0 + k / nr, kk = k % nr;
  if (z > P) return false;
  const int tt = s == 2 ? kk : (s == 0 ? NRF2 + kk : NRF2 + NRF0 + kk);
  return layer_row<P, SP>(z, tt, s, x);
}

// coarse entity slot (element-local classes) of the dof of family s at x
template <int P, int SP>
__device__ __forceinline__ int dof_tau(int s, const int x[3]) {
  int t = 0, m = 1;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    t += m * (ptk<SP>(s, a) ? lcls(x[a], P) : 1);
    m *= 3;
  }
  return t;
}

// is stencil slot k (column family s2, offset d) of the row (s, x) a column: some cell of the box
// [clo, chi] contains both dofs (per axis: cells [x-1, x] along point-index axes, [x, x] along
// cell-index axes)
template <int SP, int S, int K>
struct SlotC {  // compile-time description of stencil slot K of a row of family S
  static constexpr int s2 = slot_s2<SP>(S, K);
  static constexpr int d0 = slot_d<SP>(S, K, 0), d1 = slot_d<SP>(S, K, 1), d2 = slot_d<SP>(S, K, 2);
};
template <int SP, int S, int S2, int A, int D>
__device__ __forceinline__ bool axis_ok(int x, int clo, int chi) {
  const int y = x + D;
  int lo = ptk<SP>(S, A) ? x - 1 : x, hi = x;
  const int lo2 = ptk<SP>(S2, A) ? y - 1 : y;
  lo = lo > lo2 ? lo : lo2;
  hi = hi < y ? hi : y;
  lo = lo > clo ? lo : clo;
  hi = hi < chi ? hi : chi;
  return lo <= hi;
}
template <int SP, int S, int K>
__device__ __forceinline__ bool slot_valid(const int x[3], const int clo[3], const int chi[3]) {
  using C = SlotC<SP, S, K>;
  return axis_ok<SP, S, C::s2, 0, C::d0>(x[0], clo[0], chi[0]) && axis_ok<SP, S, C::s2, 1, C::d1>(x[1], clo[1], chi[1]) &&
         axis_ok<SP, S, C::s2, 2, C::d2>(x[2], clo[2], chi[2]);
}

// keys of the row's slots: the global ids (absent: 0x7fffffff), and whether the slot is present
template <int P, int NB, int SP, int S, int... K>
__device__ __forceinline__ void slot_keys(const int x[3], const int clo[3], const int chi[3], const uint32_t *XV,
                                          int kb, int (&key)[XvT<SP>::W], std::integer_sequence<int, K...>) {
  constexpr int NVF = XvCfg<P, NB, SP>::NVF;
  auto one = [&](auto kc) {
    constexpr int k = decltype(kc)::value;
    using C = SlotC<SP, S, k>;
    if (slot_valid<SP, S, k>(x, clo, chi)) {
      const int u[3] = {x[0] + C::d0 - clo[0], x[1] + C::d1 - clo[1], x[2] + C::d2 - clo[2]};
      key[k] = (int)(XV[C::s2 * NVF + fidx<SP, NB>(C::s2, u)] & 0x7fffffffu) - kb;
    } else {
      key[k] = 0x7fffffff;
    }
  };
  (one(std::integral_constant<int, K>{}), ...);
}

// ------------------------------------------------------------------------------ setup kernel
// Extended element restriction: for every dof position of the three families in the box, the
// element that holds it (the neighbour containing the dof's midpoint), the dof's coordinates in that
// element's local frame (lor_xframe.h XNbr::code), its global id from that element's affine block
// (App. A numbering, lor_device.cuh block_affine) and its sign in the owner's frame (the block's
// orientation sign times the direction of the owner's +axis in the holder's frame).
template <int P, int NB, int SP>
__global__ void __launch_bounds__(128) k_xv_setup(XvArgs A) {
  using CF = XvCfg<P, NB, SP>;
  const int64_t bs = blockIdx.x;
  if (bs >= A.nel_local) return;
  __shared__ XElem H;
  {
    const int4 *src = reinterpret_cast<const int4 *>(A.xe + bs);
    int4 *dst = reinterpret_cast<int4 *>(&H);
    for (int i = threadIdx.x; i < (int)(sizeof(XElem) / 16); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const uint32_t ident = 0u | (1u << 2) | (2u << 4) | (1u << 9) | (1u << 11) | (1u << 13);
  for (int i = threadIdx.x; i < 3 * CF::NVF; i += blockDim.x) {
    const int s = i / CF::NVF, l = i % CF::NVF;
    const int e0 = fext<SP, NB>(s, 0), e1 = fext<SP, NB>(s, 1);
    const int u[3] = {l % e0, (l / e0) % e1, l / (e0 * e1)};
    int y[3];
    bool in = true;
    for (int a = 0; a < 3; ++a) {
      y[a] = H.clo[a] + u[a];
      const int hi = ptk<SP>(s, a) ? H.chi[a] + 1 : H.chi[a];
      in = in && y[a] <= hi;
    }
    uint32_t out = 0xffffffffu;
    if (in) {
      // the element holding the dof: the one containing its midpoint
      int ni = 0, m = 1;
      for (int a = 0; a < 3; ++a) {
        const int d = ptk<SP>(s, a) ? ydelta(y[a], P) : (y[a] < 0 ? -1 : (y[a] >= P ? 1 : 0));
        ni += m * (d + 1);
        m *= 3;
      }
      int64_t f = -1;
      uint32_t code = ident;
      if (ni == 13) f = H.el;
      else {
        f = H.nbr[ni].el;
        code = H.nbr[ni].code;
      }
      if (f >= 0) {
        int L0[3], L1[3], L2[3], L3[3], xl[3], sl = -1, sn = 1;
        x_to_local(P, code, y, L0);
        if (SP == SP_ND) {  // edge [y, y + e_s]
          int y1[3] = {y[0], y[1], y[2]};
          y1[s] += 1;
          x_to_local(P, code, y1, L1);
          for (int a = 0; a < 3; ++a) {
            xl[a] = L0[a] < L1[a] ? L0[a] : L1[a];
            if (L0[a] != L1[a]) { sl = a; sn = L1[a] > L0[a] ? 1 : -1; }
          }
        } else {  // face normal s through y: in-face corners y + e_u, y + e_v; y + e_s off the face
          const int uu = s == 0 ? 1 : 0, vv = s == 2 ? 1 : 2;
          int yu[3] = {y[0], y[1], y[2]}, yv[3] = {y[0], y[1], y[2]}, ys[3] = {y[0], y[1], y[2]};
          yu[uu] += 1;
          yv[vv] += 1;
          ys[s] += 1;
          x_to_local(P, code, yu, L1);
          x_to_local(P, code, yv, L2);
          x_to_local(P, code, ys, L3);
          for (int a = 0; a < 3; ++a) {
            int mn = L0[a] < L1[a] ? L0[a] : L1[a];
            mn = mn < L2[a] ? mn : L2[a];
            xl[a] = mn;
            if (L0[a] == L1[a] && L0[a] == L2[a]) { sl = a; sn = L3[a] > L0[a] ? 1 : -1; xl[a] = L0[a]; }
          }
        }
        int tau = 0, mm = 1;
        for (int a = 0; a < 3; ++a) {
          tau += mm * (ptk<SP>(sl, a) ? lcls(xl[a], P) : 1);
          mm *= 3;
        }
        Blk B;
        block_affine<3, SP>(P, sl, tau, A.topo[f], A.base, B);
        if (sl < 0 || B.size <= 0) {
          atomicExch(A.err, 1);
        } else {
          const int g = B.g0 + B.str[0] * xl[0] + B.str[1] * xl[1] + B.str[2] * xl[2];
          out = (uint32_t)g | ((B.sigma * sn) < 0 ? 0x80000000u : 0u);
        }
      }
    }
    A.xvmap[bs * 3 * CF::NVF + i] = out;
  }
}

// ------------------------------------------------------------------------------ symbolic pass
template <int P, int NB, int SP, int S>
__device__ __forceinline__ void sym_row(const XvArgs &A, const int x[3], const int clo[3], const int chi[3],
                                        const uint32_t *XV, uint8_t *scratch) {
  using CF = XvCfg<P, NB, SP>;
  constexpr int W = CF::W;
  int key[W];
  slot_keys<P, NB, SP, S>(x, clo, chi, XV, A.key_base, key, std::make_integer_sequence<int, W>{});
  const int u[3] = {x[0] - clo[0], x[1] - clo[1], x[2] - clo[2]};
  const int64_t r = (int64_t)(XV[S * CF::NVF + fidx<SP, NB>(S, u)] & 0x7fffffffu) - A.row_begin;
  int n = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) n += key[k] != 0x7fffffff;
  A.cnt[r] = n;
  uint32_t pw[(W + 3) / 4];
  row_positions<W>(key, A.sort32 != 0, scratch, pw);
  uint32_t *dst = A.pos + r * CF::PW;
#pragma unroll
  for (int q = 0; q < CF::PW; q += 4) {
    uint4 v;
    v.x = q < (W + 3) / 4 ? pw[q] : 0xffffffffu;
    v.y = q + 1 < (W + 3) / 4 ? pw[q + 1] : 0xffffffffu;
    v.z = q + 2 < (W + 3) / 4 ? pw[q + 2] : 0xffffffffu;
    v.w = q + 3 < (W + 3) / 4 ? pw[q + 3] : 0xffffffffu;
    reinterpret_cast<uint4 *>(dst)[q / 4] = v;
  }
}

template <int P, int NB, int SP>
__global__ void __launch_bounds__(128) k_xv_sym(XvArgs A) {
  using CF = XvCfg<P, NB, SP>;
  __shared__ uint32_t XV[3 * CF::NVF];
  __shared__ __align__(16) uint8_t s_pos[128 * 36];
  const int tid = threadIdx.x;
  const int64_t bs = blockIdx.x;
  if (bs >= A.nel_local) return;
  const int4 hw = __ldg(reinterpret_cast<const int4 *>(A.xe + bs));
  for (int i = tid; i < 3 * CF::NVF; i += 128) XV[i] = __ldg(A.xvmap + bs * 3 * CF::NVF + i);
  const int clo[3] = {(int8_t)(hw.y & 255), (int8_t)((hw.y >> 8) & 255), (int8_t)((hw.y >> 16) & 255)};
  const int chi[3] = {(int8_t)((hw.y >> 24) & 255), (int8_t)(hw.z & 255), (int8_t)((hw.z >> 8) & 255)};
  const uint32_t own = (uint32_t)hw.x;
  __syncthreads();
  // the element's OWNED rows, compacted per family (about 2/3 of its dofs), then processed in
  // family-major warp-aligned segments (no divergence between the families' unrolled code paths
  // within a warp, no lanes spent on rows other elements own)
  constexpr int NRF2 = CF::NRF2, NRF0 = CF::NRF0;
  constexpr int NF2 = (P + 1) * NRF2, NF0 = (P + 1) * NRF0;
  constexpr int B0 = (NF2 + 31) / 32 * 32, B1 = B0 + (NF0 + 31) / 32 * 32, NT = B1 + NF0;
  __shared__ uint16_t s_list[3][NF2 > NF0 ? NF2 : NF0];
  __shared__ int s_nf[3];
  if (tid < 3) s_nf[tid] = 0;
  __syncthreads();
  for (int i0 = 0; i0 < NT; i0 += 128) {
    const int i = i0 + tid;
    int s = -1, x[3];
    const bool ok = i < NT && group_row<P, SP, P + 1, B0, B1, NF2, NF0>(0, i, s, x) && ((own >> dof_tau<P, SP>(s, x)) & 1);
    // segments are warp-aligned per family: a warp's slots belong to one family
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    int base = 0;
    const int fam = __shfl_sync(0xffffffffu, s, __ffs(m | 0x80000000u) - 1);
    if ((tid & 31) == 0 && m) base = atomicAdd(&s_nf[fam], __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (ok) s_list[s][base + __popc(m & ((1u << (tid & 31)) - 1u))] = (uint16_t)i;
  }
  __syncthreads();
  const int n2 = s_nf[2], n0 = s_nf[0], n1 = s_nf[1];
  const int c0 = (n2 + 31) / 32 * 32, c1 = c0 + (n0 + 31) / 32 * 32, ct = c1 + n1;
  for (int t = tid; t < ct; t += 128) {
    int fam, k;
    if (t < c0) { fam = 2; k = t; if (k >= n2) continue; }
    else if (t < c1) { fam = 0; k = t - c0; if (k >= n0) continue; }
    else { fam = 1; k = t - c1; }
    int s, x[3];
    group_row<P, SP, P + 1, B0, B1, NF2, NF0>(0, s_list[fam][k], s, x);
    if (s == 0) sym_row<P, NB, SP, 0>(A, x, clo, chi, XV, s_pos + tid * 36);
    else if (s == 1) sym_row<P, NB, SP, 1>(A, x, clo, chi, XV, s_pos + tid * 36);
    else sym_row<P, NB, SP, 2>(A, x, clo, chi, XV, s_pos + tid * 36);
  }
}

// ------------------------------------------------------------------------------ fill kernel
// RT vertex rule straight into the cell's packed slots out[t * NC]: mass M[F_d(q)][F_e(q)] +=
// w beta (J^T J / det)_de at corner q, div-div (sum_q w alpha / det_q) d d^T (lor_cells.cuh cell_rt)
template <typename XF>
__device__ __forceinline__ bool cell_rt_vertex_to(XF X, double alpha, double beta, double *__restrict__ out, int NC,
                                                  const double *ca = nullptr, const double *cb = nullptr) {
  double M[21];
#pragma unroll
  for (int i = 0; i < 21; ++i) M[i] = 0.0;
  const double w = 0.125;
  double sdiv = 0.0;
  bool ok = true;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    Jac3 J;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int hi = q | (1 << d), lo = q & ~(1 << d);
#pragma unroll
      for (int k = 0; k < 3; ++k) J.j[d][k] = X(hi, k) - X(lo, k);
    }
    const double det = J.j[0][0] * (J.j[1][1] * J.j[2][2] - J.j[1][2] * J.j[2][1]) +
                       J.j[0][1] * (J.j[1][2] * J.j[2][0] - J.j[1][0] * J.j[2][2]) +
                       J.j[0][2] * (J.j[1][0] * J.j[2][1] - J.j[1][1] * J.j[2][0]);
    ok = ok && det > 0.0;
    const double rd = rcp_pos(det), sm = w * beta * coef_q<0, 8>(cb, q) * rd;
    sdiv += w * alpha * coef_q<0, 8>(ca, q) * rd;
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int e = d; e < 3; ++e) M[tri(6, 2 * d + ((q >> d) & 1), 2 * e + ((q >> e) & 1))] += sm * dot3(J.j[d], J.j[e]);
  }
#pragma unroll
  for (int f = 0; f < 6; ++f)
#pragma unroll
    for (int g = f; g < 6; ++g) out[tri(6, f, g) * NC] = M[tri(6, f, g)] + sdiv * (double)(((f & 1) ? 1 : -1) * ((g & 1) ? 1 : -1));
  return ok;
}

// ND: the cells containing edge (S, x): c_S = x_S, c_u = x_u - b1, c_v = x_v - b2 (u < v the other
// axes); the row is the cell's edge 4S + b1 + 2 b2 and cell edge eps = 4a + j1 + 2 j2 sits at offset
// (c + j1 e_u(a) + j2 e_v(a)) - x.  RT: cells c_S = x_S - 1 + o... (o = 1: the row is side 1 of cell
// x_S - 1; o = 0: side 0 of cell x_S), cell face 2a + side at (c + side e_a) - x.
template <int SP, int S, int O, int J>
__host__ __device__ constexpr int gather_slot() {
  if (SP == SP_ND) {
    const int u = S == 0 ? 1 : 0, v = S == 2 ? 1 : 2;
    const int b1 = O & 1, b2 = O >> 1;
    int c[3] = {0, 0, 0};  // cell relative to x
    c[u] = -b1;
    c[v] = -b2;
    const int a = J / 4, j1 = J & 1, j2 = (J >> 1) & 1;
    const int ua = a == 0 ? 1 : 0, va = a == 2 ? 1 : 2;
    int d[3] = {c[0], c[1], c[2]};
    d[ua] += j1;
    d[va] += j2;
    return st_slot<3, SP_ND>(S, a, d[0], d[1], d[2]);
  } else {
    int c[3] = {0, 0, 0};
    c[S] = O == 1 ? -1 : 0;
    const int a = J / 2, side = J & 1;
    int d[3] = {c[0], c[1], c[2]};
    d[a] += side;
    return st_slot<3, SP_RT>(S, a, d[0], d[1], d[2]);
  }
}
template <int SP, int S, int O>
__host__ __device__ constexpr int row_local() {
  if (SP == SP_ND) return 4 * S + (O & 1) + 2 * (O >> 1);
  return 2 * S + O;
}

template <int P, int NB, int SP, int S, int O, int... J>
__device__ __forceinline__ void gather_cell(const double *__restrict__ ce, int NC, double (&acc)[XvT<SP>::W],
                                            std::integer_sequence<int, J...>) {
  constexpr int NL = SP == SP_ND ? 12 : 6;
  constexpr int i = row_local<SP, S, O>();
  ((acc[std::integral_constant<int, gather_slot<SP, S, O, J>()>::value] +=
    ce[std::integral_constant<int, tri(NL, i, J)>::value * NC]), ...);
}

template <int P, int NB, int SP, int S, int... O>
__device__ __forceinline__ void gather_row(const int x[3], const int clo[3], const int ex[3], const double *cm, int cz0,
                                           double (&acc)[XvT<SP>::W], std::integer_sequence<int, O...>) {
  using CF = XvCfg<P, NB, SP>;
  auto one = [&](auto oc) {
    constexpr int o = decltype(oc)::value;
    int c[3] = {x[0], x[1], x[2]};
    if (SP == SP_ND) {
      constexpr int u = S == 0 ? 1 : 0, v = S == 2 ? 1 : 2;
      c[u] -= o & 1;
      c[v] -= o >> 1;
    } else {
      c[S] -= o;
    }
    const int b0 = c[0] - clo[0], b1 = c[1] - clo[1], b2 = c[2] - clo[2];
    if (b0 < 0 || b0 >= ex[0] || b1 < 0 || b1 >= ex[1] || b2 < 0 || b2 >= ex[2]) return;
    const int slot = CF::ONE ? b2 : ((c[2] % 2) + 2) % 2;
    const double *ce = cm + slot * CF::NE * CF::NCP + b0 + NB * b1;
    gather_cell<P, NB, SP, S, o>(ce, CF::NCP, acc, std::make_integer_sequence<int, SP == SP_ND ? 12 : 6>{});
    asm volatile("" ::: "memory");
  };
  (one(std::integral_constant<int, O>{}), ...);
  (void)cz0;
}

template <int P, int NB, int SP, int S, int... K>
__device__ __forceinline__ void stage_row(const int x[3], const int clo[3], const uint32_t *XV, bool srow,
                                          const uint32_t *pw, double (&acc)[XvT<SP>::W], double *sv, int32_t *sc,
                                          std::integer_sequence<int, K...>) {
  using CF = XvCfg<P, NB, SP>;
  auto one = [&](auto kc) {
    constexpr int k = decltype(kc)::value;
    using C = SlotC<SP, S, k>;
    const int ps = (int)((pw[k >> 2] >> (8 * (k & 3))) & 255u);
    if (ps != 255) {
      const int u[3] = {x[0] + C::d0 - clo[0], x[1] + C::d1 - clo[1], x[2] + C::d2 - clo[2]};
      const uint32_t m = XV[C::s2 * CF::NVF + fidx<SP, NB>(C::s2, u)];
      const bool neg = srow != ((m >> 31) != 0);
      sv[ps] = neg ? -acc[k] : acc[k];
      sc[ps] = (int32_t)(m & 0x7fffffffu);
    }
  };
  (one(std::integral_constant<int, K>{}), ...);
}

template <int P, int NB, int SP, int S>
__device__ __forceinline__ void fill_row(const XvArgs &A, const int x[3], const int clo[3], const int ex[3],
                                         const double *cm, const uint32_t *XV, double *sv, int32_t *sc,
                                         const uint32_t (&pw)[XvT<SP>::PW]) {
  using CF = XvCfg<P, NB, SP>;
  constexpr int W = CF::W;
  const int u[3] = {x[0] - clo[0], x[1] - clo[1], x[2] - clo[2]};
  const uint32_t mr = XV[S * CF::NVF + fidx<SP, NB>(S, u)];
  double acc[W];
#pragma unroll
  for (int k = 0; k < W; ++k) acc[k] = 0.0;
  gather_row<P, NB, SP, S>(x, clo, ex, cm, 0, acc, std::make_integer_sequence<int, SP == SP_ND ? 4 : 2>{});
  stage_row<P, NB, SP, S>(x, clo, XV, (mr >> 31) != 0, pw, acc, sv, sc, std::make_integer_sequence<int, W>{});
}

template <int P, int NB, int SP, int MINB, bool WCOL, bool VC = false>
__global__ void __launch_bounds__(128, MINB) k_xv_fill(XvArgs A) {
  using CF = XvCfg<P, NB, SP, VC ? 5 : 3>;
  constexpr int PB = CF::PB, NPB = CF::NPB, NP1 = P + 1, NPT = NP1 * NP1 * NP1, W = CF::W, NE = CF::NE;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_bad;
  double *XE = reinterpret_cast<double *>(smem);
  double *cm = reinterpret_cast<double *>(smem + CF::OFF_CM);
  double *stv = reinterpret_cast<double *>(smem + CF::OFF_ST);
  int32_t *stc = reinterpret_cast<int32_t *>(smem + CF::OFF_SC);
  uint32_t *XV = reinterpret_cast<uint32_t *>(smem + CF::OFF_XV);
  int32_t *m_wt = reinterpret_cast<int32_t *>(smem + CF::OFF_MO);  // per (rr, warp): staged entries
  int32_t *w_end = reinterpret_cast<int32_t *>(smem + CF::OFF_WE);
  int64_t *w_dst = reinterpret_cast<int64_t *>(smem + CF::OFF_WD);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t bs = blockIdx.x;
  if (bs >= A.nel_local) return;
  const int4 hw = __ldg(reinterpret_cast<const int4 *>(A.xe + bs));
  const int64_t el = __ldg(&A.xe[bs].el);
  const int clo[3] = {(int8_t)(hw.y & 255), (int8_t)((hw.y >> 8) & 255), (int8_t)((hw.y >> 16) & 255)};
  const int chi[3] = {(int8_t)((hw.y >> 24) & 255), (int8_t)(hw.z & 255), (int8_t)((hw.z >> 8) & 255)};
  const int ex[3] = {chi[0] - clo[0] + 1, chi[1] - clo[1] + 1, chi[2] - clo[2] + 1};
  const uint32_t own = (uint32_t)hw.x;
  // next layer's rows: family, position, CSR offset, length, slot positions (registers)
  int ns[CF::RPT], nx[CF::RPT][3], nn[CF::RPT];
  int64_t nout[CF::RPT];
  uint32_t npw[CF::RPT][CF::PW];
  auto load_layer = [&](int zg) {  // rows of the group starting at layer zg
#pragma unroll
    for (int rr = 0; rr < CF::RPT; ++rr) {
      const int tg = tid + 128 * rr;
      ns[rr] = -1;
      nn[rr] = 0;
      nout[rr] = -1;
#pragma unroll
      for (int q = 0; q < CF::PW; ++q) npw[rr][q] = 0xffffffffu;
      int sf = 0, xx[3] = {0, 0, 0};
      if (tg < CF::MAXG && group_row<P, SP, CF::GZ, CF::B0, CF::B1, CF::NF2, CF::NF0>(zg, tg, sf, xx) &&
          ((own >> dof_tau<P, SP>(sf, xx)) & 1)) {
        const int u[3] = {xx[0] - clo[0], xx[1] - clo[1], xx[2] - clo[2]};
        const int idx = sf == 0 ? fidx<SP, NB>(0, u) : (sf == 1 ? fidx<SP, NB>(1, u) : fidx<SP, NB>(2, u));
        const int64_t r = (int64_t)(__ldg(A.xvmap + bs * 3 * CF::NVF + sf * CF::NVF + idx) & 0x7fffffffu) - A.row_begin;
        ns[rr] = sf;
        nout[rr] = __ldg(A.row_ptr + r);
        nn[rr] = (int)(__ldg(A.row_ptr + r + 1) - nout[rr]);
        const uint4 *pp = reinterpret_cast<const uint4 *>(A.pos + r * CF::PW);
#pragma unroll
        for (int q = 0; q < CF::PW / 4; ++q) {
          const uint4 v = __ldcs(pp + q);
          npw[rr][4 * q] = v.x; npw[rr][4 * q + 1] = v.y; npw[rr][4 * q + 2] = v.z; npw[rr][4 * q + 3] = v.w;
        }
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) nx[rr][a] = xx[a];
    }
  };
  // L2 prefetch for the CTA that takes this CTA's place one residency later: its record, extended
  // restriction and gather list now, its E-vector once its element id has arrived (as k_xh1_fill)
  {
    const int64_t nbs = bs + A.pf_dist;
    if (A.pf_dist > 0 && nbs < A.nel_local) {
      constexpr int HC2 = NPB - NPT;
      constexpr int LX = (int)((sizeof(XElem) + 127) / 128), LM = (3 * CF::NVF * 4 + 127) / 128 + 1,
                    LH = (HC2 * 8 + 127) / 128 + 1;
      if (tid < LX) pf_l2(reinterpret_cast<const char *>(A.xe + nbs) + 128 * tid);
      else if (tid < LX + LM) pf_l2(reinterpret_cast<const char *>(A.xvmap + nbs * 3 * CF::NVF) + 128 * (tid - LX));
      else if (tid < LX + LM + LH) pf_l2(reinterpret_cast<const char *>(A.xhalo + nbs * HC2) + 128 * (tid - LX - LM));
      else if (tid == 127) {
        const int64_t pe = __ldg(&A.xe[nbs].el);
        const char *xp = reinterpret_cast<const char *>(A.X + pe * A.xstride);
        for (int l = 0; l < (3 * NPT * 8 + 127) / 128; ++l) pf_l2(xp + 128 * l);
      }
    }
  }
  load_layer(0);
  {
    if (tid == 0) s_bad = 0;
    for (int i = tid; i < 3 * CF::NVF; i += 128) XV[i] = __ldg(A.xvmap + bs * 3 * CF::NVF + i);
    // own E-vector into the dense box, then the neighbour points (gather list of the H1 setup)
    const double *xs = A.X + el * A.xstride;
    for (int i = tid; i < (VC ? 5 : 3) * NPT; i += 128) {
      const int d = i / NPT, l = i - d * NPT;
      const int x0 = l % NP1, x1 = (l / NP1) % NP1, x2 = l / (NP1 * NP1);
      XE[d * NPB + (x0 - clo[0]) + PB * ((x1 - clo[1]) + PB * (x2 - clo[2]))] =
          d < 3 ? __ldg(xs + i) : __ldg((d == 3 ? A.ca : A.cb) + el * NPT + l);
    }
    constexpr int HC = NPB - NPT;
    const int2 *hl = A.xhalo + bs * HC;
    for (int h = tid; h < HC; h += 128) {
      const int2 hv = __ldg(hl + h);
      if (hv.x >= 0) {
        XE[hv.y] = __ldg(A.X + hv.x);
        XE[NPB + hv.y] = __ldg(A.X + hv.x + NPT);
        XE[2 * NPB + hv.y] = __ldg(A.X + hv.x + 2 * NPT);
        if (VC) {  // the neighbour's coefficients at the same point
          const int64_t e2 = hv.x / A.xstride, l2 = hv.x - e2 * A.xstride;
          XE[3 * NPB + hv.y] = __ldg(A.ca + e2 * NPT + l2);
          XE[4 * NPB + hv.y] = __ldg(A.cb + e2 * NPT + l2);
        }
      }
    }
  }
  __syncthreads();
  const double alpha = A.alpha, beta = A.beta;
  // L2 prefetch of the row pointers and slot positions of the rows of the CTA one residency later
  // (their addresses need its record and extended restriction, prefetched into L2 at the start):
  // the dependent chain record -> restriction -> row_ptr / positions of its first row group
  if (XV_PF_ROWS && A.pf_dist > 0 && bs + A.pf_dist < A.nel_local) {
    const int64_t nbs = bs + A.pf_dist;
    const int4 nh = __ldg(reinterpret_cast<const int4 *>(A.xe + nbs));
    const int nclo[3] = {(int8_t)(nh.y & 255), (int8_t)((nh.y >> 8) & 255), (int8_t)((nh.y >> 16) & 255)};
    const uint32_t nown = (uint32_t)nh.x;
    for (int tg = tid; tg < CF::MAXG; tg += 128) {
      int sf = 0, xx[3];
      if (!group_row<P, SP, CF::GZ, CF::B0, CF::B1, CF::NF2, CF::NF0>(0, tg, sf, xx) || !((nown >> dof_tau<P, SP>(sf, xx)) & 1))
        continue;
      const int u[3] = {xx[0] - nclo[0], xx[1] - nclo[1], xx[2] - nclo[2]};
      const int idx = sf == 0 ? fidx<SP, NB>(0, u) : (sf == 1 ? fidx<SP, NB>(1, u) : fidx<SP, NB>(2, u));
      const int64_t r = (int64_t)(__ldg(A.xvmap + nbs * 3 * CF::NVF + sf * CF::NVF + idx) & 0x7fffffffu) - A.row_begin;
      pf_l2(A.row_ptr + r);
      pf_l2(A.pos + r * CF::PW);
    }
  }
  for (int z = 0; z <= P; z += CF::GZ) {
    // cell layers of this row layer: z - 1 (first layer only; later it is still resident) and z
    // cells: all layers at the first row layer (ONE), else layer z (and z - 1 at the first)
    const int cz0 = CF::ONE ? clo[2] : (z == 0 ? -1 : z), cz1 = CF::ONE ? chi[2] : z;
    if (!CF::ONE || z == 0) {
      const int nlay = cz1 - cz0 + 1;
      for (int c = tid; c < nlay * CF::LAY; c += 128) {
        const int cz = cz0 + c / CF::LAY, cc = c % CF::LAY;
        if (cz < clo[2] || cz > chi[2]) continue;
        const int b0 = cc % NB, b1 = cc / NB;
        if (b0 >= ex[0] || b1 >= ex[1]) continue;
        double *cl = cm + (CF::ONE ? cz - clo[2] : ((cz % 2) + 2) % 2) * NE * CF::NCP;
        const int pb = b0 + PB * (b1 + PB * (cz - clo[2]));
        auto X = [&](int v, int k) -> double {
          return XE[k * NPB + pb + (v & 1) + PB * ((v >> 1) & 1) + PB * PB * ((v >> 2) & 1)];
        };
        bool ok;
        if (VC) {  // the cell's corner coefficient values (NEXT-3)
          double a8[8], b8[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            a8[v] = X(v, 3);
            b8[v] = X(v, 4);
          }
          if (SP == SP_ND) ok = cell_nd_vertex_to(X, alpha, beta, cl + cc, CF::NCP, a8, b8);
          else ok = cell_rt_vertex_to(X, alpha, beta, cl + cc, CF::NCP, a8, b8);
        } else {
          if (SP == SP_ND) ok = cell_nd_vertex_to(X, alpha, beta, cl + cc, CF::NCP);
          else ok = cell_rt_vertex_to(X, alpha, beta, cl + cc, CF::NCP);
        }
        if (!ok) s_bad = 1 + (clo[0] + b0 + 1) + (P + 2) * ((clo[1] + b1 + 1) + (P + 2) * (cz + 1));
      }
    }
    __syncthreads();
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
    // rows of the layer (thread order t = tid + 128 rr): their CSR offset, length and slot positions
    // were loaded one layer ahead (below); staging offsets by an exclusive scan of the lengths in t
    // order (consecutive rows of one coarse entity are consecutive CSR rows: contiguous in staging
    // and in CSR)
    int rs[CF::RPT], rx[CF::RPT][3], rn[CF::RPT], rso[CF::RPT];
    int64_t rout[CF::RPT];
    uint32_t rpw[CF::RPT][CF::PW];
#pragma unroll
    for (int rr = 0; rr < CF::RPT; ++rr) {
      rs[rr] = ns[rr];
      rn[rr] = nn[rr];
      rout[rr] = nout[rr];
#pragma unroll
      for (int a = 0; a < 3; ++a) rx[rr][a] = nx[rr][a];
#pragma unroll
      for (int q = 0; q < CF::PW; ++q) rpw[rr][q] = npw[rr][q];
    }
    if (z + CF::GZ <= P) load_layer(z + CF::GZ);
#pragma unroll
    for (int rr = 0; rr < CF::RPT; ++rr) {
      int incl = rn[rr];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      rso[rr] = incl - rn[rr];
      if (lane == 31) m_wt[rr * 4 + warp] = incl;
    }
    __syncthreads();
    {
      int base = 0;
#pragma unroll
      for (int rr = 0; rr < CF::RPT; ++rr) {
        int off = base;
        for (int w = 0; w < warp; ++w) off += m_wt[rr * 4 + w];
        rso[rr] += off;
        for (int w = 0; w < 4; ++w) base += m_wt[rr * 4 + w];
      }
    }
#pragma unroll
    for (int rr = 0; rr < CF::RPT; ++rr) {
      const int t = tid + 128 * rr;
      if (rs[rr] >= 0) {
        double *sv = stv + rso[rr];
        int32_t *sc = stc + rso[rr];
        if (rs[rr] == 0) fill_row<P, NB, SP, 0>(A, rx[rr], clo, ex, cm, XV, sv, sc, rpw[rr]);
        else if (rs[rr] == 1) fill_row<P, NB, SP, 1>(A, rx[rr], clo, ex, cm, XV, sv, sc, rpw[rr]);
        else fill_row<P, NB, SP, 2>(A, rx[rr], clo, ex, cm, XV, sv, sc, rpw[rr]);
      }
      (void)t;
    }
    __syncthreads();
    // write-out, each warp its own rows: the warp's staged range (its rows' entries, consecutive in
    // staging) streamed with all 32 lanes; an entry's CSR position = its staged index + the
    // destination offset of its row, found by a binary search over the warp's 32 staged row ends
#pragma unroll
    for (int rr = 0; rr < CF::RPT; ++rr) {
      w_end[warp * 32 + lane] = rso[rr] + rn[rr];
      w_dst[warp * 32 + lane] = rout[rr] - rso[rr];
      __syncwarp();
      const int S0 = __shfl_sync(0xffffffffu, rso[rr], 0), E0 = __shfl_sync(0xffffffffu, rso[rr] + rn[rr], 31);
      // one contiguous CSR run (every row with entries starts where the previous one ends; common
      // for element-interior rows): a single destination offset, no search
      const int64_t dst = rout[rr] - rso[rr];
      const long long dfirst = __shfl_sync(0xffffffffu, (long long)dst, __ffs(__ballot_sync(0xffffffffu, rn[rr] > 0) | 0x80000000u) - 1);
      const bool one_run = __all_sync(0xffffffffu, rn[rr] == 0 || dst == dfirst);
      if (one_run) {
        for (int k = S0 + lane; k < E0; k += 32) {
          if (WCOL) __stcs(A.col + dfirst + k, stc[k]);
          __stcs(A.val + dfirst + k, stv[k]);
        }
      } else {
        for (int k = S0 + lane; k < E0; k += 32) {
          int cur = 0;  // the entry's row: first of the warp's rows whose staged end exceeds k (5 steps)
#pragma unroll
          for (int st = 16; st > 0; st >>= 1) cur += (w_end[warp * 32 + cur + st - 1] <= k) ? st : 0;
          const int64_t d = w_dst[warp * 32 + cur] + k;
          if (WCOL) __stcs(A.col + d, stc[k]);
          __stcs(A.val + d, stv[k]);
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ launchers
template <int P, int NB, int SP>
constexpr bool xv_fits() {
  return XvCfg<P, NB, SP>::SMEM <= 200 * 1024;
}

template <int P, int SP>
static int nb_of(const XvArgs &a) {
  return (a.ncx <= P + 1 && a.ncy <= P + 1 && a.ncz <= P + 1) ? P + 1 : P + 2;
}

// variable coefficients: the instantiation with the coefficient boxes (one rank)
template <int P, int NB, int SP>
static cudaError_t fill_nb_vc(const XvArgs &a, cudaStream_t st) {
  using CF = XvCfg<P, NB, SP, 5>;
  if constexpr (CF::SMEM > 200 * 1024) {
    return cudaErrorInvalidValue;
  } else {
    constexpr int smem = CF::SMEM;
    constexpr int MINB = (smem + 1024) * 5 <= 228 * 1024 ? 5 : ((smem + 1024) * 4 <= 228 * 1024 ? 4 :
                         ((smem + 1024) * 3 <= 228 * 1024 ? 3 : ((smem + 1024) * 2 <= 228 * 1024 ? 2 : 1)));
    static bool attr = false;
    if (!attr) {
      for (auto k : {k_xv_fill<P, NB, SP, MINB, false, true>, k_xv_fill<P, NB, SP, MINB, true, true>}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      }
      attr = true;
    }
    if (a.values_only) k_xv_fill<P, NB, SP, MINB, false, true><<<(unsigned)a.nel_local, 128, smem, st>>>(a);
    else k_xv_fill<P, NB, SP, MINB, true, true><<<(unsigned)a.nel_local, 128, smem, st>>>(a);
    return cudaGetLastError();
  }
}

template <int P, int NB, int SP>
static cudaError_t fill_nb(const XvArgs &a, cudaStream_t st) {
  if constexpr (!xv_fits<P, NB, SP>()) {
    return cudaErrorInvalidValue;
  } else {
    if (a.ca) return fill_nb_vc<P, NB, SP>(a, st);
    using CF = XvCfg<P, NB, SP>;
    constexpr int smem = CF::SMEM;
    // CTAs per SM the shared memory allows (at most 5: >= 96 registers per thread)
    constexpr int MINB = (smem + 1024) * 5 <= 228 * 1024 ? 5 : ((smem + 1024) * 4 <= 228 * 1024 ? 4 :
                         ((smem + 1024) * 3 <= 228 * 1024 ? 3 : ((smem + 1024) * 2 <= 228 * 1024 ? 2 : 1)));
    static bool attr = false;
    if (!attr) {
      for (auto k : {k_xv_fill<P, NB, SP, MINB, false>, k_xv_fill<P, NB, SP, MINB, true>}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      }
      attr = true;
    }
    // L2 prefetch distance = resident CTAs of the grid (cached per instantiation; LOR_XPF=0: off)
    static int64_t resident = -1;
    if (resident < 0) {
      int dev = 0, nsm = 0, occ = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_xv_fill<P, NB, SP, MINB, true>, 128, smem);
      const char *e = getenv("LOR_XPF");
      resident = (e && !atoi(e)) ? 0 : (int64_t)nsm * occ;
    }
    XvArgs b = a;
    b.pf_dist = resident;
    if (a.values_only) k_xv_fill<P, NB, SP, MINB, false><<<(unsigned)a.nel_local, 128, smem, st>>>(b);
    else k_xv_fill<P, NB, SP, MINB, true><<<(unsigned)a.nel_local, 128, smem, st>>>(b);
    return cudaGetLastError();
  }
}

template <int P, int SP>
static cudaError_t run_p(int what, const XvArgs &a, cudaStream_t st) {
  if (a.nel_local <= 0) return cudaSuccess;
  const bool one = nb_of<P, SP>(a) == P + 1;
  if (what == 0) {
    if (one) k_xv_setup<P, P + 1, SP><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
    else k_xv_setup<P, P + 2, SP><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
  } else if (what == 1) {
    if (one) k_xv_sym<P, P + 1, SP><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
    else k_xv_sym<P, P + 2, SP><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
  } else {
    return one ? fill_nb<P, P + 1, SP>(a, st) : fill_nb<P, P + 2, SP>(a, st);
  }
  return cudaGetLastError();
}

template <int SP>
static cudaError_t run_sp(int what, int p, const XvArgs &a, cudaStream_t st) {
  switch (p) {
    case 1: return run_p<1, SP>(what, a, st);
    case 2: return run_p<2, SP>(what, a, st);
    case 3: return run_p<3, SP>(what, a, st);
    case 4: return run_p<4, SP>(what, a, st);
    case 5: return run_p<5, SP>(what, a, st);
    case 6: return run_p<6, SP>(what, a, st);
    case 7: return run_p<7, SP>(what, a, st);
    case 8: return run_p<8, SP>(what, a, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int P, int SP>
static int supported_p(const int cmax[3]) {
  const bool one = cmax[0] <= P + 1 && cmax[1] <= P + 1 && cmax[2] <= P + 1;
  return one ? (int)xv_fits<P, P + 1, SP>() : (int)xv_fits<P, P + 2, SP>();
}
template <int P, int SP>
static int64_t words_p(const int cmax[3]) {
  const bool one = cmax[0] <= P + 1 && cmax[1] <= P + 1 && cmax[2] <= P + 1;
  return one ? 3 * (int64_t)XvCfg<P, P + 1, SP>::NVF : 3 * (int64_t)XvCfg<P, P + 2, SP>::NVF;
}

}  // namespace

#define XV_SWITCH(FN, ...)                                  \
  switch (p) {                                              \
    case 1: return FN<1, SP>(__VA_ARGS__);                  \
    case 2: return FN<2, SP>(__VA_ARGS__);                  \
    case 3: return FN<3, SP>(__VA_ARGS__);                  \
    case 4: return FN<4, SP>(__VA_ARGS__);                  \
    case 5: return FN<5, SP>(__VA_ARGS__);                  \
    case 6: return FN<6, SP>(__VA_ARGS__);                  \
    case 7: return FN<7, SP>(__VA_ARGS__);                  \
    case 8: return FN<8, SP>(__VA_ARGS__);                  \
    default: return 0;                                      \
  }
namespace {
template <int SP>
int supported_sp(int p, const int cmax[3]) { XV_SWITCH(supported_p, cmax) }
template <int SP>
int64_t words_sp(int p, const int cmax[3]) { XV_SWITCH(words_p, cmax) }
}  // namespace
#undef XV_SWITCH

// per-space entry points (lor_xv_nd.cu, lor_xv_rt.cu)
cudaError_t xv_run_nd(int what, int p, const XvArgs &a, cudaStream_t st);
cudaError_t xv_run_rt(int what, int p, const XvArgs &a, cudaStream_t st);
int xv_supported_nd(int p, const int cmax[3]);
int xv_supported_rt(int p, const int cmax[3]);
int64_t xv_words_nd(int p, const int cmax[3]);
int64_t xv_words_rt(int p, const int cmax[3]);

}  // namespace lorb
