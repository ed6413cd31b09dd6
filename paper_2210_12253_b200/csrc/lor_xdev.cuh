// lor_xdev.cuh -- device helpers shared by the extended-frame ("owner computes") kernels of every
// space (lor_xh1.cu: H1; lor_xv.cu: Nedelec / Raviart-Thomas).  See lor_xframe.h.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "lor_sortnet.h"
#include "lor_xframe.h"

namespace lorb {
namespace xdev {

// class of an extended-frame lattice coordinate: -1 layer | 0 | [1, p-1] | p | p+1 layer
__device__ __forceinline__ int ycls(int y, int p) { return y < 0 ? 0 : (y == 0 ? 1 : (y < p ? 2 : (y == p ? 3 : 4))); }
// neighbour delta of an extended-frame lattice point along one axis
__device__ __forceinline__ int ydelta(int y, int p) { return y < 0 ? -1 : (y > p ? 1 : 0); }
// coarse-entity class of an element-local lattice (vertex) coordinate: 0 | interior | p
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

__device__ __forceinline__ void pf_l2(const void *a) { asm volatile("prefetch.global.L2 [%0];" ::"l"(a)); }

__device__ __forceinline__ void xreport(int *err, int code, int64_t e, int cell) {
  if (atomicCAS(err, 0, code) == 0) {
    err[1] = (int)e;
    err[2] = cell;
  }
}

// 1/x for x > 0: float seed + two Newton steps (relative error ~1e-28 before rounding).  The seed
// needs x inside the normal float range: outside [2^-120, 2^120] (cell volumes of meshes scaled far
// from unit size, e.g. coordinates x 1e-14) x = m 2^e is reduced to m in [0.5, 1) first and the
// result scaled back by 2^-e (inline, no division slow path), so the result never depends on the
// float range (tests/test_gpu_boundary.py scaled meshes).
__device__ __forceinline__ double rcp_newton(double x) {
  float rf;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"((float)x));
  double r = (double)rf;
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rcp_pos(double x) {
  if (__builtin_expect(x > 7.52316384526264e-37 && x < 1.329227995784916e36, 1)) return rcp_newton(x);
  const int hi = __double2hiint(x), ex = ((hi >> 20) & 0x7ff) - 1022;  // x = m 2^ex, m in [0.5, 1)
  const double m = __hiloint2double((hi & 0x800fffff) | (1022 << 20), __double2loint(x));
  const double r = rcp_newton(m);
  // 2^-ex in two factors (each a normal double for |ex| <= 1022)
  const int e1 = -ex / 2, e2 = -ex - e1;
  return r * __hiloint2double((e1 + 1023) << 20, 0) * __hiloint2double((e2 + 1023) << 20, 0);
}

// ---- ranks of a row's column ids = final positions in the ascending-column CSR row (reading P-5)
// sorting network on packed keys (id << SB | slot), generated tables (lor_sortnet.h)
template <int N>
struct Net;
template <>
struct Net<11> {
  static constexpr int LEN = kNetLen11;
  static constexpr const uint16_t *tab() { return kNet11; }
};
template <>
struct Net<27> {
  static constexpr int LEN = kNetLen27;
  static constexpr const uint16_t *tab() { return kNet27; }
};
template <>
struct Net<33> {
  static constexpr int LEN = kNetLen33;
  static constexpr const uint16_t *tab() { return kNet33; }
};
template <int N, int C>
__device__ __forceinline__ void net_cmp(int (&v)[N]) {
  constexpr uint16_t c = N == 11 ? kNet11[C] : (N == 27 ? kNet27[C] : kNet33[C]);
  constexpr int a = c >> 6, b = c & 63;
  const int lo = min(v[a], v[b]), hi = max(v[a], v[b]);
  v[a] = lo;
  v[b] = hi;
}
template <int N, int... C>
__device__ __forceinline__ void sortnet(int (&v)[N], std::integer_sequence<int, C...>) {
  (net_cmp<N, C>(v), ...);
}

// pairwise ranks (any id range): ranks as bytes of pw, byte k starts at k (every j < k counted as
// smaller) and each pair (j, k) moves one count from k to j when key_k < key_j (branch-free)
__host__ __device__ constexpr int pair_j(int t, int n) {
  int j = 0;
  while (t >= n - 1 - j) { t -= n - 1 - j; ++j; }
  return j;
}
__host__ __device__ constexpr int pair_k(int t, int n) {
  int j = 0;
  while (t >= n - 1 - j) { t -= n - 1 - j; ++j; }
  return j + 1 + t;
}
template <int N, int NW, int T>
__device__ __forceinline__ void rank_pair(const int (&key)[N], uint32_t (&pw)[NW]) {
  constexpr int j = pair_j(T, N), k = pair_k(T, N);
  const uint32_t lt = (uint32_t)(key[k] < key[j]);
  pw[j >> 2] += lt << (8 * (j & 3));
  pw[k >> 2] -= lt << (8 * (k & 3));
}
template <int N, int NW, int... T>
__device__ __forceinline__ void rank_pairs(const int (&key)[N], uint32_t (&pw)[NW], std::integer_sequence<int, T...>) {
  (rank_pair<N, NW, T>(key, pw), ...);
}

// positions of N keys (absent slots: key 0x7fffffff) into the bytes of pw (255 = absent).
// sort32: ids < 2^(31 - SB); scratch: N bytes of this thread's shared memory.
template <int N>
__device__ __forceinline__ void row_positions(const int (&key)[N], bool sort32, uint8_t *scratch,
                                              uint32_t (&pw)[(N + 3) / 4]) {
  constexpr int NW = (N + 3) / 4;
  constexpr int SB = N <= 16 ? 4 : (N <= 32 ? 5 : 6);
  constexpr int ABS = 0x7fffffff & ~((1 << SB) - 1);  // absent: sorts after every present key
  if (sort32) {
    int v[N];
#pragma unroll
    for (int j = 0; j < N; ++j) v[j] = key[j] == 0x7fffffff ? (ABS | j) : ((key[j] << SB) | j);
    sortnet<N>(v, std::make_integer_sequence<int, Net<N>::LEN>{});
#pragma unroll
    for (int q = 0; q < NW; ++q) reinterpret_cast<uint32_t *>(scratch)[q] = 0xffffffffu;
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (v[i] < ABS) scratch[v[i] & ((1 << SB) - 1)] = (uint8_t)i;
#pragma unroll
    for (int q = 0; q < NW; ++q) pw[q] = reinterpret_cast<const uint32_t *>(scratch)[q];
  } else {
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      uint32_t w = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (4 * q + b < N) w |= (uint32_t)(4 * q + b) << (8 * b);
      pw[q] = w;
    }
    rank_pairs<N, NW>(key, pw, std::make_integer_sequence<int, N * (N - 1) / 2>{});
#pragma unroll
    for (int j = 0; j < N; ++j) pw[j >> 2] |= (key[j] == 0x7fffffff ? 0xffu : 0u) << (8 * (j & 3));
  }
}

}  // namespace xdev
}  // namespace lorb
