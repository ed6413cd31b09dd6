// lor_kernels.cu -- hand-written sm_100a fp64 kernels of the B200 LOR assembly library.
//
// Per assembly call (PAPER.md Step S1.2, A1-A3):
//   k_count     A2 part 1: per (element, local row) the number of columns this element "owns"
//               under the minimal-macro-element rule; exclusive rows are
//               stored, shared rows accumulated with integer atomics.
//   k_scan      A2: decoupled look-back exclusive scan -> int64 row_ptr.
//   k_assemble  A1 + A2 part 2 of the general path (lor_asm.cuh; Gauss-2, 2D H1, variable-coefficient
//               ND, ...): one CTA per macro element ("one block of threads per macro
//               element"): sub-cell matrices staged in shared memory (never written to HBM), then per
//               local row the values gathered from the <= 2^d cells containing it and the columns
//               emitted in ascending global order from the element's affine "block" numbering (no
//               sort).  Rows owned by one element go straight to CSR; rows on shared coarse
//               entities go out as natural-order partial rows, summed by k_merge_rows with the setup
//               merge plan.
//   k_finalize_list  interface rows whose partial rows came over NCCL (A3 replacement).
//   k_discrete_map / k_discrete  discrete gradient (Algorithm 1, l.417-438) / curl (l.440-445).
//   k_dofmap    element restriction (for parity tests of the numbering).
//   k_coords    LOR vertex coordinate vectors: E-vector -> owned H1 dofs.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "lor_cells.cuh"
#include "lor_device.cuh"
#include "lor_kernels.h"
#include "lor_asm.cuh"

namespace lorb {

// ================================================================================ tables
// k_build_tables: one CTA per (sub-lattice s, row key rk).  Uses the same geometric helpers as the
// reference-checked v1 kernels (seg_bounds / coord_cls / join_cls) on a representative row.
template <int DIM, int SP>
__global__ void k_build_tables(int p, uint32_t *tslot, uint8_t *tsize, uint32_t *tpb, uint8_t *tnpb, uint8_t *tlex) {
  using C = Tr<DIM, SP>;
  constexpr int S = C::S, W = C::W, NB = S * 27;
  __shared__ int32_t s_zero[1];
  if (threadIdx.x == 0) s_zero[0] = 0;
  __syncthreads();
  const int s = blockIdx.x / NROWKEY, rk = blockIdx.x % NROWKEY;
  int x[3] = {0, 0, 0};
  bool valid = true;
  int kk = rk;
  for (int a = 0; a < 3; ++a) {
    const int key = kk % 9;
    kk /= 9;
    if (a >= DIM) { valid &= (key == 0); continue; }
    const int ext = ext_of<SP>(p, s, a);
    const int kl = key / 3, kh = key % 3;
    int xa = (kl < 2) ? kl : ((kh < 2) ? ext - 1 - kh : 2);
    const int dl = xa < 2 ? xa : 2, d = ext - 1 - xa, dh = d < 2 ? d : 2;
    valid &= (xa >= 0 && xa < ext && dl == kl && dh == kh);
    x[a] = xa;
  }
  uint32_t *ts = tslot + (int64_t)blockIdx.x * W;
  uint8_t *tz = tsize + (int64_t)blockIdx.x * tab_tzs(NB);
  uint32_t *tp = tpb + (int64_t)blockIdx.x * NB;
  int cr[3] = {1, 1, 1};
  for (int a = 0; a < DIM; ++a) cr[a] = coord_cls(vkind<SP>(s, a), x[a], p);
  // slots.  Word: bits 0-6 column block b' = s2*27 + tau' (127 = slot outside the element),
  // 7-11 join slot tau_J, 12-23 per axis a (at 12+4a) offset and length-1 inside the block's
  // sub-box, 24-25 s2, 26-31 (dx+1) | (dy+1) << 2 | (dz+1) << 4.
  for (int j = threadIdx.x; j < W; j += blockDim.x) {
    uint32_t w = 127u;
    if (valid) {
      // find (s2, d) of slot j in the natural order
      int jj = j, s2 = 0;
      while (s2 < S && jj >= st_n<DIM, SP>(s, s2)) { jj -= st_n<DIM, SP>(s, s2); ++s2; }
      const int nx = st_hi<SP>(s, s2, 0) - st_lo<SP>(s, s2, 0) + 1, ny = st_hi<SP>(s, s2, 1) - st_lo<SP>(s, s2, 1) + 1;
      int d[3];
      d[0] = st_lo<SP>(s, s2, 0) + jj % nx;
      d[1] = st_lo<SP>(s, s2, 1) + (jj / nx) % ny;
      d[2] = (DIM == 3) ? st_lo<SP>(s, s2, 2) + jj / (nx * ny) : 0;
      int y[3] = {x[0] + d[0], x[1] + d[1], x[2] + d[2]};
      bool in = true;
      for (int a = 0; a < DIM; ++a) in &= (y[a] >= 0 && y[a] < ext_of<SP>(p, s2, a));
      w = ((uint32_t)s2 << 24) | ((uint32_t)(d[0] + 1) << 26) | ((uint32_t)(d[1] + 1) << 28) | ((uint32_t)(d[2] + 1) << 30);
      if (in) {
        int cc[3] = {0, 0, 0};
        for (int a = 0; a < DIM; ++a) cc[a] = coord_cls(vkind<SP>(s2, a), y[a], p);
        const int t2 = cc[0] + 3 * cc[1] + (DIM == 3 ? 9 * cc[2] : 0);
        int tj = join_cls(cr[0], cc[0]) + 3 * join_cls(cr[1], cc[1]);
        if (DIM == 3) tj += 9 * join_cls(cr[2], cc[2]);
        w |= (uint32_t)(s2 * 27 + t2) | ((uint32_t)tj << 7);
        int off[3] = {0, 0, 0}, len[3] = {1, 1, 1};
        for (int a = 0; a < DIM; ++a) {
          int lo, hi;
          seg_bounds<SP>(p, s, s2, a, x[a], cc[a], lo, hi);
          w |= (uint32_t)(y[a] - lo) << (12 + 4 * a);
          w |= (uint32_t)(hi - lo) << (14 + 4 * a);
          off[a] = y[a] - lo;
          len[a] = hi - lo + 1;
        }
        // lexicographic rank inside the sub-box for each orientation code of the block's entity:
        // the block's canonical axis order / directions come from block_affine (bases irrelevant)
        for (int code = 0; code < 8; ++code) {
          ElemTopo Tz;
          for (int q = 0; q < 27; ++q) { Tz.ent[q] = 0; Tz.orient[q] = 0; Tz.val[q] = 1; Tz.flags[q] = 0; }
          Tz.orient[t2] = (uint8_t)code;
          const int32_t *zb[4] = {s_zero, s_zero, s_zero, s_zero};
          Blk B;
          block_affine<DIM, SP>(p, s2, t2, Tz, zb, B);
          int o2[3];
          for (int a = 0; a < 3; ++a) o2[a] = (B.str[a] < 0) ? len[a] - 1 - off[a] : off[a];
          const int f = B.ord & 3, m = (B.ord >> 2) & 3, sl = (B.ord >> 4) & 3;
          tlex[((int64_t)blockIdx.x * W + j) * 8 + code] = (uint8_t)(o2[f] + len[f] * (o2[m] + len[m] * o2[sl]));
        }
      } else {
        w |= 127u;
      }
    }
    ts[j] = w;
  }
  // block sizes and the compact present-block list
  for (int b = threadIdx.x; b < NB; b += blockDim.x) {
    int n = 0;
    if (valid) {
      const int s2 = b / 27, t2 = b % 27;
      n = 1;
      for (int a = 0; a < 3; ++a) {
        const int c = cls_of(t2, a);
        if (a >= DIM) { n *= (c == 0) ? 1 : 0; continue; }  // 2D blocks: tau < 9
        int lo, hi;
        seg_bounds<SP>(p, s, s2, a, x[a], c, lo, hi);
        n *= hi >= lo ? hi - lo + 1 : 0;
      }
    }
    tz[b] = (uint8_t)n;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0;
    for (int b = 0; b < NB; ++b) {
      if (!tz[b]) continue;
      const int t2 = b % 27;
      int tj = join_cls(cr[0], cls_of(t2, 0)) + 3 * join_cls(cr[1], cls_of(t2, 1));
      if (DIM == 3) tj += 9 * join_cls(cr[2], cls_of(t2, 2));
      tp[n++] = (uint32_t)b | ((uint32_t)tj << 7) | ((uint32_t)tz[b] << 12);
    }
    tnpb[blockIdx.x] = (uint8_t)n;
  }
}

// ================================================================================ k_count
// A2 part 1: per (element, local row) the number of columns whose join entity
// has this element as its minimal element; exclusive rows are stored, shared rows atomically added.
template <int DIM, int SP>
__global__ void __launch_bounds__(128) k_count(CountArgs A) {
  constexpr int S = Tr<DIM, SP>::S;
  constexpr int NB = S * 27;
  const int64_t ei = blockIdx.x;
  if (ei >= A.ntopo) return;
  __shared__ ElemTopo T;
  __shared__ Blk blk[NB];
  {
    const int4 *src = reinterpret_cast<const int4 *>(A.topo + ei);
    int4 *dst = reinterpret_cast<int4 *>(&T);
    for (int i = threadIdx.x; i < (int)(sizeof(ElemTopo) / 16); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int p = A.p;
  for (int b = threadIdx.x; b < NB; b += blockDim.x) {
    const int s = b / 27, tau = b % 27;
    if (DIM == 2 && tau >= 9) { blk[b].size = 0; continue; }
    if (T.flags[tau] & TF_OWNED) block_affine<DIM, SP>(p, s, tau, T, A.base, blk[b]);
    else blk[b].size = 0;
  }
  __syncthreads();
  const int ndpe = A.ndpe;
  for (int l = threadIdx.x; l < ndpe; l += blockDim.x) {
    int s, x[3];
    decode_local<DIM, SP>(p, l, s, x);
    const int tr = row_tau<DIM, SP>(p, s, x);
    if (!(T.flags[tr] & TF_OWNED)) continue;
    const Blk &B = blk[s * 27 + tr];
    const int gid = B.g0 + B.str[0] * x[0] + B.str[1] * x[1] + B.str[2] * x[2];
    const int key = s * NROWKEY + row_key<DIM, SP>(p, s, x);
    const int n = __ldg(A.tabs.npb + key);
    const uint32_t *pb = A.tabs.pb + (int64_t)key * NB;
    int cnt = 0;
    for (int i = 0; i < n; ++i) {
      const uint32_t w = __ldg(pb + i);
      if (T.flags[(w >> 7) & 31] & TF_MIN) cnt += (int)(w >> 12);
    }
    int32_t *dst = A.cnt + (gid - A.row_begin);
    if (T.val[tr] <= 1) *dst = cnt;
    else atomicAdd(dst, cnt);
  }
}

// ================================================================================ k_scan
// Decoupled look-back exclusive scan (single pass).  Tile = 128 threads x 16 items.
constexpr int SCAN_T = 128, SCAN_I = 16, SCAN_TILE = SCAN_T * SCAN_I;
constexpr unsigned long long FLAG_A = 1ull << 62, FLAG_P = 2ull << 62, VAL_MASK = (1ull << 62) - 1;

__global__ void __launch_bounds__(SCAN_T) k_scan(const int32_t *__restrict__ cnt, int64_t *__restrict__ row_ptr, int64_t n,
                                                 unsigned long long *status, unsigned int *tile_ctr) {
  __shared__ unsigned int s_tile;
  __shared__ long long s_warp[SCAN_T / 32];
  __shared__ long long s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t tb = tile * SCAN_TILE;
  const int64_t base = tb + (int64_t)threadIdx.x * SCAN_I;
  // the tile's counts are read coalesced (lane = consecutive rows) and transposed through shared
  // memory to the blocked order of the per-thread scan; the row offsets go back the same way.
  // Row-major [SCAN_T][SCAN_I + 1] (padded: conflict-free in both directions).
  __shared__ long long s_buf[SCAN_T * (SCAN_I + 1)];
  auto padi = [](int e) { return (e / SCAN_I) * (SCAN_I + 1) + e % SCAN_I; };
#pragma unroll
  for (int i = 0; i < SCAN_I; ++i) {
    const int e = i * SCAN_T + threadIdx.x;
    const int64_t k = tb + e;
    s_buf[padi(e)] = (k < n) ? cnt[k] : 0;
  }
  __syncthreads();
  int v[SCAN_I];
  long long tsum = 0;
#pragma unroll
  for (int i = 0; i < SCAN_I; ++i) {
    v[i] = (int)s_buf[threadIdx.x * (SCAN_I + 1) + i];
    tsum += v[i];
  }
  // block-level exclusive scan of thread sums
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long incl = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  long long woff = 0, total = 0;
#pragma unroll
  for (int w = 0; w < SCAN_T / 32; ++w) {
    if (w < wid) woff += s_warp[w];
    total += s_warp[w];
  }
  const long long texcl = woff + incl - tsum;
  // look-back (warp 0)
  if (wid == 0) {
    long long prefix = 0;
    if (tile == 0) {
      if (lane == 0) {
        __threadfence();
        atomicExch(status + tile, FLAG_P | (unsigned long long)total);
      }
    } else {
      if (lane == 0) atomicExch(status + tile, FLAG_A | (unsigned long long)total);
      int64_t look = tile - 1;
      while (true) {
        const int64_t idx = look - lane;
        unsigned long long st = 0;
        if (idx >= 0) {
          do {
            st = atomicAdd(status + idx, 0ull);
          } while ((st >> 62) == 0);
        } else {
          st = FLAG_P;  // before the first tile: inclusive prefix 0
        }
        const unsigned pmask = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        // lanes up to (and including) the first P flag contribute
        const int firstp = pmask ? __ffs(pmask) - 1 : 32;
        long long contrib = (lane <= firstp) ? (long long)(st & VAL_MASK) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
        prefix += contrib;
        if (pmask) break;
        look -= 32;
      }
      if (lane == 0) atomicExch(status + tile, FLAG_P | (unsigned long long)(prefix + total));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  long long run = s_prefix + texcl;
#pragma unroll
  for (int i = 0; i < SCAN_I; ++i) {
    s_buf[threadIdx.x * (SCAN_I + 1) + i] = run;  // own counts were read before the barrier above
    run += v[i];
  }
  if (base <= n - 1 && n - 1 < base + SCAN_I) row_ptr[n] = run;  // thread holding the last item
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SCAN_I; ++i) {
    const int e = i * SCAN_T + threadIdx.x;
    if (tb + e < n) row_ptr[tb + e] = s_buf[padi(e)];
  }
  if (n == 0 && tile == 0 && threadIdx.x == 0) row_ptr[0] = 0;
}

__global__ void __launch_bounds__(128) k_finalize_list(FinArgs F) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int i = blockIdx.x;
  if (i >= F.n) return;
  const Ose O = F.ose[F.list[i]];
  finalize_ose(O, F.ose_slots, F.scratch, F.rstride, F.maxl, F.maxu, F.row_begin, F.row_ptr, F.col, F.val, smem,
               F.smem_bytes);
}

// ================================================================================ setup merge plan
// One CTA per owned shared entity whose contributors are all local; one thread per row.  Reads the
// partial-row records written by k_assemble in plan mode (each contributor's row sorted by column,
// entries tagged with their block base and stencil slot; header = length, local row), merges the
// block runs of the k contributors by base (= the final row order) and records, for every final
// position q and contributor m, m's stencil slot at q (255 = m does not hold q), plus m's local row.
// Topological: computed once in lor_setup; at run time the last contributor gathers with it.
__global__ void k_plan_merge(PlanArgs A) {
  const int oi = blockIdx.x;
  if (oi >= A.n || A.is_defer[oi]) return;
  const Ose O = A.ose[oi];
  const int k = O.k, W = A.W;
  const int rstr = plan_row_bytes(k, W);
  for (int r = threadIdx.x; r < O.nrows; r += blockDim.x) {
    uint8_t *pr = A.plan + A.pbase[oi] + (int64_t)r * rstr;
    int32_t *rrow = reinterpret_cast<int32_t *>(pr);
    uint16_t *hm = reinterpret_cast<uint16_t *>(pr + 4 * k);
    int32_t *cq = reinterpret_cast<int32_t *>(pr + plan_col_off(k, W));
    uint8_t *js = pr + plan_col_off(k, W) + 4 * W;
    for (int i = 0; i < W; ++i) { hm[i] = 0; cq[i] = -1; }
    for (int i = 0; i < W * k; ++i) js[i] = 255;
    int64_t rid[MAX_VALENCE];
    int len[MAX_VALENCE], ptr[MAX_VALENCE];
    for (int m = 0; m < k; ++m) {
      rid[m] = ((int64_t)A.ose_slots[O.slot_off + m] + r) * A.rstride;
      const RecEntry h = A.scratch[rid[m] + A.rstride - 1];
      len[m] = h.col;
      rrow[m] = A.ose_elem[O.slot_off + m] * A.ndpe + h.bbase;
      ptr[m] = 0;
    }
    int P = 0;
    while (true) {
      int minb = 0x7fffffff;
      for (int m = 0; m < k; ++m)
        if (ptr[m] < len[m]) {
          const int b = A.scratch[rid[m] + ptr[m]].bbase;
          minb = b < minb ? b : minb;
        }
      if (minb == 0x7fffffff) break;
      int size = 0;
      for (int m = 0; m < k; ++m) {
        if (ptr[m] >= len[m] || A.scratch[rid[m] + ptr[m]].bbase != minb) continue;
        int e = ptr[m];
        while (e < len[m] && A.scratch[rid[m] + e].bbase == minb) {
          const int q = P + (e - ptr[m]);
          if (q < W) {
            const RecEntry &re = A.scratch[rid[m] + e];
            js[q * k + m] = (uint8_t)(int)re.val;
            if (!hm[q]) cq[q] = re.col;
            hm[q] |= (uint16_t)(1u << m);
          }
          ++e;
        }
        size = e - ptr[m];
        ptr[m] = e;
      }
      P += size;
    }
  }
}

// Merge pass over all in-kernel-merged shared rows (every contributor local to this rank): one
// warp per row, lane = final column position q.  The column comes from the setup merge plan, the
// value is the sum over the contributors holding q, in element order, of their natural-order
// partial rows written by k_assemble (column sign from the plan).
constexpr int MERGE_RPW = 4;  // rows per warp, their loads interleaved (memory-level parallelism)

__global__ void __launch_bounds__(256) k_merge_rows(MergeArgs A) {
  constexpr int R = MERGE_RPW;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t i0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * R;
  if (i0 >= A.n) return;
  const int W = A.W;
  MergeRow d{0, 0, 0};
  if (lane < R && i0 + lane < A.n) d = A.rows[i0 + lane];
  const uint8_t *pr[R];
  int k[R], len[R];
  int64_t rb[R], ro[R];
#pragma unroll
  for (int u = 0; u < R; ++u) {
    const int64_t po = __shfl_sync(FULL, d.plan_off, u);
    const int g = __shfl_sync(FULL, d.g, u);
    k[u] = __shfl_sync(FULL, d.k, u);
    pr[u] = A.plan + po;
    rb[u] = lane < k[u] ? (int64_t)__ldg(reinterpret_cast<const int32_t *>(pr[u]) + lane) * A.W8 : 0;
    ro[u] = k[u] ? __ldg(A.row_ptr + g) : 0;
    len[u] = k[u] ? (int)(__ldg(A.row_ptr + g + 1) - ro[u]) : 0;
  }
  for (int q0 = 0; q0 < W; q0 += 32) {
    const int q = q0 + lane;
    unsigned hm[R];
    int gid[R];
    const uint8_t *js[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const bool on = q < len[u];
      const int coff = plan_col_off(k[u], W);
      hm[u] = on ? __ldg(reinterpret_cast<const uint16_t *>(pr[u] + 4 * k[u]) + q) : 0u;
      gid[u] = on ? __ldg(reinterpret_cast<const int32_t *>(pr[u] + coff) + q) : 0;
      js[u] = pr[u] + coff + 4 * W + q * k[u];
    }
    double xv[R][4];
#pragma unroll
    for (int u = 0; u < R; ++u) {
#pragma unroll
      for (int m4 = 0; m4 < 4; ++m4) {  // first four holders of every row: all loads in flight together
        const bool has = hm[u] != 0;
        const int m = has ? __ffs(hm[u]) - 1 : 0;
        if (has) hm[u] &= hm[u] - 1;
        const int64_t rr = __shfl_sync(FULL, rb[u], m);
        double x = 0.0;
        if (has) {
          const int jm = __ldg(js[u] + m);
          x = A.nval[rr + (jm & 63)];
          x = (jm & 64) ? -x : x;
        }
        xv[u][m4] = x;
      }
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      double sum = ((xv[u][0] + xv[u][1]) + xv[u][2]) + xv[u][3];
      while (__any_sync(FULL, hm[u] != 0)) {  // rare: more than four holders (vertex rows)
        const bool has = hm[u] != 0;
        const int m = has ? __ffs(hm[u]) - 1 : 0;
        if (has) hm[u] &= hm[u] - 1;
        const int64_t rr = __shfl_sync(FULL, rb[u], m);
        if (has) {
          const int jm = __ldg(js[u] + m);
          const double x = A.nval[rr + (jm & 63)];
          sum += (jm & 64) ? -x : x;
        }
      }
      if (q < len[u]) {
        __stcs(A.col + ro[u] + q, gid[u]);
        __stcs(A.val + ro[u] + q, sum);
      }
    }
  }
}

cudaError_t launch_merge_rows(const MergeArgs &a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  const int64_t warps = (a.n + MERGE_RPW - 1) / MERGE_RPW;
  k_merge_rows<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_plan_merge(const PlanArgs &a, int n_ose, cudaStream_t st) {
  if (n_ose <= 0) return cudaSuccess;
  k_plan_merge<<<(unsigned)n_ose, 64, 0, st>>>(a);
  return cudaGetLastError();
}

// ================================================================================ G, C, dof map
// One CTA per local element; the row's element writes it if it is the minimal element containing
// the row's entity (rows owned by this rank).  Columns sorted ascending (reading P-5).
template <int WHICH>  // 0 = gradient (ND rows, H1 cols), 1 = curl (RT rows, ND cols)
__global__ void __launch_bounds__(128) k_discrete(DiscArgs A) {
  constexpr int RSP = WHICH == 0 ? SP_ND : SP_RT;
  constexpr int CSP = WHICH == 0 ? SP_H1 : SP_ND;
  constexpr int CS = Tr<3, CSP>::S;
  __shared__ ElemTopo T;
  __shared__ Blk brow[81];
  __shared__ Blk bcol[81];
  const int64_t el = blockIdx.x;
  if (el >= A.nel_local) return;
  {
    const int4 *src = reinterpret_cast<const int4 *>(A.topo + el);
    int4 *dst = reinterpret_cast<int4 *>(&T);
    for (int i = threadIdx.x; i < (int)(sizeof(ElemTopo) / 16); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int p = A.p;
  if (threadIdx.x < 81) {
    const int s = threadIdx.x / 27, tau = threadIdx.x % 27;
    block_affine<3, RSP>(p, s, tau, T, A.base_row, brow[threadIdx.x]);
    if (s < CS) block_affine<3, CSP>(p, s, tau, T, A.base_col, bcol[threadIdx.x]);
  }
  __syncthreads();
  const int ndpe = (WHICH == 0) ? 3 * p * (p + 1) * (p + 1) : 3 * p * p * (p + 1);
  for (int l = threadIdx.x; l < ndpe; l += blockDim.x) {
    int s, x[3];
    decode_local<3, RSP>(p, l, s, x);
    const int tr = row_tau<3, RSP>(p, s, x);
    if (!(T.flags[tr] & TF_OWNED) || !(T.flags[tr] & TF_MIN)) continue;
    const Blk &B = brow[s * 27 + tr];
    const int gid = B.g0 + B.str[0] * x[0] + B.str[1] * x[1] + B.str[2] * x[2];
    const int64_t row = gid - A.row_begin;
    if (WHICH == 0) {
      int y[3] = {x[0], x[1], x[2]};
      const int tt = row_tau<3, SP_H1>(p, 0, y);
      const Blk &Bt = bcol[tt];
      const int gt = Bt.g0 + Bt.str[0] * y[0] + Bt.str[1] * y[1] + Bt.str[2] * y[2];
      y[s] += 1;
      const int th = row_tau<3, SP_H1>(p, 0, y);
      const Blk &Bh = bcol[th];
      const int gh = Bh.g0 + Bh.str[0] * y[0] + Bh.str[1] * y[1] + Bh.str[2] * y[2];
      const double sg = (double)B.sigma;
      const bool sw = gh < gt;
      A.col[2 * row] = sw ? gh : gt;
      A.col[2 * row + 1] = sw ? gt : gh;
      A.val[2 * row] = sw ? sg : -sg;
      A.val[2 * row + 1] = sw ? -sg : sg;
    } else {
      // face (s, x): cyclic in-face axes (u', v') = (s+1, s+2) mod 3; edges:
      // u'-edge at v'=0 (+1), v'-edge at u'=1 (+1), u'-edge at v'=1 (-1), v'-edge at u'=0 (-1)
      const int up = (s + 1) % 3, vp = (s + 2) % 3;
      int c[4];
      double v[4];
      const int eax[4] = {up, vp, up, vp};
      const int eoff[4] = {0, 1, 1, 0};
      const double es[4] = {1.0, 1.0, -1.0, -1.0};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int y[3] = {x[0], x[1], x[2]};
        const int other = (eax[q] == up) ? vp : up;
        y[other] += eoff[q];
        const int te = row_tau<3, SP_ND>(p, eax[q], y);
        const Blk &Be = bcol[eax[q] * 27 + te];
        c[q] = Be.g0 + Be.str[0] * y[0] + Be.str[1] * y[1] + Be.str[2] * y[2];
        v[q] = es[q] * (double)B.sigma * (double)Be.sigma;
      }
      // sort 4 (network)
#define CSWAP(i, j)                                   \
  if (c[j] < c[i]) {                                  \
    int tc = c[i]; c[i] = c[j]; c[j] = tc;            \
    double tv = v[i]; v[i] = v[j]; v[j] = tv;         \
  }
      CSWAP(0, 1) CSWAP(2, 3) CSWAP(0, 2) CSWAP(1, 3) CSWAP(1, 2)
#undef CSWAP
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        A.col[4 * row + q] = c[q];
        A.val[4 * row + q] = v[q];
      }
    }
  }
}

// G and C from the setup element restrictions (the reused HO element restriction): one
// CTA per element, one thread per local row dof in local order (consecutive threads -> consecutive
// rows of a coarse entity), the column restriction of the element staged in shared memory; the
// owning element (minimal element containing the row's entity, this rank) writes the row's 2 / 4
// entries with one vector store each (row_ptr[i] = 2i / 4i keeps them 8 / 16-byte aligned).  Reads
// exactly the map bytes of SURVEY d.3's B_G / B_C.
template <int WHICH>
__global__ void __launch_bounds__(128) k_discrete_map(DiscMapArgs A) {
  constexpr int RSP = WHICH == 0 ? SP_ND : SP_RT;
  __shared__ uint8_t flags[27];
  extern __shared__ int32_t cmap[];  // [ndpe_col] ids, then (curl) [ndpe_col] signs as int8
  const int64_t el = blockIdx.x;
  if (el >= A.nel_local) return;
  const int p = A.p;
  const int ndr = WHICH == 0 ? 3 * p * (p + 1) * (p + 1) : 3 * p * p * (p + 1);
  const int ndc = WHICH == 0 ? (p + 1) * (p + 1) * (p + 1) : 3 * p * (p + 1) * (p + 1);
  int8_t *csg = reinterpret_cast<int8_t *>(cmap + ndc);
  if (threadIdx.x < 27) flags[threadIdx.x] = A.topo[el].flags[threadIdx.x];
  for (int i = threadIdx.x; i < ndc; i += blockDim.x) {
    cmap[i] = __ldg(A.cmap + el * ndc + i);
    if (WHICH == 1) csg[i] = __ldg(A.csgn + el * ndc + i);
  }
  __syncthreads();
  for (int l = threadIdx.x; l < ndr; l += blockDim.x) {
    int s, x[3];
    decode_local<3, RSP>(p, l, s, x);
    const int tr = row_tau<3, RSP>(p, s, x);
    if ((flags[tr] & (TF_OWNED | TF_MIN)) != (TF_OWNED | TF_MIN)) continue;
    const int64_t row = (int64_t)__ldg(A.rmap + el * ndr + l) - A.row_begin;
    const double sg = (double)__ldg(A.rsgn + el * ndr + l);
    if (A.row_ptr) {  // the stride row pointer, fused (every owned row is written exactly once)
      A.row_ptr[row] = (WHICH == 0 ? 2 : 4) * row;
      if (row == A.n_rows - 1) A.row_ptr[A.n_rows] = (WHICH == 0 ? 2 : 4) * A.n_rows;
    }
    if (WHICH == 0) {
      const int lt = x[0] + (p + 1) * (x[1] + (p + 1) * x[2]);
      const int lh = lt + (s == 0 ? 1 : (s == 1 ? p + 1 : (p + 1) * (p + 1)));
      const int gt = cmap[lt], gh = cmap[lh];
      const bool sw = gh < gt;
      reinterpret_cast<int2 *>(A.col)[row] = sw ? make_int2(gh, gt) : make_int2(gt, gh);
      reinterpret_cast<double2 *>(A.val)[row] = sw ? make_double2(sg, -sg) : make_double2(-sg, sg);
    } else {
      // face (s, x): cyclic in-face axes (u', v') = (s+1, s+2) mod 3; edges u'-edge at v'=0 (+1),
      // v'-edge at u'=1 (+1), u'-edge at v'=1 (-1), v'-edge at u'=0 (-1) (App. A.5, reading P-15)
      const int up = (s + 1) % 3, vp = (s + 2) % 3;
      int c[4];
      double v[4];
      const int eax[4] = {up, vp, up, vp};
      const int eoff[4] = {0, 1, 1, 0};
      const double es[4] = {1.0, 1.0, -1.0, -1.0};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int y[3] = {x[0], x[1], x[2]};
        const int other = (eax[q] == up) ? vp : up;
        y[other] += eoff[q];
        const int a = eax[q];
        const int e0 = a == 0 ? p : p + 1, e1 = a == 1 ? p : p + 1;
        const int le = a * p * (p + 1) * (p + 1) + y[0] + e0 * (y[1] + e1 * y[2]);
        c[q] = cmap[le];
        v[q] = es[q] * sg * (double)csg[le];
      }
#define CSWAP(i, j)                                   \
  if (c[j] < c[i]) {                                  \
    int tc = c[i]; c[i] = c[j]; c[j] = tc;            \
    double tv = v[i]; v[i] = v[j]; v[j] = tv;         \
  }
      CSWAP(0, 1) CSWAP(2, 3) CSWAP(0, 2) CSWAP(1, 3) CSWAP(1, 2)
#undef CSWAP
      reinterpret_cast<int4 *>(A.col)[row] = make_int4(c[0], c[1], c[2], c[3]);
      reinterpret_cast<double2 *>(A.val)[2 * row] = make_double2(v[0], v[1]);
      reinterpret_cast<double2 *>(A.val)[2 * row + 1] = make_double2(v[2], v[3]);
    }
  }
}

cudaError_t launch_discrete_map(int which, const DiscMapArgs &a, cudaStream_t st) {
  if (a.nel_local <= 0) return cudaSuccess;
  const int p = a.p;
  const int ndc = which == 0 ? (p + 1) * (p + 1) * (p + 1) : 3 * p * (p + 1) * (p + 1);
  const size_t smem = (size_t)ndc * (which == 0 ? 4 : 5);
  if (which == 0) k_discrete_map<0><<<(unsigned)a.nel_local, 128, smem, st>>>(a);
  else k_discrete_map<1><<<(unsigned)a.nel_local, 128, smem, st>>>(a);
  return cudaGetLastError();
}

template <int DIM, int SP>
__global__ void __launch_bounds__(128) k_dofmap(DofmapArgs A) {
  __shared__ ElemTopo T;
  __shared__ Blk blk[81];
  const int64_t el = blockIdx.x;
  if (el >= A.nel_local) return;
  {
    const int4 *src = reinterpret_cast<const int4 *>(A.topo + el);
    int4 *dst = reinterpret_cast<int4 *>(&T);
    for (int i = threadIdx.x; i < (int)(sizeof(ElemTopo) / 16); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  constexpr int S = Tr<DIM, SP>::S;
  if (threadIdx.x < S * 27) {
    const int s = threadIdx.x / 27, tau = threadIdx.x % 27;
    if (DIM == 2 && tau >= 9) blk[threadIdx.x].size = 0;
    else block_affine<DIM, SP>(A.p, s, tau, T, A.base, blk[threadIdx.x]);
  }
  __syncthreads();
  for (int l = threadIdx.x; l < A.ndpe; l += blockDim.x) {
    int s, x[3];
    decode_local<DIM, SP>(A.p, l, s, x);
    const int tr = row_tau<DIM, SP>(A.p, s, x);
    const Blk &B = blk[s * 27 + tr];
    A.map[el * A.ndpe + l] = B.g0 + B.str[0] * x[0] + B.str[1] * x[1] + B.str[2] * x[2];
    if (A.sign) A.sign[el * A.ndpe + l] = B.sigma;
  }
}

// ================================================================================ coordinate vectors
// The LOR mesh vertex coordinates AMS/ADS need: "Deduplicating this vector is
// performed efficiently using the element restriction degree of freedom index mappings ... with
// one thread per deduplicated DOF without requiring any MPI communication."  The E-vector at the
// GLL points holds exactly the LOR vertex coordinates (the GLL interpolation of the HO nodes is the
// identity for nodes given at the GLL points, reading P-27); each owned H1 dof is written once, by
// the minimal element containing its coarse entity (the same rule as A2, l.352) -- one thread per
// deduplicated dof, its index mapping from the element's affine blocks.
template <int DIM>
__global__ void __launch_bounds__(128) k_coords(CoordArgs A) {
  __shared__ ElemTopo T;
  __shared__ Blk blk[27];
  const int64_t el = blockIdx.x;
  if (el >= A.nel_local) return;
  {
    const int4 *src = reinterpret_cast<const int4 *>(A.topo + el);
    int4 *dst = reinterpret_cast<int4 *>(&T);
    for (int i = threadIdx.x; i < (int)(sizeof(ElemTopo) / 16); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  if (threadIdx.x < 27) {
    if (DIM == 2 && threadIdx.x >= 9) blk[threadIdx.x].size = 0;
    else block_affine<DIM, SP_H1>(A.p, 0, threadIdx.x, T, A.base, blk[threadIdx.x]);
  }
  __syncthreads();
  const int np = DIM == 3 ? (A.p + 1) * (A.p + 1) * (A.p + 1) : (A.p + 1) * (A.p + 1);
  const double *xe = A.X + el * A.xstride;
  for (int l = threadIdx.x; l < np; l += blockDim.x) {
    int s, x[3];
    decode_local<DIM, SP_H1>(A.p, l, s, x);
    const int tr = row_tau<DIM, SP_H1>(A.p, s, x);
    if ((T.flags[tr] & (TF_MIN | TF_OWNED)) != (TF_MIN | TF_OWNED)) continue;
    const Blk &B = blk[tr];
    const int64_t r = (int64_t)(B.g0 + B.str[0] * x[0] + B.str[1] * x[1] + B.str[2] * x[2]) - A.row_begin;
#pragma unroll
    for (int d = 0; d < DIM; ++d) __stcs(A.out + d * A.n_local + r, __ldcs(xe + d * np + l));
  }
}

// With the setup element restriction: one thread per (element, point) over the flat E-vector order --
// the point's global id from the restriction (coalesced), the writer test from its entity slot's
// flags in the element's topology record, its coordinates from the E-vector (coalesced).
template <int DIM>
__global__ void __launch_bounds__(256) k_coords_flat(CoordArgs A) {
  const int np1 = A.p + 1, npt = DIM == 3 ? np1 * np1 * np1 : np1 * np1;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= A.nel_local * npt) return;
  const int64_t e = t / npt;
  const int l = (int)(t - e * npt);
  const int x0 = l % np1, x1 = (l / np1) % np1, x2 = DIM == 3 ? l / (np1 * np1) : 0;
  auto cls = [&](int x) { return x == 0 ? 0 : (x == A.p ? 2 : 1); };
  const int tau = cls(x0) + 3 * cls(x1) + (DIM == 3 ? 9 * cls(x2) : 0);
  const uint8_t f = __ldg(&A.topo[e].flags[tau]);
  if ((f & (TF_MIN | TF_OWNED)) != (TF_MIN | TF_OWNED)) return;
  const int64_t r = (int64_t)__ldg(A.emap + t) - A.row_begin;
  const double *xe = A.X + e * A.xstride + l;
#pragma unroll
  for (int d = 0; d < DIM; ++d) __stcs(A.out + d * A.n_local + r, __ldg(xe + d * npt));
}

cudaError_t launch_coords(int dim, const CoordArgs &a, cudaStream_t st) {
  if (a.nel_local <= 0) return cudaSuccess;
  if (a.emap) {
    const int64_t n = a.nel_local * (dim == 3 ? (int64_t)(a.p + 1) * (a.p + 1) * (a.p + 1) : (int64_t)(a.p + 1) * (a.p + 1));
    if (dim == 2) k_coords_flat<2><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a);
    else k_coords_flat<3><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a);
    return cudaGetLastError();
  }
  if (dim == 2) k_coords<2><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
  else k_coords<3><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
  return cudaGetLastError();
}

// ================================================================================ dof transpose
// The dof -> (element, local dof) transpose of the element restriction (the paper's "inverse
// offsets" of the element restriction): rows = this rank's owned dofs, entries
// = local element * ndpe + local dof, ascending.  Count (integer atomics), scan (k_scan), fill
// (atomic cursor), then each row's few entries sorted in place (insertion sort; valence <= 255).
__global__ void k_tr_count(const int32_t *__restrict__ map, int64_t n_ent, int64_t row_begin, int64_t n_local,
                           int32_t *__restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_ent; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = (int64_t)__ldg(map + i) - row_begin;
    if (r >= 0 && r < n_local) atomicAdd(cnt + r, 1);
  }
}

__global__ void k_tr_fill(const int32_t *__restrict__ map, int64_t n_ent, int64_t row_begin, int64_t n_local,
                          const int64_t *__restrict__ off, int32_t *__restrict__ cursor, int32_t *__restrict__ ent) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_ent; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = (int64_t)__ldg(map + i) - row_begin;
    if (r >= 0 && r < n_local) ent[off[r] + atomicAdd(cursor + r, 1)] = (int32_t)i;
  }
}

__global__ void k_tr_sort(const int64_t *__restrict__ off, int64_t n_local, int32_t *__restrict__ ent) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_local; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = off[r], e = off[r + 1];
    for (int64_t a = s + 1; a < e; ++a) {
      const int32_t v = ent[a];
      int64_t b = a;
      while (b > s && ent[b - 1] > v) {
        ent[b] = ent[b - 1];
        --b;
      }
      ent[b] = v;
    }
  }
}

cudaError_t launch_transpose(const int32_t *map, int64_t n_ent, int64_t row_begin, int64_t n_local, int32_t *cnt,
                             int64_t *off, int32_t *ent, unsigned long long *status, unsigned int *tile_ctr,
                             cudaStream_t st) {
  const unsigned ge = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n_ent + 255) / 256, 148 * 16));
  const unsigned gr = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n_local + 255) / 256, 148 * 16));
  cudaError_t e;
  if (n_local > 0 && (e = cudaMemsetAsync(cnt, 0, sizeof(int32_t) * n_local, st)) != cudaSuccess) return e;
  k_tr_count<<<ge, 256, 0, st>>>(map, n_ent, row_begin, n_local, cnt);
  if ((e = launch_scan(cnt, off, n_local, status, tile_ctr, st)) != cudaSuccess) return e;
  if (n_local > 0 && (e = cudaMemsetAsync(cnt, 0, sizeof(int32_t) * n_local, st)) != cudaSuccess) return e;
  k_tr_fill<<<ge, 256, 0, st>>>(map, n_ent, row_begin, n_local, off, cnt, ent);
  k_tr_sort<<<gr, 256, 0, st>>>(off, n_local, ent);
  return cudaGetLastError();
}

// rows (stride doubles each) of X at the listed indices, packed into buf (ghost-layer coordinates
// of the extended frame sent to a peer rank)
__global__ void k_gather_rows(const double *__restrict__ X, int64_t stride, const int32_t *__restrict__ idx, int64_t n,
                              double *__restrict__ buf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * stride; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / stride, k = i - r * stride;
    buf[i] = X[(int64_t)idx[r] * stride + k];
  }
}

cudaError_t launch_gather_rows(const double *X, int64_t stride, const int32_t *idx, int64_t n, double *buf, cudaStream_t st) {
  const int64_t tot = n * stride;
  if (tot <= 0) return cudaSuccess;
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, 148 * 16));
  k_gather_rows<<<g, 256, 0, st>>>(X, stride, idx, n, buf);
  return cudaGetLastError();
}

__global__ void k_rowptr_stride(int64_t *row_ptr, int64_t n, int w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    row_ptr[i] = (int64_t)w * i;
}

cudaError_t launch_rowptr_stride(int64_t *row_ptr, int64_t n, int w, cudaStream_t st) {
  int64_t blocks = (n + 1 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_rowptr_stride<<<(unsigned)blocks, 256, 0, st>>>(row_ptr, n, w);
  return cudaGetLastError();
}

// ================================================================================ launchers
template <int DIM, int SP>
static cudaError_t launch_count_t(const CountArgs &a, int64_t grid, cudaStream_t st) {
  if (grid <= 0) return cudaSuccess;
  k_count<DIM, SP><<<(unsigned)grid, 128, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_count(int dim, int space, const CountArgs &a, cudaStream_t st) {
  if (dim == 2) return launch_count_t<2, SP_H1>(a, a.ntopo, st);
  if (space == SP_H1) return launch_count_t<3, SP_H1>(a, a.ntopo, st);
  if (space == SP_ND) return launch_count_t<3, SP_ND>(a, a.ntopo, st);
  return launch_count_t<3, SP_RT>(a, a.ntopo, st);
}

int64_t tab_slot_entries(int dim, int space) {
  if (dim == 2) return (int64_t)1 * NROWKEY * Tr<2, SP_H1>::W;
  if (space == SP_H1) return (int64_t)1 * NROWKEY * Tr<3, SP_H1>::W;
  if (space == SP_ND) return (int64_t)3 * NROWKEY * Tr<3, SP_ND>::W;
  return (int64_t)3 * NROWKEY * Tr<3, SP_RT>::W;
}
int64_t tab_size_entries(int dim, int space) {
  const int S = (dim == 2 || space == SP_H1) ? 1 : 3;
  return (int64_t)S * NROWKEY * tab_tzs(S * 27);
}

cudaError_t launch_build_tables(int dim, int space, int p, uint32_t *slot, uint8_t *size, uint32_t *pb, uint8_t *npb,
                                uint8_t *lex, cudaStream_t st) {
  if (dim == 2) k_build_tables<2, SP_H1><<<NROWKEY, 64, 0, st>>>(p, slot, size, pb, npb, lex);
  else if (space == SP_H1) k_build_tables<3, SP_H1><<<NROWKEY, 64, 0, st>>>(p, slot, size, pb, npb, lex);
  else if (space == SP_ND) k_build_tables<3, SP_ND><<<3 * NROWKEY, 64, 0, st>>>(p, slot, size, pb, npb, lex);
  else k_build_tables<3, SP_RT><<<3 * NROWKEY, 64, 0, st>>>(p, slot, size, pb, npb, lex);
  return cudaGetLastError();
}

cudaError_t launch_scan(const int32_t *cnt, int64_t *row_ptr, int64_t n, unsigned long long *status,
                        unsigned int *tile_ctr, cudaStream_t st) {
  const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  cudaMemsetAsync(status, 0, sizeof(unsigned long long) * (tiles + 1), st);
  cudaMemsetAsync(tile_ctr, 0, sizeof(unsigned int), st);
  k_scan<<<(unsigned)(tiles > 0 ? tiles : 1), SCAN_T, 0, st>>>(cnt, row_ptr, n, status, tile_ctr);
  return cudaGetLastError();
}

int64_t scan_status_words(int64_t n) { return (n + SCAN_TILE - 1) / SCAN_TILE + 1; }

// per-(dim, space, p) launchers live in generated translation units (build.py)
#define LOR_DECL_ASM(D, SPC, P) cudaError_t launch_asm_##D##_##SPC##_##P(const AsmArgs &, int, cudaStream_t, int *);
#define LOR_DECL_ALLP(D, SPC) LOR_DECL_ASM(D, SPC, 1) LOR_DECL_ASM(D, SPC, 2) LOR_DECL_ASM(D, SPC, 3) \
  LOR_DECL_ASM(D, SPC, 4) LOR_DECL_ASM(D, SPC, 5) LOR_DECL_ASM(D, SPC, 6) LOR_DECL_ASM(D, SPC, 7) LOR_DECL_ASM(D, SPC, 8)
LOR_DECL_ALLP(2, 0)
LOR_DECL_ALLP(3, 0)
LOR_DECL_ALLP(3, 1)
LOR_DECL_ALLP(3, 2)

#define LOR_SWITCH_P(D, SPC)                                          \
  switch (p) {                                                        \
    case 1: return launch_asm_##D##_##SPC##_1(a, quad, st, smem_out); \
    case 2: return launch_asm_##D##_##SPC##_2(a, quad, st, smem_out); \
    case 3: return launch_asm_##D##_##SPC##_3(a, quad, st, smem_out); \
    case 4: return launch_asm_##D##_##SPC##_4(a, quad, st, smem_out); \
    case 5: return launch_asm_##D##_##SPC##_5(a, quad, st, smem_out); \
    case 6: return launch_asm_##D##_##SPC##_6(a, quad, st, smem_out); \
    case 7: return launch_asm_##D##_##SPC##_7(a, quad, st, smem_out); \
    case 8: return launch_asm_##D##_##SPC##_8(a, quad, st, smem_out); \
    default: return cudaErrorInvalidValue;                            \
  }

cudaError_t launch_assemble(int dim, int space, int p, int quad, const AsmArgs &a, cudaStream_t st, int *smem_out) {
  if (dim == 2) { LOR_SWITCH_P(2, 0) }
  if (space == SP_H1) { LOR_SWITCH_P(3, 0) }
  if (space == SP_ND) { LOR_SWITCH_P(3, 1) }
  LOR_SWITCH_P(3, 2)
}

cudaError_t launch_finalize_list(const FinArgs &f, cudaStream_t st) {
  if (f.n <= 0) return cudaSuccess;
  cudaFuncSetAttribute(k_finalize_list, cudaFuncAttributeMaxDynamicSharedMemorySize, f.smem_bytes);
  k_finalize_list<<<(unsigned)f.n, 128, f.smem_bytes, st>>>(f);
  return cudaGetLastError();
}

cudaError_t launch_discrete(int which, const DiscArgs &a, cudaStream_t st) {
  if (a.nel_local <= 0) return cudaSuccess;
  if (which == 0) k_discrete<0><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
  else k_discrete<1><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_dofmap(int dim, int space, const DofmapArgs &a, cudaStream_t st) {
  if (a.nel_local <= 0) return cudaSuccess;
  if (dim == 2) k_dofmap<2, SP_H1><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
  else if (space == SP_H1) k_dofmap<3, SP_H1><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
  else if (space == SP_ND) k_dofmap<3, SP_ND><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
  else k_dofmap<3, SP_RT><<<(unsigned)a.nel_local, 128, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace lorb
