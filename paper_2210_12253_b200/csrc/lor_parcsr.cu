// lor_parcsr.cu -- Steps A3/A4 of PAPER.md l.365-388 after the local assembly: the hypre-style
// parallel CSR split (diagonal block / off-diagonal block + col_map_offd, l.369-370) and the
// elimination of essential boundary conditions (l.376-388), as device kernels on the caller's
// CSR.  Host orchestration (marker exchange over NCCL, overlap) is in lor_capi.cu.
//
//   k_pc_count   per row: entries in the rank's own column range (diag) and outside (offd); offd
//                columns set bits of a global column bitmap, their owner ranks a per-row peer mask.
//                Columns are sorted ascending (reading P-5), so a row whose first and last column
//                are both owned has no offd entry (two loads).
//   k_pc_popc    popcount of every bitmap word (scanned by k_scan -> offd index of every word).
//   k_pc_colmap  col_map_offd: the set bits in ascending global order.
//   k_pc_fill_*  diag entries with local column ids (square operators: the diagonal first, the
//                others ascending -- hypre's ParCSR convention), offd entries with their index into
//                col_map_offd (rank of the column among the set bits); rows without offd entries
//                streamed 32 rows per warp, rows with offd entries one warp each.
//   k_bc_*       essential-dof elimination: marker of the owned essential
//                rows, the per-peer marker packs, rows + columns of the diag block and rows of the
//                offd block threaded over the essential dofs, then offd columns from the received
//                markers.
#include <cuda_runtime.h>
#include <stdint.h>

#include "lor_parcsr.h"

namespace lorb {

namespace {

__device__ __forceinline__ int owner_of(int64_t c, const int64_t *roff, int nranks) {
  int q = 0;
  for (int k = 1; k < nranks; ++k) q += (c >= roff[k]);
  return q;
}

__global__ void k_pc_count(PcArgs a) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.n) return;
  const int64_t s = a.rp[r], e = a.rp[r + 1];
  int cd = 0, co = 0;
  uint32_t mask = 0;
  bool has_diag = !a.square;
  const int64_t d = a.row_begin + r;
  if (e > s) {
    const int64_t c0 = a.col[s], c1 = a.col[e - 1];
    if (c0 >= a.cb && c1 < a.ce) {  // every column owned
      cd = (int)(e - s);
      if (a.square) {  // the diagonal must be among them (binary search, columns ascending)
        int64_t lo = s, hi = e - 1;
        while (lo < hi) {
          const int64_t m = (lo + hi) >> 1;
          if (a.col[m] < d) lo = m + 1;
          else hi = m;
        }
        has_diag = a.col[lo] == d;
      }
    } else {
      for (int64_t j = s; j < e; ++j) {
        const int64_t c = a.col[j];
        if (c >= a.cb && c < a.ce) {
          ++cd;
          has_diag = has_diag || c == d;
        } else if (c < 0 || c >= a.ncols) {
          atomicExch(a.err, 2);
        } else {
          ++co;
          atomicOr(a.bitmap + (c >> 5), 1u << (c & 31));
          mask |= 1u << owner_of(c, a.croff, a.nranks);
        }
      }
    }
  }
  if (a.square && !has_diag) atomicExch(a.err, 1);
  a.cnt_d[r] = cd;
  a.cnt_o[r] = co;
  a.rowmask[r] = mask;
}

__global__ void k_pc_popc(const uint32_t *bm, int64_t nw, int32_t *pc) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w < nw) pc[w] = __popc(bm[w]);
}

__global__ void k_pc_colmap(const uint32_t *bm, const int64_t *wpre, int64_t nw, int64_t *colmap) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nw) return;
  uint32_t b = bm[w];
  int64_t o = wpre[w];
  while (b) {
    const int k = __ffs(b) - 1;
    b &= b - 1;
    colmap[o++] = (w << 5) + k;
  }
}

// offd index of the first column >= bound for every rank boundary (the per-peer col_map segments)
__global__ void k_pc_peer_lo(const uint32_t *bm, const int64_t *wpre, int64_t nw, const int64_t *roff, int nranks,
                             int64_t *lo) {
  const int q = threadIdx.x;
  if (q > nranks) return;
  const int64_t b = roff[q], w = b >> 5;
  lo[q] = w >= nw ? wpre[nw] : wpre[w] + __popc(bm[w] & ((1u << (b & 31)) - 1u));
}

__global__ void k_pc_flag(const uint32_t *rowmask, int64_t n, int q, int32_t *f) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) f[r] = (rowmask[r] >> q) & 1u;
}

__global__ void k_pc_scatter(const uint32_t *rowmask, const int64_t *pos, int64_t n, int q, int32_t *list) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n && ((rowmask[r] >> q) & 1u)) list[pos[r]] = (int32_t)r;
}

// Rows without offd entries (every row on one rank; all but the slab-interface rows otherwise): one
// warp per 32 consecutive rows streams their contiguous entry range with all lanes (coalesced
// loads; the stores are shifted by at most one slot for the diagonal-first convention).  A lane's
// row follows from a cursor over the warp's 33 row offsets in shared memory.
__global__ void __launch_bounds__(256) k_pc_fill_flat(PcArgs a, PcOut o) {
  __shared__ int64_t s_rp[8][33], s_od[8][32];
  __shared__ int s_mixed[8][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = ((int64_t)blockIdx.x * 8 + w) * 32;
  if (r0 >= a.n) return;
  const int nr = a.n - r0 < 32 ? (int)(a.n - r0) : 32;
  if (lane < nr) {
    s_rp[w][lane] = a.rp[r0 + lane];
    s_od[w][lane] = o.drp[r0 + lane];
    s_mixed[w][lane] = a.cnt_o[r0 + lane];
  }
  if (lane == 0) s_rp[w][nr] = a.rp[r0 + nr];
  __syncwarp();
  const int64_t S = s_rp[w][0], E = s_rp[w][nr];
  int cur = 0;
  for (int64_t j = S + lane; j < E; j += 32) {
    while (j >= s_rp[w][cur + 1]) ++cur;
    if (s_mixed[w][cur]) continue;
    const int64_t r = r0 + cur, s = s_rp[w][cur];
    const int64_t c = __ldcs(a.col + j);
    const double x = __ldcs(a.val + j);
    const int64_t dc = a.row_begin + r, k = j - s;
    const int64_t pos = a.square ? (c == dc ? 0 : (c < dc ? k + 1 : k)) : k;
    __stcs(o.dcol + s_od[w][cur] + pos, (int32_t)(c - a.cb));
    __stcs(o.dval + s_od[w][cur] + pos, x);
  }
}

// Rows with offd entries: warp per row; lanes over the row's entries (columns ascending).
__global__ void __launch_bounds__(256) k_pc_fill_mixed(PcArgs a, PcOut o) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= a.n || a.cnt_o[r] == 0) return;
  const int64_t s = a.rp[r], e = a.rp[r + 1];
  const int64_t od = o.drp[r], oo = o.orp[r];
  const int64_t dc = a.row_begin + r;
  const uint32_t lt = (1u << lane) - 1u;
  int bd = 0, bo = 0;
  for (int64_t j0 = s; j0 < e; j0 += 32) {
    const int64_t j = j0 + lane;
    const bool v = j < e;
    const int64_t c = v ? (int64_t)__ldcs(a.col + j) : -1;
    const double x = v ? __ldcs(a.val + j) : 0.0;
    const bool isd = v && c >= a.cb && c < a.ce;
    const uint32_t md = __ballot_sync(0xffffffffu, isd), mo = __ballot_sync(0xffffffffu, v && !isd);
    if (isd) {
      const int kd = bd + __popc(md & lt);
      const int pos = a.square ? (c == dc ? 0 : (c < dc ? kd + 1 : kd)) : kd;
      __stcs(o.dcol + od + pos, (int32_t)(c - a.cb));
      __stcs(o.dval + od + pos, x);
    } else if (v) {
      const int ko = bo + __popc(mo & lt);
      const int64_t w = c >> 5;
      const int64_t loc = a.wpre[w] + __popc(a.bitmap[w] & ((1u << (c & 31)) - 1u));
      __stcs(o.ocol + oo + ko, (int32_t)loc);
      __stcs(o.oval + oo + ko, x);
    }
    bd += __popc(md);
    bo += __popc(mo);
  }
}

__global__ void k_bc_mark(const int32_t *ess, int64_t n_ess, int64_t n, uint8_t *marker, int *err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_ess) return;
  const int32_t j = ess[i];
  if (j < 0 || j >= n) atomicExch(err, 1);
  else marker[j] = 1;
}

__global__ void k_bc_pack(const uint8_t *marker, const int32_t *list, int64_t n, uint8_t *buf) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) buf[i] = marker[list[i]];
}

// warp per essential row j: diag row j -> (1 on the diagonal, 0 elsewhere); for every other column
// k of that row the entry (k, j) of row k is zeroed (the LOR pattern is structurally symmetric:
// pairs of dofs sharing a LOR cell, reading P-3); offd row j -> 0.  Concurrent writers of one entry
// all write 0.0, the diagonal is written only by its own row's warp.
__global__ void __launch_bounds__(256) k_bc_rows(const int32_t *ess, int64_t n_ess, BcArgs b) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n_ess) return;
  const int32_t j = ess[i];
  if (j < 0 || j >= b.n) return;
  const int64_t s = b.drp[j], e = b.drp[j + 1];
  for (int64_t t = s + lane; t < e; t += 32) {
    const int32_t k = b.dcol[t];
    if (k == j) {
      b.dval[t] = 1.0;
    } else {
      b.dval[t] = 0.0;
      int64_t lo = b.drp[k] + 1, hi = b.drp[k + 1] - 1;  // row k: diagonal first, the rest ascending
      while (lo < hi) {
        const int64_t m = (lo + hi) >> 1;
        if (b.dcol[m] < j) lo = m + 1;
        else hi = m;
      }
      if (lo <= hi && b.dcol[lo] == j) b.dval[lo] = 0.0;
    }
  }
  for (int64_t t = b.orp[j] + lane; t < b.orp[j + 1]; t += 32) b.oval[t] = 0.0;
}

__global__ void k_bc_offd_cols(const int32_t *ocol, int64_t nnz_o, const uint8_t *omark, double *oval) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nnz_o && omark[ocol[t]]) oval[t] = 0.0;
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t > 0 ? (n + t - 1) / t : 1); }

}  // namespace

cudaError_t launch_pc_count(const PcArgs &a, cudaStream_t st) {
  if (a.n > 0) k_pc_count<<<nblk(a.n, 256), 256, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_pc_popc(const uint32_t *bm, int64_t nw, int32_t *pc, cudaStream_t st) {
  if (nw > 0) k_pc_popc<<<nblk(nw, 256), 256, 0, st>>>(bm, nw, pc);
  return cudaGetLastError();
}
cudaError_t launch_pc_colmap(const uint32_t *bm, const int64_t *wpre, int64_t nw, int64_t *colmap, cudaStream_t st) {
  if (nw > 0) k_pc_colmap<<<nblk(nw, 256), 256, 0, st>>>(bm, wpre, nw, colmap);
  return cudaGetLastError();
}
cudaError_t launch_pc_peer_lo(const uint32_t *bm, const int64_t *wpre, int64_t nw, const int64_t *roff, int nranks,
                              int64_t *lo, cudaStream_t st) {
  k_pc_peer_lo<<<1, 64, 0, st>>>(bm, wpre, nw, roff, nranks, lo);
  return cudaGetLastError();
}
cudaError_t launch_pc_flag(const uint32_t *rowmask, int64_t n, int q, int32_t *f, cudaStream_t st) {
  if (n > 0) k_pc_flag<<<nblk(n, 256), 256, 0, st>>>(rowmask, n, q, f);
  return cudaGetLastError();
}
cudaError_t launch_pc_scatter(const uint32_t *rowmask, const int64_t *pos, int64_t n, int q, int32_t *list,
                              cudaStream_t st) {
  if (n > 0) k_pc_scatter<<<nblk(n, 256), 256, 0, st>>>(rowmask, pos, n, q, list);
  return cudaGetLastError();
}
cudaError_t launch_pc_fill(const PcArgs &a, const PcOut &o, bool mixed, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  k_pc_fill_flat<<<nblk(a.n, 256), 256, 0, st>>>(a, o);
  if (mixed) k_pc_fill_mixed<<<nblk(a.n * 32, 256), 256, 0, st>>>(a, o);
  return cudaGetLastError();
}
cudaError_t launch_bc_mark(const int32_t *ess, int64_t n_ess, int64_t n, uint8_t *marker, int *err, cudaStream_t st) {
  if (n_ess > 0) k_bc_mark<<<nblk(n_ess, 256), 256, 0, st>>>(ess, n_ess, n, marker, err);
  return cudaGetLastError();
}
cudaError_t launch_bc_pack(const uint8_t *marker, const int32_t *list, int64_t n, uint8_t *buf, cudaStream_t st) {
  if (n > 0) k_bc_pack<<<nblk(n, 256), 256, 0, st>>>(marker, list, n, buf);
  return cudaGetLastError();
}
cudaError_t launch_bc_rows(const int32_t *ess, int64_t n_ess, const BcArgs &b, cudaStream_t st) {
  if (n_ess > 0) k_bc_rows<<<nblk(n_ess * 32, 256), 256, 0, st>>>(ess, n_ess, b);
  return cudaGetLastError();
}
cudaError_t launch_bc_offd_cols(const int32_t *ocol, int64_t nnz_o, const uint8_t *omark, double *oval,
                                cudaStream_t st) {
  if (nnz_o > 0) k_bc_offd_cols<<<nblk(nnz_o, 256), 256, 0, st>>>(ocol, nnz_o, omark, oval);
  return cudaGetLastError();
}

}  // namespace lorb
