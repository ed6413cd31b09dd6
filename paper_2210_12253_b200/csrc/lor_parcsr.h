// lor_parcsr.h -- device side of the ParCSR split and essential-BC elimination (lor_parcsr.cu);
// internal, not part of the public ABI (include/lor.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lorb {

// input CSR (local rows, global columns ascending) and the rank's column range
struct PcArgs {
  int64_t n;               // local rows
  const int64_t *rp;       // [n+1]
  const int32_t *col;      // global ids
  const double *val;
  int64_t cb, ce;          // owned column range [cb, ce)
  int64_t row_begin;       // global id of local row 0 (square operators: the diagonal column)
  int square;              // 1: diag block stores the diagonal first (hypre convention)
  const int64_t *croff;    // [nranks+1] column ownership ranges (device)
  int nranks;
  int64_t ncols;           // global columns (columns outside [0, ncols) are reported, not written)
  uint32_t *bitmap;        // [ceil(n_cols_global / 32)] offd columns
  const int64_t *wpre;     // [words+1] exclusive popcount prefix (fill)
  int32_t *cnt_d, *cnt_o;  // [n]
  uint32_t *rowmask;       // [n] owner ranks of the row's offd columns (bit q)
  int *err;                // 1: a square operator's row lacks its diagonal; 2: column out of range
};

struct PcOut {
  const int64_t *drp, *orp;
  int32_t *dcol, *ocol;
  double *dval, *oval;
};

struct BcArgs {
  int64_t n;
  const int64_t *drp, *orp;
  const int32_t *dcol;
  double *dval, *oval;
};

cudaError_t launch_pc_count(const PcArgs &a, cudaStream_t st);
cudaError_t launch_pc_popc(const uint32_t *bm, int64_t nw, int32_t *pc, cudaStream_t st);
cudaError_t launch_pc_colmap(const uint32_t *bm, const int64_t *wpre, int64_t nw, int64_t *colmap, cudaStream_t st);
cudaError_t launch_pc_peer_lo(const uint32_t *bm, const int64_t *wpre, int64_t nw, const int64_t *roff, int nranks,
                              int64_t *lo, cudaStream_t st);
cudaError_t launch_pc_flag(const uint32_t *rowmask, int64_t n, int q, int32_t *f, cudaStream_t st);
cudaError_t launch_pc_scatter(const uint32_t *rowmask, const int64_t *pos, int64_t n, int q, int32_t *list,
                              cudaStream_t st);
// mixed: some row has offd entries (nnz_offd > 0)
cudaError_t launch_pc_fill(const PcArgs &a, const PcOut &o, bool mixed, cudaStream_t st);
cudaError_t launch_bc_mark(const int32_t *ess, int64_t n_ess, int64_t n, uint8_t *marker, int *err, cudaStream_t st);
cudaError_t launch_bc_pack(const uint8_t *marker, const int32_t *list, int64_t n, uint8_t *buf, cudaStream_t st);
cudaError_t launch_bc_rows(const int32_t *ess, int64_t n_ess, const BcArgs &b, cudaStream_t st);
cudaError_t launch_bc_offd_cols(const int32_t *ocol, int64_t nnz_o, const uint8_t *omark, double *oval,
                                cudaStream_t st);

}  // namespace lorb
