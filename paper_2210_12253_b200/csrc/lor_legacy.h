// lor_legacy.h -- device side of the unstructured ("legacy") comparator (lor_legacy.cu); internal.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lorb {

struct LegArgs {
  int64_t n;                 // rows (owned H1 dofs)
  const int64_t *off;        // [n+1] dof -> (cell, corner) transpose offsets
  const int32_t *ent;        // cell * 8 + corner, ascending per row
  const int32_t *lmap;       // [ncell][8] LOR element restriction (global H1 ids)
  const double *ea;          // [ncell][8][8] element matrices
  const int64_t *row_ptr;    // fill pass
  int32_t *col;
  double *val;
  int32_t *cnt;              // count pass
};

cudaError_t launch_leg_mesh(int p, int64_t nel, const int32_t *emap, const double *X, int64_t xstride, int32_t *lmap,
                            double *lx, cudaStream_t st);
cudaError_t launch_leg_ea(int64_t ncell, int ncpe, const double *lx, double alpha, double beta, double *ea, int *err,
                          cudaStream_t st);
cudaError_t launch_leg_rows(const LegArgs &a, bool fill, cudaStream_t st);

// p = 1 vector spaces (sp = 1 ND, 2 RT) through the same per-row scheme: map / sgn = the space's
// element restriction and orientation signs (element = LOR cell at p = 1), ea = packed cell matrices
struct RvArgs {
  int64_t n;                 // owned rows
  const int64_t *off;        // [n + 1] dof -> (cell, local) transpose
  const int32_t *ent;        // flat index cell * K + local
  const int32_t *map;        // [ncell][K] global column ids
  const int8_t *sgn;         // [ncell][K] orientation signs
  const double *ea;          // [ncell][K(K+1)/2]
  const int64_t *row_ptr;
  int32_t *col;
  double *val;
  int32_t *cnt;
  int *err;
};
// X = the local E-vector (stride xstride per element; at p = 1 lattice point q is cell corner q)
cudaError_t launch_rv_ea(int sp, int64_t ncell, const double *X, int64_t xstride, double alpha, double beta, double *ea,
                         int *err, cudaStream_t st);
cudaError_t launch_rv_rows(int sp, const RvArgs &a, bool fill, cudaStream_t st);
int rv_dofs_per_cell(int sp);
int64_t rv_ea_words(int sp);

}  // namespace lorb
