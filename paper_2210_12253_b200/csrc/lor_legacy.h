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

}  // namespace lorb
