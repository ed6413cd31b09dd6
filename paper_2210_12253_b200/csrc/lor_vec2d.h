// lor_vec2d.h -- device side of the 2D Nedelec / Raviart-Thomas path (lor_vec2d.cu); internal.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lor_internal.h"

namespace lorb {

struct V2Args {
  int p;
  int64_t ncell;
  const double *X;          // E-vector [nel][2][(p+1)^2], element stride xstride
  int64_t xstride;
  const double *ca, *cb;    // variable coefficients [nel][(p+1)^2] or null
  double alpha, beta;
  const int8_t *csgn;       // [ncell][4] dof signs
  double *ea;               // [ncell][16] signed cell matrices
  int *err;
};

struct V2Rows {
  int64_t n;
  const int64_t *off;       // dof -> (cell * 4 + local) transpose
  const int32_t *ent;
  const int32_t *cmap;      // [ncell][4] global dof ids
  const double *ea;
  const int64_t *row_ptr;
  int32_t *col;
  double *val;
  int32_t *cnt;
};

struct V2Disc {
  int sp, p;
  int64_t nel, row_begin;
  const int32_t *rmap;      // [nel][2p(p+1)] ND / RT element restriction
  const int8_t *rsgn;
  const uint8_t *writer;    // the minimal element containing the dof writes its row
  const int32_t *hmap;      // [nel][(p+1)^2] H1 element restriction
  int32_t *col;
  double *val;
};

cudaError_t launch_v2_cells(int sp, int p, int64_t nel, const int32_t *emap, const int8_t *esgn, int32_t *cmap,
                            int8_t *csgn, cudaStream_t st);
cudaError_t launch_v2_ea(int sp, int quad, const V2Args &a, cudaStream_t st);
cudaError_t launch_v2_rows(const V2Rows &a, bool fill, cudaStream_t st);
cudaError_t launch_v2_disc(const V2Disc &a, cudaStream_t st);

}  // namespace lorb
