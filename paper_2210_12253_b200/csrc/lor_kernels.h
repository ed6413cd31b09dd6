// lor_kernels.h -- launch interface between the host runtime (lor_capi.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lor_internal.h"

namespace lorb {

struct CountArgs {
  int p, ndpe;
  int64_t ntopo;                 // local + ghost elements
  const ElemTopo *topo;
  const int32_t *base[4];        // entity first-dof ids (vertex, edge, face, interior)
  int64_t row_begin;
  int32_t *cnt;                  // [n_local] zero-initialised
};

struct AsmArgs {
  int64_t nel_local, elem_begin;
  const ElemTopo *topo;
  const ElemSpace *esp;
  const double *X;               // local E-vector, element stride xstride doubles
  int64_t xstride;
  const int32_t *base[4];
  int64_t row_begin;
  const int64_t *row_ptr;
  int32_t *col;
  double *val;
  RecEntry *scratch;
  int rstride;                   // entries per record
  const Ose *ose;
  const int32_t *ose_slots;
  int32_t *counters;
  double alpha, beta;
  int *err;                      // [0] code, [1] element, [2] cell
};

struct FinArgs {
  int n;                         // number of OSEs in list
  const int32_t *list;
  const Ose *ose;
  const int32_t *ose_slots;
  const RecEntry *scratch;
  int rstride;
  int64_t row_begin;
  const int64_t *row_ptr;
  int32_t *col;
  double *val;
  int smem_bytes;
};

struct DiscArgs {
  int p;
  int64_t nel_local;
  const ElemTopo *topo;
  const int32_t *base_row[4];
  const int32_t *base_col[4];
  int64_t row_begin;
  int32_t *col;
  double *val;
};

struct DofmapArgs {
  int p, ndpe;
  int64_t nel_local;
  const ElemTopo *topo;
  const int32_t *base[4];
  int32_t *map;
  int8_t *sign;
};

cudaError_t launch_count(int dim, int space, const CountArgs &a, cudaStream_t st);
cudaError_t launch_scan(const int32_t *cnt, int64_t *row_ptr, int64_t n, unsigned long long *status,
                        unsigned int *tile_ctr, cudaStream_t st);
int64_t scan_status_words(int64_t n);
// smem_out != NULL: only report the dynamic shared memory the kernel needs
cudaError_t launch_assemble(int dim, int space, int p, int quad, const AsmArgs &a, cudaStream_t st, int *smem_out);
cudaError_t launch_finalize_list(const FinArgs &f, cudaStream_t st);
cudaError_t launch_discrete(int which, const DiscArgs &a, cudaStream_t st);
cudaError_t launch_rowptr_stride(int64_t *row_ptr, int64_t n, int w, cudaStream_t st);
cudaError_t launch_dofmap(int dim, int space, const DofmapArgs &a, cudaStream_t st);

}  // namespace lorb
