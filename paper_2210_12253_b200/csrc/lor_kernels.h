// lor_kernels.h -- launch interface between the host runtime (lor_capi.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lor_internal.h"

namespace lorb {

// Row-class tables (built once at setup by k_build_tables): a row's stencil
// structure depends only on its sub-lattice s and, per axis, on (min(x,2), min(ext-1-x,2)) -- the
// "row key" rk in [0, 729).  Per (s, rk):
//   slot[W]  : bit 0 valid | bits 1-7 column block b' = s'*27 + tau' | bits 8-12 join slot tau_J |
//              bits 13+4a.. : offset (2 bits) and length-1 (2 bits) of the column inside its
//              block's sub-box along axis a (for the lexicographic rank inside the sub-box)
//   size[NB] : size of the sub-box of block b' in the row's stencil (0 if absent)
//   pb[NB], npb : compact list of present blocks: b' | tau_J << 7 | size << 12
constexpr int NROWKEY = 729;
// byte stride of a row of the block-size table (16-byte aligned rows for vector loads)
// merge plan row of a shared entity with k contributors, per final column position q:
// [k x i32 record row of contributor m (local element * ndpe + its local row)]
// [W x u16 holder mask over contributors] (pad to 4 B) [W x i32 global column]
// [W x k u8: slot j of q in holder m's natural record | 64 if the column dof is sign-flipped in m
// (255 none)] (pad to 16 B)
__host__ __device__ constexpr int plan_col_off(int k, int W) { return (4 * k + 2 * W + 3) & ~3; }
__host__ __device__ constexpr int plan_row_bytes(int k, int W) { return (plan_col_off(k, W) + 4 * W + W * k + 15) & ~15; }

// one shared (merged) row for the merge pass
struct MergeRow {
  int64_t plan_off;              // byte offset of the row's plan row
  int32_t g;                     // local row index
  int32_t k;                     // contributors
};

// own-row position table row (bytes): whole 16-byte vectors
__host__ __device__ constexpr int own_w(int W) { return (W + 15) / 16 * 16; }

__host__ __device__ constexpr int tab_tzs(int nb) { return (nb + 15) / 16 * 16; }
struct Tabs {
  const uint32_t *slot;
  const uint8_t *size;
  const uint32_t *pb;
  const uint8_t *npb;
  const uint8_t *lex;   // [S][729][W][8]: rank of the slot's column inside its block's sub-box, per
                        // orientation code (ElemTopo::orient) of the column block's entity
};

struct CountArgs {
  int p, ndpe;
  int64_t ntopo;                 // local + ghost elements
  const ElemTopo *topo;
  const int32_t *base[4];        // entity first-dof ids (vertex, edge, face, interior)
  int64_t row_begin;
  int32_t *cnt;                  // [n_local] zero-initialised
  Tabs tabs;
};

struct AsmArgs {
  int64_t nel_local, elem_begin;
  const double *ca = nullptr, *cb = nullptr;  // variable coefficients: E-vectors [nel_local][(p+1)^dim] (NEXT-3)
  const int32_t *order;          // CTA -> local element (Morton order of element centroids), or NULL
  const ElemTopo *topo;
  const ElemSpace *esp;
  const double *X;               // local E-vector, element stride xstride doubles
  int64_t xstride;
  const int32_t *base[4];
  Tabs tabs;
  int64_t row_begin;
  const int64_t *row_ptr;
  int32_t *col;
  double *val;
  RecEntry *scratch;
  int rstride;                   // entries per record
  const Ose *ose;
  const int32_t *ose_slots;
  // shared rows whose contributors are all local: every contributor
  // writes its partial row in natural stencil-slot order; the last one to arrive emits the row
  double *nval;                  // [nel_local][NDPE][rec_w8(W)] natural-order partial rows (row sign applied)
  const int32_t *ose_elem;       // per OSE slot (ose_slots order): local index of the contributing element
  const int64_t *pbase;          // [n_ose] byte offset of the OSE's merge-plan rows
  const uint8_t *plan;           // per OSE row: k x uint16 contributor local rows, then W x k slot bytes
  int maxl;
  int plan_mode;                 // 1: setup plan pass (partial-row records of every shared row, no CSR
                                 //    output)
                                 // 2: setup own-row position pass (final position of every stencil slot of
                                 //    every own row -> ownpos)
  const int64_t *ownbase;        // [nel_local] first own-row ordinal of the element
  uint8_t *ownpos;               // [own rows][own_w(W)] slot -> position in the CSR row (255: not a column)
  double alpha, beta;
  int *err;                      // [0] code, [1] element, [2] cell
  unsigned long long *tstamp;    // optional [grid][16] per-CTA phase clocks (LOR_PHASE_TIMING=1)
  int dbg;                       // dev experiments (LOR_DBG bits; 0 in production)
  // one-rank assembly: the element restriction (global id and orientation sign of every local dof)
  // from setup (lor_setup runs k_dofmap once; reused like the HO element restriction, PAPER.md
  // l.537), so the element pass skips its block-table prologue.  NULL: computed per element.
  const int32_t *emap = nullptr; // [nel_local][NDPE]
  const int8_t *esgn = nullptr;  // [nel_local][NDPE] +-1
  int64_t pf_dist = 0;           // L2 prefetch of the prologue data of CTA blockIdx + pf_dist (0: off)
};

struct PlanArgs {
  int n;                         // number of OSEs
  const Ose *ose;
  const int32_t *ose_slots;
  const uint8_t *is_defer;       // [n_ose]
  const RecEntry *scratch;       // plan-mode records: entries (col, block base, slot index as double),
                                 // header (len, local row)
  int rstride, W;
  const int64_t *pbase;
  const int32_t *ose_elem;       // local element of every contributor
  int ndpe;
  uint8_t *plan;
};

// merge pass of the natural-order partial rows of shared rows: one warp per row
struct MergeArgs {
  int64_t n;                     // merged rows
  int W, W8;
  const MergeRow *rows;
  const uint8_t *plan;
  const double *nval;
  const int64_t *row_ptr;
  int32_t *col;
  double *val;
};

struct FinArgs {
  int n;                         // number of OSEs in list
  const int32_t *list;
  const Ose *ose;
  const int32_t *ose_slots;
  const RecEntry *scratch;
  int rstride, maxl, maxu;
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

// discrete gradient / curl from the element restrictions (rows: ND / RT, columns: H1 / ND)
struct DiscMapArgs {
  int p;
  int64_t nel_local;
  const ElemTopo *topo;
  const int32_t *rmap;  // [nel_local][ndpe_row]
  const int8_t *rsgn;
  const int32_t *cmap;  // [nel_local][ndpe_col]
  const int8_t *csgn;   // curl only
  int64_t row_begin;
  int32_t *col;
  double *val;
  int64_t *row_ptr = nullptr;  // written in the same pass (row_ptr[i] = w i, w = 2 / 4), or null
  int64_t n_rows = 0;
};

struct DofmapArgs {
  int p, ndpe;
  int64_t nel_local;
  const ElemTopo *topo;
  const int32_t *base[4];
  int32_t *map;
  int8_t *sign;
};

// LOR vertex coordinate vectors: E-vector -> owned H1 dofs
struct CoordArgs {
  int p;
  int64_t nel_local;
  const ElemTopo *topo;
  const int32_t *base[4];
  const double *X;   // E-vector [local element][dim][(p+1)^dim], element stride xstride
  int64_t xstride;
  int64_t row_begin, n_local;
  double *out;       // [dim][n_local]
  const int32_t *emap = nullptr;  // H1 element restriction [nel_local][(p+1)^dim] (setup), or NULL
};
cudaError_t launch_coords(int dim, const CoordArgs &a, cudaStream_t st);

cudaError_t launch_count(int dim, int space, const CountArgs &a, cudaStream_t st);
// table sizes (entries) and builder
int64_t tab_slot_entries(int dim, int space);
int64_t tab_size_entries(int dim, int space);
cudaError_t launch_build_tables(int dim, int space, int p, uint32_t *slot, uint8_t *size, uint32_t *pb, uint8_t *npb,
                                uint8_t *lex, cudaStream_t st);
cudaError_t launch_scan(const int32_t *cnt, int64_t *row_ptr, int64_t n, unsigned long long *status,
                        unsigned int *tile_ctr, cudaStream_t st);
int64_t scan_status_words(int64_t n);
// smem_out != NULL: only report the dynamic shared memory the kernel needs
cudaError_t launch_assemble(int dim, int space, int p, int quad, const AsmArgs &a, cudaStream_t st, int *smem_out);
cudaError_t launch_finalize_list(const FinArgs &f, cudaStream_t st);
cudaError_t launch_plan_merge(const PlanArgs &a, int n_ose, cudaStream_t st);
cudaError_t launch_merge_rows(const MergeArgs &a, cudaStream_t st);
cudaError_t launch_discrete(int which, const DiscArgs &a, cudaStream_t st);
cudaError_t launch_discrete_map(int which, const DiscMapArgs &a, cudaStream_t st);
cudaError_t launch_rowptr_stride(int64_t *row_ptr, int64_t n, int w, cudaStream_t st);
cudaError_t launch_gather_rows(const double *X, int64_t stride, const int32_t *idx, int64_t n, double *buf, cudaStream_t st);
cudaError_t launch_dofmap(int dim, int space, const DofmapArgs &a, cudaStream_t st);
// dof -> (local element * ndpe + local dof) transpose of an element restriction map[n_ent] for the
// owned rows [row_begin, row_begin + n_local): off[n_local+1], ent[off[n_local]] ascending per row.
// Launches 4 kernels (count, scan, fill, sort).
cudaError_t launch_transpose(const int32_t *map, int64_t n_ent, int64_t row_begin, int64_t n_local, int32_t *cnt,
                             int64_t *off, int32_t *ent, unsigned long long *status, unsigned int *tile_ctr,
                             cudaStream_t st);

}  // namespace lorb
