// lor_xframe.h -- the extended-frame ("owner computes") H1 fill path (DESIGN.md §4 "k_xh1").
//
// Every element writes the complete CSR rows of the dofs it owns (the minimal element containing
// the dof's coarse entity), shared rows included: the LOR cells of the neighbouring
// macro elements that touch those rows are recomputed in the owner's own lattice frame extended by
// one cell layer on every side ("extended frame", lattice coordinates y in [-1, p+1]^3).  No
// partial rows, no merge pass, no value atomics.
//
// The extended frame needs a regular neighbourhood: the (up to) 26 elements around an element
// form a 3x3x3 block of hexes (any local orientations, any element numbering).  lor_setup checks
// this per mesh (xframe_build) and otherwise keeps the general element pass + merge pass.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "lor_internal.h"

namespace lorb {

// neighbour delta index: (dx+1) + 3 (dy+1) + 9 (dz+1); 13 = the element itself
struct XNbr {
  int32_t el;     // local element index, -1: no element there
  uint32_t code;  // bits 0-5: ax[a] (2 bits per neighbour-local axis a: the extended-frame axis it
                  // runs along); bits 6-8: sn[a] (1 = runs along -ax[a]); bits 9-14: o[k] + 1
                  // (2 bits per extended axis k: coarse position of the neighbour's local corner 0)
                  // => local lattice coordinate L_a = sn_a * (y[ax_a] - p * o[ax_a])
};

struct __align__(16) XElem {
  uint32_t own;      // bit tau: this element writes the rows of entity slot tau (TF_MIN & TF_OWNED)
  int8_t clo[3];     // cell box [clo, chi] per axis in extended-frame cell coordinates
  int8_t chi[3];
  int8_t olo[3];     // bounding box [olo, ohi] of the owned rows (lattice coordinates)
  int8_t ohi[3];
  XNbr nbr[27];
  int32_t el;        // the local element (records are stored in processing (CTA) order)
  uint8_t pad2[4];
};
static_assert(sizeof(XElem) == 240, "layout");

// extended-frame box table entry: points y with per-axis class (-1 | 0 | [1,p-1] | p | p+1) share
// one coarse entity of one element, so gid = g0 + sum_k s[k] y[k] (App. A numbering is affine)
struct XBox {
  int32_t g0;
  int8_t s[3];
  uint8_t valid;
};
static_assert(sizeof(XBox) == 8, "layout");

struct XSetupArgs {
  int64_t nel_local;
  const XElem *xe;      // [nel_local] in processing order (CTA b -> element xe[b].el); xmap, xhalo,
                        // box and piece below are stored in the same order
  const ElemTopo *topo;
  const int32_t *base[4];
  int64_t row_begin;
  XBox *box;           // [nel_local][125]
  int nb;              // cell-box extent the fill kernel is built for (p+1 or p+2)
  int32_t *xmap;       // [nel_local][(nb+1)^3] extended element restriction: global id of every point
                       // of the element's point box [clo, clo+nb]^3 (-1 outside [clo, chi+1])
  int2 *xhalo;         // [nel_local][(nb+1)^3 - (p+1)^3] coordinate gather list of the box points outside
                       // the element: {E-vector index of the x component (-1: outside [clo, chi+1]),
                       // point index in the box}
  int64_t xstride;
  int *err;            // set to 1 on any inconsistency
};

struct XFillArgs {
  int64_t nel_local, elem_begin;
  const int32_t *order;
  const XElem *xe;
  const int32_t *xmap;
  const int2 *xhalo;
  const double *X;
  int64_t xstride;
  int64_t row_begin;
  int32_t *cnt;                // k_xh1_sym output: row lengths [n_local]
  uint32_t *pos;               // k_xh1_sym output: [n_local][8] final position of each stencil slot
                               // (bytes 0-26, 255 = not a column)
  const int64_t *row_ptr;
  int32_t *col;
  double *val;
  double alpha, beta;
  const double *ca, *cb;       // variable coefficient E-vectors [nel_local][(p+1)^3] (NEXT-3) or null
  int ncx, ncy, ncz;  // max cell-box extents over the elements (shared-memory sizing)
  int *err;
  unsigned long long *tstamp;  // debug (LOR_PHASE_TIMING=1): per-CTA phase clocks, 16 per CTA
  int64_t pf_dist;             // L2 prefetch distance in CTAs (resident CTAs of the grid; 0: off)
  int values_only;             // 1: numeric-only re-assembly, col is not written (pattern reuse)
  int sort32;                  // 1: column ids - key_base < 2^26, the symbolic pass sorts packed 32-bit keys
  int key_base;                // smallest column id this rank's rows can reference (slab neighbour r - 1)
  uint8_t cperm[128];          // one-chunk kernels: thread -> box cell (>= ncell: none), set by the launcher
  uint8_t cinv[128];           // box cell -> thread (storage slot)
};

// ---- extended frame of the vector spaces (lor_xv.cu): Nedelec (SP_ND) and Raviart-Thomas (SP_RT).
// Family s: ND = edges along s (cell index along s, lattice point index along the other axes),
// RT = faces normal to s (point index along s, cell indices along the others).  Box positions of a
// family: per axis the cell range [clo, clo + nb - 1] (cell-index axes) or the point range
// [clo, clo + nb] (point-index axes), lexicographic.  Map entry: global id | 0x80000000 when the
// dof's global orientation is opposite to the extended frame's +axis orientation (sign -1);
// 0xffffffff = no dof there.
struct XvArgs {
  int64_t nel_local, elem_begin;
  const XElem *xe;             // shared with the H1 path (processing order)
  const int2 *xhalo;           // coordinate gather list (shared with the H1 path)
  const ElemTopo *topo;
  const int32_t *base[4];      // entity first-dof ids of this space
  uint32_t *xvmap;             // [nel_local][3][nvf] (setup)
  const double *X;
  int64_t xstride;
  int64_t row_begin;
  int32_t *cnt;                // symbolic pass: row lengths [n_local]
  uint32_t *pos;               // symbolic pass: [n_local][pw] final position of each stencil slot (bytes, 255 = none)
  const int64_t *row_ptr;
  int32_t *col;
  double *val;
  double alpha, beta;
  const double *ca, *cb;       // variable coefficient E-vectors [nel_local][(p+1)^3] (NEXT-3) or null
  int64_t pf_dist;             // L2 prefetch distance in CTAs (resident CTAs of the grid; 0: off)
  int ncx, ncy, ncz;
  int *err;
  int values_only;
  int sort32;                  // ids - key_base < 2^(31 - slot bits): sorting network on packed keys
  int key_base;                // smallest column id this rank's rows can reference (slab neighbour r - 1)
};
cudaError_t launch_xv_setup(int space, int p, const XvArgs &a, cudaStream_t st);
cudaError_t launch_xv_sym(int space, int p, const XvArgs &a, cudaStream_t st);
cudaError_t launch_xv_fill(int space, int p, const XvArgs &a, cudaStream_t st);
int xv_supported(int space, int p, const int cmax[3]);   // 1: a fill kernel is instantiated (smem fits)
int64_t xv_map_words(int space, int p, const int cmax[3]);  // per element
int xv_pos_words(int space);                              // per row

// host: regular-neighbourhood check and per-element extended-frame records.  nranks > 1 needs
// xghost: the ghost layer (sorted global ids of the non-local elements sharing a vertex with a local
// element) is returned there and neighbour indices >= n_elem_local refer to it.
struct HostPlan;
bool xframe_build(const HostPlan &plan, const int64_t *elem_vert, std::vector<XElem> &out, int cmax[3],
                  std::string *why, std::vector<int64_t> *xghost = nullptr);
std::vector<int64_t> xframe_ghosts(const HostPlan &plan, int rank);

// cell-box extent the fill kernel is instantiated for, and points per element of the extended map
inline int xfill_nb(int p, const int cmax[3]) {
  return (cmax[0] <= p + 1 && cmax[1] <= p + 1 && cmax[2] <= p + 1) ? p + 1 : p + 2;
}
inline int64_t xmap_points(int p, const int cmax[3]) {
  const int pb = xfill_nb(p, cmax) + 1;
  return (int64_t)pb * pb * pb;
}


cudaError_t launch_xh1_setup(int p, const XSetupArgs &a, cudaStream_t st);
cudaError_t launch_xh1_fill(int p, const XFillArgs &a, cudaStream_t st, int *smem_out);
cudaError_t launch_xh1_count(int p, const XFillArgs &a, cudaStream_t st);  // k_xh1_sym

}  // namespace lorb
