/*
 * lor.h -- C ABI of the B200-native batched low-order-refined (LOR) assembly library
 * (liblor_b200.so).  arXiv 2210.12253, Step S1.2 "Low-order-refined matrix assembly"
 * and its auxiliary discrete operators (l.390-445, Algorithm 1).
 *
 * Problem statement: a user holds a degree-p bilinear form on a
 * conforming quad/hex mesh and asks for "the LOR discretization ... assembled ... in parallel
 * CSR format", plus the discrete gradient (AMS) and discrete curl (ADS).
 *
 * Conventions (all entry points):
 *   * Ownership.  Host inputs are copied during lor_setup; the caller may free them on return.
 *     Outputs go into CALLER-ALLOCATED DEVICE buffers whose sizes come from lor_query*.  The
 *     library never frees caller memory.  Internal workspaces live in the context and are
 *     released by lor_destroy.
 *   * Errors.  Every call returns a lor_status; nothing throws or aborts across the ABI.
 *     lor_last_error(ctx) gives a message (including element / sub-cell for geometry errors).
 *   * Asynchrony.  Assembly calls are enqueued on the context's CUDA stream and return without
 *     synchronising.  Device-side errors (det J <= 0) are reported by lor_sync.  lor_query* are
 *     synchronous host calls whose values are fixed at setup (the pattern is topological).
 *   * Threads.  A context is not thread-safe; one context per rank (process) per GPU.
 *   * Index widths.  col is int32 of GLOBAL ids (n_global < 2^31); row_ptr is int64 and
 *     LOCAL (row_ptr[0] = 0); each rank owns the contiguous global rows
 *     [row_begin, row_begin + n_rows_local) (ParCSR convention).
 *   * Pattern.  Structural: every pair of dofs sharing a LOR cell, explicit zeros kept; both
 *     triangles; columns ascending within each row (readings P-3/P-4/P-5).
 *   * Numbering / orientation / signs: DESIGN.md "Numbering": vertices, then
 *     edges, faces, element interiors; rank-major renumbering by owner = rank of the minimal
 *     element containing the dof.
 */
#ifndef LOR_B200_H
#define LOR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lor_ctx_s *lor_ctx; /* opaque, one per GPU / rank */

typedef enum { LOR_H1 = 0, LOR_ND = 1, LOR_RT = 2 } lor_space;
/* sub-cell quadrature (reading P-1): vertex = tensor 2-point Gauss-Lobatto
 * (geometric factors at the sub-element vertices); gauss2 = tensor 2-point Gauss */
typedef enum { LOR_QUAD_VERTEX = 0, LOR_QUAD_GAUSS2 = 1 } lor_quad;

typedef enum {
  LOR_OK = 0,
  LOR_ERR_INVALID_ARGUMENT = 1,
  LOR_ERR_DEGENERATE_GEOMETRY = 2,
  LOR_ERR_OUT_OF_MEMORY = 3,
  LOR_ERR_CUDA = 4,
  LOR_ERR_NCCL = 5,
  LOR_ERR_UNSUPPORTED = 6,
  LOR_ERR_BUFFER_TOO_SMALL = 7
} lor_status;

typedef struct {
  int dim;                      /* 2 or 3                                                     */
  int p;                        /* polynomial degree, 1 <= p <= 8                             */
  int64_t n_vert;               /* coarse vertices                                            */
  const double *vert_xyz;       /* HOST [n_vert][dim] (used only when elem_nodes == NULL)      */
  int64_t n_elem;               /* coarse (macro) elements, GLOBAL count                       */
  const int64_t *elem_vert;     /* HOST [n_elem][2^dim], local corner order a + 2b + 4c;
                                   every rank passes the whole mesh (the coarse mesh is small) */
  const double *elem_nodes;     /* HOST [n_elem][dim][(p+1)^dim]: the high-order coordinate
                                   E-vector at the tensor Gauss-Lobatto points (PAPER.md
                                   l.342-345).  Only this rank's elements are read.  NULL =>
                                   (bi/tri)linear interpolation of vert_xyz at GLL points.     */
  int rank, nranks;             /* this process and the job size                              */
  const int64_t *elem_rank_begin; /* HOST [nranks+1] contiguous element ranges per rank;
                                   NULL allowed when nranks == 1                              */
  const void *nccl_unique_id;   /* HOST 128-byte ncclUniqueId from lor_nccl_get_unique_id on
                                   rank 0, broadcast by the caller; NULL when nranks == 1      */
  void *cuda_stream;            /* cudaStream_t for all work (NULL = legacy default stream)    */
  int device;                   /* CUDA device ordinal of this rank                            */
  int space_mask;               /* bit s set: set up space s (H1 = 1, ND = 2, RT = 4; H1 always);
                                   0 = all.  The element + merge passes keep per-element buffers of
                                   every local dof, so skipping unused spaces saves device memory on
                                   large meshes (48^3 elements at p = 8: > 100 GB for ND + RT). */
} lor_setup_args;

/* Caller-owned DEVICE buffers.  cap_nnz = capacity of col/val (entries); row_ptr must hold
 * n_rows_local + 1 entries. */
typedef struct {
  int64_t *row_ptr;
  int32_t *col;
  double *val;
  int64_t cap_nnz;
} lor_csr;

/* Setup (untimed in the paper's sense, "reuse of the element restriction"):
 * coarse topology, canonical numbering + signs, ownership, rank-major ids, per-element
 * topology records, interface exchange plan and NCCL communicator, device uploads.
 * Errors: INVALID_ARGUMENT (dim, p, null pointers, inconsistent ranks, n_global >= 2^31,
 * negative corner orientation), OUT_OF_MEMORY, CUDA, NCCL. */
lor_status lor_setup(const lor_setup_args *args, lor_ctx *out);
lor_status lor_destroy(lor_ctx ctx);

/* Waits on the context stream; returns DEGENERATE_GEOMETRY if any sub-cell had det J <= 0
 * in an earlier call (message names element and sub-cell), CUDA on launch failures. */
lor_status lor_sync(lor_ctx ctx);
/* Message of the last failure on ctx; lor_last_error(NULL) returns the message of this thread's last
 * failed lor_setup / lor_plan_dry_run (which have no context to hold it). */
const char *lor_last_error(lor_ctx ctx);

/* Sizes of the assembled operator of `space` on this rank (synchronous, fixed at setup). */
lor_status lor_query(lor_ctx ctx, lor_space space, int64_t *n_rows_local, int64_t *row_begin,
                     int64_t *n_rows_global, int64_t *nnz_local);
/* which = 0: discrete gradient (rows: owned ND dofs, cols: global H1 dofs);
 * which = 1: discrete curl (rows: owned RT dofs, cols: global ND dofs; dim == 3);
 * which = 2: rotated gradient (rows: RT dofs, cols: H1 dofs; dim == 2, one rank). */
lor_status lor_query_discrete(lor_ctx ctx, int which, int64_t *n_rows_local, int64_t *nnz_local,
                              int64_t *n_cols_global);

/* LOR matrix assembly, Steps A1-A3: per macro element the p^d sub-cell
 * matrices at GLL-point geometry (A1), the processor-local CSR with row counts, scan and
 * column/value fill (A2), and on nranks > 1 the interface exchange over NCCL that replaces the
 * P^T A P triple product (A3).  Forms: H1 alpha grad.grad + beta mass; ND alpha curl.curl +
 * beta mass; RT alpha div.div + beta mass (constant coefficients, reading P-2).
 * ND/RT with dim == 2 (NEXT-2; reading P-29): one rank (UNSUPPORTED
 * otherwise), lattice-edge dofs, scalar curl / divergence, assembled from the signed 4x4 cell
 * matrices (lor_vec2d.cu).  Output: row_ptr[n_rows_local+1], col/val[nnz_local]. */
lor_status lor_assemble_h1(lor_ctx ctx, double alpha, double beta, lor_quad quad, lor_csr *out);
lor_status lor_assemble_nd(lor_ctx ctx, double alpha, double beta, lor_quad quad, lor_csr *out);
lor_status lor_assemble_rt(lor_ctx ctx, double alpha, double beta, lor_quad quad, lor_csr *out);

/* Numeric-only re-assembly (pattern reuse; "mesh motion or time-dependent
 * variable coefficients"): `out` must hold the row_ptr / col written by an earlier
 * lor_assemble_<space> call of this context with the same quadrature rule (the pattern is
 * topological); only the values are recomputed from the current coordinates and alpha, beta.  No
 * row lengths, no scan; on the extended-frame H1 path col is not written.  Same errors as
 * lor_assemble_<space>; the caller guarantees the buffers are unchanged since that call. */
lor_status lor_reassemble_h1(lor_ctx ctx, double alpha, double beta, lor_quad quad, lor_csr *out);
lor_status lor_reassemble_nd(lor_ctx ctx, double alpha, double beta, lor_quad quad, lor_csr *out);
lor_status lor_reassemble_rt(lor_ctx ctx, double alpha, double beta, lor_quad quad, lor_csr *out);

/* Discrete gradient, Algorithm 1: row i (owned ND dof) has -sigma_i at the
 * H1 id of the edge's local tail and +sigma_i at its head, columns sorted; row_ptr[i] = 2i.
 * Discrete curl: row f (owned RT dof) has +-1 on its 4 LOR edges
 * (right-hand-rule circulation about the face's global normal, in each edge's global
 * orientation), columns sorted; row_ptr[f] = 4f.  No communication. */
lor_status lor_discrete_grad(lor_ctx ctx, lor_csr *out);
lor_status lor_discrete_curl(lor_ctx ctx, lor_csr *out);
/* 2D rotated gradient grad-perp = (-d/dy, d/dx): H1 -> H(div) for grad-div problems with AMS (PAPER.md
 * l.409-410): row of an RT dof = +-1 at the H1 ids of its lattice edge's end points, the flux of
 * grad-perp u through the edge (u at the head minus u at the tail of the tangent that turns into the
 * dof's normal by +90 degrees), times the dof's sign; row_ptr[f] = 2f.  dim == 2, one rank. */
lor_status lor_discrete_rotgrad(lor_ctx ctx, lor_csr *out);

/* Element restriction of `space` for this rank's elements:
 * elem_dofs[n_elem_local][ndof_per_el] global ids in the macro-element local order of
 * DESIGN.md, signs[...] in {-1,+1} (NULL allowed; must be NULL-or-valid for H1).
 * DEVICE buffers.  n_elem_local = elem_rank_begin[rank+1] - elem_rank_begin[rank]. */
lor_status lor_dof_map(lor_ctx ctx, lor_space space, int32_t *elem_dofs, int8_t *signs);
/* Transpose of the element restriction (the dof -> element "inverse offsets", PAPER.md l.412-415
 * and SURVEY 8(b)): for every owned row r (local index, [0, n_rows_local)) the list of
 * (local element * ndof_per_el + local dof) pairs of this rank's elements whose dof is r, in
 * ascending order: entries[offsets[r] .. offsets[r+1]).  offsets[n_rows_local+1] int64, entries
 * int32, both caller-owned DEVICE buffers; cap_entries >= lor_query_transpose's count, else
 * BUFFER_TOO_SMALL with nothing written.  On one rank this is the complete transpose; on several
 * ranks it lists the pairs of the rank's own elements only.  Enqueued on the context stream
 * (count, scan, fill, per-row sort).  INVALID_ARGUMENT if n_elem_local * ndof_per_el >= 2^31. */
lor_status lor_query_transpose(lor_ctx ctx, lor_space space, int64_t *n_entries);
lor_status lor_dof_transpose(lor_ctx ctx, lor_space space, int64_t *offsets, int32_t *entries, int64_t cap_entries);
lor_status lor_query_elements(lor_ctx ctx, int64_t *elem_begin, int64_t *n_elem_local, int *ndof_per_el_h1,
                              int *ndof_per_el_nd, int *ndof_per_el_rt);

/* Replace this rank's coordinate E-vector (mesh motion / per-step inputs):
 * elem_nodes = [n_elem_local][dim][(p+1)^dim] for elements elem_rank_begin[rank] .. +n_elem_local,
 * HOST (pinned for asynchrony) or DEVICE memory; enqueued on the context stream.  With nranks > 1
 * and an NCCL communicator the extended frame's ghost layer (neighbour elements of other ranks)
 * is then refreshed from the peers (grouped ncclSend/ncclRecv on the same stream; every rank must
 * call it).  In LOR_EXCHANGE_MANUAL mode the ghost layer keeps the coordinates given at setup. */
lor_status lor_update_coordinates(lor_ctx ctx, const double *elem_nodes);

/* Variable coefficients ("definite Helmholtz", l.546 "time-dependent
 * variable coefficients"; reading P-28): alpha_e / beta_e = coefficient E-vectors
 * [n_elem_local][(p+1)^dim] at the GLL points (= the LOR vertices, the layout of elem_nodes), HOST or
 * DEVICE, copied on the context stream.  Subsequent lor_assemble_* / lor_reassemble_* integrate
 * alpha * a(x) (grad | curl | div part) and beta * b(x) (mass part), a and b sampled at the LOR
 * vertices: the corner value under the vertex rule, the multilinear interpolant of the cell's corner
 * values at the Gauss points under Gauss-2.  Both NULL: back to constant coefficients.  With
 * variable coefficients every space takes the element + merge passes (lor_fill_path returns 0).
 * INVALID_ARGUMENT if exactly one pointer is NULL. */
lor_status lor_set_coefficients(lor_ctx ctx, const double *alpha_e, const double *beta_e);
/* The same from the GLOBAL coefficient E-vectors [n_elem][(p+1)^dim] (HOST, every rank passes the
 * whole mesh's, as elem_nodes at setup): the context also keeps the coefficients of its ghost layer,
 * so on several ranks H1 and RT keep the extended-frame single pass with variable coefficients
 * (lor_set_coefficients alone: the element + merge passes there).  Synchronous. */
lor_status lor_set_coefficients_global(lor_ctx ctx, const double *alpha_all, const double *beta_all);

/* Unstructured ("legacy") comparator -- NOT the product path:
 * the LOR mesh treated as an arbitrary low-order hex mesh.  lor_legacy_setup builds the explicit LOR
 * element restriction (8 global H1 ids per LOR cell), the LOR coordinates in broken per-cell format
 * and the dof -> (cell, corner) transpose (the overhead l.604-606 says "can dominate"; synchronous).
 * lor_legacy_assemble_h1 then, per call, computes the dense 8x8 matrix of every LOR cell (vertex rule,
 * alpha grad.grad + beta mass) and assembles the global CSR directly from them: per row the 8 x 8
 * candidate (column, value) pairs of its cells ranked by column, row lengths, scan, then columns
 * ascending with duplicates summed -- the same matrix as lor_assemble_h1 (vertex rule) up to
 * rounding.  3D, one rank; UNSUPPORTED otherwise.  Phases in lor_last_phase_ms: element matrices,
 * count + scan, fill. */
lor_status lor_legacy_setup(lor_ctx ctx);
lor_status lor_legacy_assemble_h1(lor_ctx ctx, double alpha, double beta, lor_csr *out);

/* Exchange mode for nranks > 1 (A3 replacement).  LOR_EXCHANGE_NCCL (0, default when
 * nccl_unique_id was given): ncclSend/ncclRecv of interface partial rows inside the assembly call.
 * LOR_EXCHANGE_MANUAL (1, default without a unique id): single-process emulation of several ranks
 * (e.g. tests on one GPU) -- the assembly call stops before the exchange; the caller moves each
 * peer's partial rows with lor_exchange_copy(dst, src, space) and completes dst's rows with
 * lor_assemble_finish.  Both modes run the same kernels on the same buffers. */
lor_status lor_set_exchange(lor_ctx ctx, int mode);
lor_status lor_exchange_copy(lor_ctx dst, lor_ctx src, lor_space space);
lor_status lor_assemble_finish(lor_ctx ctx, lor_space space, lor_csr *out);

/* Host-only dry run of lor_setup's plan for one rank (no GPU touched): per space s = 0..2,
 * info[8*s + 0..7] = {valid, n_global, row_begin, n_rows_local, n_records, n_shared_owned,
 * n_deferred (owned shared entities with remote contributors), n_ghost_elements};
 * send_counts / recv_counts [3][nranks] = partial-row records exchanged with each peer (NULL ok).
 * Used by the multi-rank CPU tests (gloo) to check that the ranks' plans agree. */
lor_status lor_plan_dry_run(const lor_setup_args *args, int64_t *info, int64_t *send_counts, int64_t *recv_counts);

/* Host-only dry run of the extended frame for one rank (no GPU; dim == 3): info[0] = 1 if every
 * local element has a regular 3x3x3 neighbourhood (the single-pass path applies), info[1] = ghost
 * layer size (non-local elements sharing a vertex with a local one; their coordinates are held
 * after the local ones), info[2] = largest cell-box extent, info[3] = local elements;
 * send_counts / recv_counts[nranks] = elements whose coordinates this rank sends to / receives
 * from each peer when the coordinates change (lor_update_coordinates, NCCL).  NULL allowed. */
lor_status lor_xframe_dry_run(const lor_setup_args *args, int64_t *info, int64_t *send_counts, int64_t *recv_counts);

/* Diagnostics: copy internal setup tables of `space` to host memory (what = 0: row-class slot
 * table uint32[S][729][W]; 1: block-size table uint8[S][729][3*27 or 27]; 2: per-CTA phase clocks
 * uint64[n_elem_local][16] of the last element pass, only if LOR_PHASE_TIMING=1 at setup).  Returns bytes copied
 * (0 on error / cap too small). */
int64_t lor_debug_dump(lor_ctx ctx, int what, lor_space space, void *host_out, int64_t cap_bytes);

/* ---- Steps A3 (layout) and A4 after the local assembly --------------------
 * hypre-style parallel CSR of an assembled operator ("Each rank has a diagonal
 * block, which contains the nonzeros for which both the row and column indices are owned by
 * itself, and an off-diagonal block, which contains the nonzeros for which the column indices are
 * owned by another rank").  Rows: this rank's owned rows.  diag: int32 column ids LOCAL to the
 * rank's column range; for the square operators (H1, ND, RT) the diagonal entry comes first in
 * every row and the others follow in ascending order (hypre's ParCSR convention, DESIGN.md reading
 * P-26); for G and C all ascending.  offd: int32 indices into col_map_offd, which lists the
 * distinct off-rank global columns in ascending order (int64).  All DEVICE, caller-owned. */
typedef struct {
  int64_t *diag_row_ptr; /* [n_rows_local + 1] */
  int32_t *diag_col;
  double *diag_val;
  int64_t cap_diag;      /* capacity of diag_col / diag_val (entries)                           */
  int64_t *offd_row_ptr; /* [n_rows_local + 1] */
  int32_t *offd_col;
  double *offd_val;
  int64_t cap_offd;
  int64_t *col_map_offd;
  int64_t cap_col_map;
} lor_parcsr;

/* Operators for lor_parcsr_*: 0 = H1, 1 = ND, 2 = RT (the matrices of lor_assemble_*, 2D included), 3 =
 * discrete gradient (rows ND, columns H1), 4 = discrete curl (rows RT, columns ND; 3D), 5 = rotated
 * gradient (rows RT, columns H1; 2D). */
enum { LOR_OP_H1 = 0, LOR_OP_ND = 1, LOR_OP_RT = 2, LOR_OP_GRAD = 3, LOR_OP_CURL = 4, LOR_OP_ROTGRAD = 5 };

/* Symbolic part of the split of the assembled operator A (row_ptr / col as written by the
 * assembly call, DEVICE): per-row diag / offd counts and their scans, the off-rank column set and,
 * for square operators on several ranks, the marker-exchange plan of lor_eliminate_bc.
 * SYNCHRONOUS (waits on the context stream); returns the sizes the caller allocates.  Errors:
 * UNSUPPORTED (operator not available, nranks > 32), INVALID_ARGUMENT (a square operator's row
 * lacks its diagonal), OUT_OF_MEMORY, CUDA.  The workspaces stay in the context for _fill and
 * lor_eliminate_bc of the same operator. */
lor_status lor_parcsr_prepare(lor_ctx ctx, int op, const lor_csr *A, int64_t *nnz_diag, int64_t *nnz_offd,
                              int64_t *n_col_offd);
/* Numeric part: copies A's values into the diag / offd blocks (enqueued on the context stream).
 * A must hold the same pattern as at lor_parcsr_prepare.  BUFFER_TOO_SMALL if a capacity is below
 * the prepared size (nothing written). */
lor_status lor_parcsr_fill(lor_ctx ctx, int op, const lor_csr *A, lor_parcsr *out);

/* The owned essential dofs of a trace condition on the whole domain boundary: local rows
 * (ascending) of the dofs of every coarse entity on a boundary facet (a face -- an edge in 2D --
 * of exactly one element): H1 all trace dofs, ND tangential edge dofs, RT normal face dofs
 * ("rows and columns corresponding to each essential degree of freedom").
 * *n = count; rows = DEVICE int32[cap] or NULL (count only); BUFFER_TOO_SMALL if cap < *n. */
lor_status lor_boundary_dofs(lor_ctx ctx, lor_space space, int32_t *rows, int64_t cap, int64_t *n);

/* Step A4, elimination of essential boundary conditions on the ParCSR M of
 * operator `space` (filled by lor_parcsr_fill): for every essential dof j (ess = DEVICE int32 local
 * rows of this rank, duplicates allowed) row j becomes the unit row (diagonal 1, every other stored
 * entry 0 in diag and offd) and column j becomes 0 in every other row of every rank; the pattern is
 * kept (explicit zeros).  On several ranks the markers of the owned essential dofs are sent to the
 * ranks whose offd blocks hold those columns (grouped ncclSend/ncclRecv on a side stream, started
 * before the diag / offd-row elimination and overlapped with it, l.383-386), then the offd columns
 * are zeroed from the received markers (l.386-387).  Collective over the ranks (NCCL mode).  In
 * LOR_EXCHANGE_MANUAL mode the call stops before the offd columns: the caller moves the markers
 * with lor_bc_exchange_copy(dst, src, space) for every pair and completes with
 * lor_eliminate_bc_finish.  ess entries outside [0, n_rows_local) are skipped and reported by the
 * next lor_sync as INVALID_ARGUMENT. */
lor_status lor_eliminate_bc(lor_ctx ctx, lor_space space, const int32_t *ess, int64_t n_ess, lor_parcsr *M);
lor_status lor_bc_exchange_copy(lor_ctx dst, lor_ctx src, lor_space space);
lor_status lor_eliminate_bc_finish(lor_ctx ctx, lor_space space, lor_parcsr *M);
/* Marker-exchange plan of a prepared square operator: per peer, markers sent / received
 * (host arrays [nranks], NULL allowed).  The plan is symmetric by construction; tests check
 * send_counts[q] on rank r == recv_counts[r] on rank q. */
lor_status lor_parcsr_exchange_counts(lor_ctx ctx, lor_space space, int64_t *send_counts, int64_t *recv_counts);

/* LOR mesh vertex coordinate vectors for AMS / ADS: the
 * coordinates of every owned H1 dof (= LOR vertex) deduplicated from the coordinate E-vector through
 * the element restriction, one thread per deduplicated dof, no communication.  xyz = DEVICE
 * double[dim][n_rows_local(H1)] (x of all owned vertices, then y, then z -- hypre's separate
 * coordinate vectors), caller-owned; enqueued on the context stream.  Bit-exact copies. */
lor_status lor_coordinates(lor_ctx ctx, double *xyz);

/* Rank 0 creates the NCCL unique id (128 bytes) that the caller broadcasts to all ranks. */
lor_status lor_nccl_get_unique_id(void *out128);

/* Number of this library's kernels launched on the context since setup (instrumentation). */
int64_t lor_kernel_launches(lor_ctx ctx);

/* Per-phase device timing of the last assembly call in milliseconds (count+scan, element pass
 * k_assemble, merge pass k_merge_rows, exchange+finalize); valid after lor_sync.  Returns number of
 * phases written (<= 8). */
int lor_last_phase_ms(lor_ctx ctx, float *ms, int cap);

/* Which value-fill path lor_assemble_<space> takes with the vertex rule: 1 = extended-frame
 * single pass (per call: row lengths k_xh1_count, scan, then every element writes the complete
 * rows it owns, column positions derived from its extended restriction and the
 * neighbour cells that touch its rows recomputed; 3D H1, one rank, meshes whose elements all have
 * a regular 3x3x3 coarse neighbourhood -- checked at setup; ND / RT on one rank at the orders where
 * it measured faster, LOR_XV=1 forces it wherever it fits), 0 = element pass + merge pass, 2 = per-row
 * path (3D, p = 1, one rank, constant coefficients, vertex rule, every space: a macro-element is a
 * single LOR cell; dense cell matrices (H1 8x8, ND 12x12, RT 6x6, orientation signs applied), one
 * warp per row gathers its <= 64 candidates through the dof -> cell transpose and writes them in
 * ascending column order, duplicates summed; LOR_ROWPATH=0 at setup turns it off).
 * LOR_XFRAME=0 in the environment at setup forces 0.  Returns -1 for an invalid context/space. */
int lor_fill_path(lor_ctx ctx, lor_space space);

#ifdef __cplusplus
}
#endif
#endif /* LOR_B200_H */
