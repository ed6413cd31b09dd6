// lor_capi.cu -- C ABI (include/lor.h) of the B200 LOR library: context, device memory, launch
// orchestration on the caller's stream, NCCL point-to-point exchange of interface partial rows.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/lor.h"
#include "lor_internal.h"
#include "lor_kernels.h"
#include "lor_legacy.h"
#include "lor_parcsr.h"
#include "lor_plan.h"
#include "lor_vec2d.h"
#include "lor_xframe.h"

// ---- minimal NCCL ABI (loaded with dlopen only when nranks > 1) ----------------------------------
typedef struct ncclComm *ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef enum { ncclInt8 = 0, ncclChar = 0, ncclUint8 = 1 } ncclDataType_t;

namespace {

struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  bool load(std::string &err) {
    if (h) return true;
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) { err = "cannot dlopen libnccl.so.2"; return false; }
#define LOAD(sym, name)                                          \
  sym = reinterpret_cast<decltype(sym)>(dlsym(h, name));         \
  if (!sym) { err = std::string("missing NCCL symbol ") + name; return false; }
    LOAD(GetUniqueId, "ncclGetUniqueId");
    LOAD(CommInitRank, "ncclCommInitRank");
    LOAD(CommDestroy, "ncclCommDestroy");
    LOAD(Send, "ncclSend");
    LOAD(Recv, "ncclRecv");
    LOAD(GroupStart, "ncclGroupStart");
    LOAD(GroupEnd, "ncclGroupEnd");
    LOAD(GetErrorString, "ncclGetErrorString");
#undef LOAD
    return true;
  }
};
NcclApi g_nccl;

using namespace lorb;

struct SpaceDev {
  bool valid = false;
  int ndpe = 0, maxl = 0, rstride = 0;
  int64_t n_global = 0, row_begin = 0, n_local = 0, nnz_local = 0;
  int32_t *base[4] = {nullptr, nullptr, nullptr, nullptr};
  ElemSpace *esp = nullptr;
  Ose *ose = nullptr;
  int32_t *ose_slots = nullptr, *defer = nullptr;
  int n_ose = 0, n_defer = 0;
  MergeRow *mrows = nullptr;  // merge-pass rows
  int64_t *ownbase = nullptr;  // own-row position table: first row per element
  uint8_t *ownpos = nullptr;
  int64_t n_own = 0;
  int64_t n_mrows = 0;
  RecEntry *scratch = nullptr;
  int64_t n_records = 0;
  int32_t *cnt = nullptr;
  unsigned long long *scan_status = nullptr;
  unsigned int *tile_ctr = nullptr;
  std::vector<int64_t> recv_begin, recv_count, send_begin, send_count;
  int pending_exchange = 0;  // manual exchange mode: assembly waiting for lor_assemble_finish
  uint32_t *tslot = nullptr, *tpb = nullptr;
  uint8_t *tsize = nullptr, *tnpb = nullptr, *tlex = nullptr;
  int W = 0;
  // shared rows: natural-order partial rows and the setup merge plan
  double *nval = nullptr;
  int32_t *ose_elem = nullptr;
  int64_t *pbase = nullptr;
  uint8_t *plan = nullptr, *is_defer = nullptr;
  // extended-frame fill path (lor_xframe.h; H1, 3D, one rank, regular neighbourhoods)
  bool xok = false;
  XElem *xe = nullptr;
  XBox *xbox = nullptr;
  int32_t *xmap = nullptr;
  int2 *xhalo = nullptr;
  // one rank: element restriction of the element pass (k_dofmap at setup), NULL otherwise
  int32_t *emap = nullptr;
  int8_t *esgn = nullptr;
  // p = 1 per-row path of the vector spaces (lor_setup): dof -> (cell, local) transpose, cell matrices
  int64_t *rv_off = nullptr;
  int32_t *rv_ent = nullptr;
  double *rv_ea = nullptr;
  bool rv = false;
  int xc[3] = {0, 0, 0};
  uint32_t *xpos = nullptr;     // extended-frame path: per-call slot positions [n_local][8]
  // extended-frame path of ND / RT (lor_xv.cuh): restriction of the box dofs, per-call positions
  bool xvok = false;
  uint32_t *xvmap = nullptr;
  uint32_t *xvpos = nullptr;
  int64_t n_tr = 0;             // entries of the dof transpose (local elements x owned local dofs)
  int32_t *trmap = nullptr;     // element restriction workspace of lor_dof_transpose (nranks > 1)
  std::vector<int64_t> rank_off;  // [nranks+1] row ranges of the ranks (column ownership)
  int64_t *droff = nullptr;       // device copy
  std::vector<int32_t> bnd;       // owned boundary rows (local, ascending; lor_boundary_dofs)
  int64_t key_lo = 0, key_hi = 0; // column-id range of the extended-frame restriction (sort keys)
};

// ParCSR split (A3 layout) and essential-BC elimination (A4, l.376-388) of one
// operator (H1, ND, RT, discrete gradient, discrete curl): workspaces of lor_parcsr_prepare, reused
// by lor_parcsr_fill and lor_eliminate_bc.
struct PcState {
  bool ready = false;
  int64_t n = 0, cb = 0, ce = 0, row_begin = 0, ncols = 0, nw = 0;
  int64_t nnz_d = 0, nnz_o = 0, n_col_offd = 0;
  int square = 0;
  const int64_t *croff = nullptr;
  uint32_t *bitmap = nullptr, *rowmask = nullptr;
  int32_t *pc = nullptr, *cnt_d = nullptr, *cnt_o = nullptr, *flag = nullptr;
  int64_t *wpre = nullptr, *drp = nullptr, *orp = nullptr, *pos = nullptr;
  unsigned long long *status = nullptr;
  unsigned int *tile_ctr = nullptr;
  // marker exchange (square operators): rows whose markers each peer needs (ascending local rows,
  // peer-major), and each peer's segment of col_map_offd (ascending: the same order on both sides)
  std::vector<int64_t> send_off, send_cnt, recv_lo;
  int32_t *send_list = nullptr;
  uint8_t *marker = nullptr, *sbuf = nullptr, *omark = nullptr;
  int64_t cap_send = 0, cap_send_b = 0, cap_omark = 0;
  int pending = 0;  // manual mode: offd columns wait for lor_eliminate_bc_finish
};

}  // namespace

struct lor_ctx_s {
  int dim = 0, p = 0, rank = 0, nranks = 1, device = 0;
  int64_t nel = 0, elem_begin = 0, nel_local = 0, ntopo = 0;
  cudaStream_t stream = nullptr;
  ElemTopo *topo = nullptr;
  int32_t *order = nullptr;  // CTA -> local element, Morton order of element centroids
  std::vector<int32_t> order_host;  // host copy (empty: natural order)
  double *X = nullptr;           // local elements, then the extended frame's ghost layer (nranks > 1)
  int64_t xstride = 0;
  // extended frame on several ranks: ghost layer (non-local elements sharing a vertex with a local
  // one), their topology records after the local ones, and the per-peer coordinate exchange lists
  int64_t n_xghost = 0;
  ElemTopo *xtopo = nullptr;
  std::vector<int64_t> xg_send_count, xg_recv_begin, xg_recv_count;  // per peer (elements)
  int32_t *xg_send_idx = nullptr;  // local element of every sent E-vector (peer-major)
  double *xg_send_buf = nullptr;
  SpaceDev sp[3];
  int *err = nullptr;
  unsigned long long *tstamp = nullptr;  // per-CTA phase clocks of the last element pass (debug)
  ncclComm_t comm = nullptr;
  int exchange_mode = 0;  // 0 NCCL, 1 manual
  std::string last_error;
  int64_t launches = 0;
  cudaEvent_t ev[8] = {};
  int nphase = 0;
  int fin_smem = 0;
  int dbg = 0;  // LOR_DBG at setup (dev experiments; 0 in production)
  std::vector<void *> allocs;
  PcState pc[6];                     // lor_parcsr_* / lor_eliminate_bc per operator
  double *ca = nullptr, *cb = nullptr;  // variable coefficient E-vectors (lor_set_coefficients)
  bool vc_ghosts = false;               // ca / cb also hold the ghost layer (lor_set_coefficients_global)
  double *ca_l = nullptr, *cb_l = nullptr, *ca_g = nullptr, *cb_g = nullptr;  // local-only / with ghosts
  std::vector<int64_t> xghost_ids;      // global ids of the ghost-layer elements (after the local ones)
  // unstructured comparator (lor_legacy_*): LOR element restriction, broken LOR coordinates, element
  // matrices, dof -> (cell, corner) transpose
  int64_t leg_ncell = 0;
  int32_t *leg_lmap = nullptr, *leg_ent = nullptr;
  double *leg_lx = nullptr, *leg_ea = nullptr;
  int64_t *leg_off = nullptr;
  bool h1_rows = false;  // p = 1, one rank: H1 through the per-row path (lor_setup)
  // 2D Nedelec / Raviart-Thomas (lor_vec2d.cu, one rank): per space the element restriction with
  // signs, the row writers of the discrete operators, the LOR cells' signed dofs, the dof -> cell
  // transpose, the cell matrices, sizes and the boundary dofs
  struct Vec2 {
    bool ok = false;
    int64_t n = 0, nnz = 0, ncell = 0;
    int32_t *map = nullptr, *cmap = nullptr, *ent = nullptr, *cnt = nullptr;
    int8_t *sgn = nullptr, *csgn = nullptr;
    uint8_t *writer = nullptr;
    int64_t *off = nullptr, *rp = nullptr;
    double *ea = nullptr;
    std::vector<int32_t> bnd;
    int64_t *droff = nullptr;  // {0, n}: the one rank's row range (ParCSR)
  } v2[3];
  bool vc = false;
  cudaStream_t side = nullptr;       // marker exchange stream (overlap)
  cudaEvent_t ev_pack = nullptr, ev_xchg = nullptr;
};

namespace {

// local rows of space `space` on entity slot tau (axis classes 0 min, 1 interior, 2 max)
int64_t class_rows(int dim, int space, int p, int tau) {
  const int cls[3] = {tau % 3, (tau / 3) % 3, tau / 9};
  const int S = space == 0 ? 1 : 3;
  int64_t tot = 0;
  for (int s2 = 0; s2 < S; ++s2) {
    int64_t n = 1;
    for (int a = 0; a < 3; ++a) {
      if (a >= dim) { n *= cls[a] == 0 ? 1 : 0; continue; }
      const bool vk = space == 0 ? true : (space == 1 ? a != s2 : a == s2);
      n *= vk ? (cls[a] == 1 ? p - 1 : 1) : (cls[a] == 1 ? p : 0);
    }
    tot += n;
  }
  return tot;
}

// message of the last failed lor_setup / lor_plan_dry_run (no context exists then), per thread
thread_local std::string g_setup_error;

lor_status fail(lor_ctx c, lor_status st, const std::string &msg) {
  if (c) c->last_error = msg;
  return st;
}

#define CUDA_TRY(ctx, expr)                                                                  \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return fail(ctx, _e == cudaErrorMemoryAllocation ? LOR_ERR_OUT_OF_MEMORY : LOR_ERR_CUDA, \
                  std::string(#expr) + ": " + cudaGetErrorString(_e));                       \
  } while (0)

template <class T>
cudaError_t dev_upload(lor_ctx c, T **dst, const T *src, size_t n) {
  *dst = nullptr;
  if (n == 0) return cudaSuccess;
  cudaError_t e = cudaMalloc((void **)dst, sizeof(T) * n);
  if (e != cudaSuccess) return e;
  c->allocs.push_back(*dst);
  return cudaMemcpy(*dst, src, sizeof(T) * n, cudaMemcpyHostToDevice);
}
template <class T>
cudaError_t dev_alloc(lor_ctx c, T **dst, size_t n) {
  *dst = nullptr;
  if (n == 0) return cudaSuccess;
  cudaError_t e = cudaMalloc((void **)dst, sizeof(T) * n);
  if (e != cudaSuccess) return e;
  c->allocs.push_back(*dst);
  return cudaMemset(*dst, 0, sizeof(T) * n);
}

void fill_base(const SpaceDev &S, const int32_t *out[4]) {
  for (int t = 0; t < 4; ++t) out[t] = S.base[t];
}

lor_status run_count_scan(lor_ctx c, int s, int64_t *row_ptr) {
  SpaceDev &S = c->sp[s];
  if (S.n_local > 0) CUDA_TRY(c, cudaMemsetAsync(S.cnt, 0, sizeof(int32_t) * S.n_local, c->stream));
  CountArgs ca;
  ca.p = c->p;
  ca.ndpe = S.ndpe;
  ca.ntopo = c->ntopo;
  ca.topo = c->topo;
  fill_base(S, ca.base);
  ca.row_begin = S.row_begin;
  ca.cnt = S.cnt;
  ca.tabs = Tabs{S.tslot, S.tsize, S.tpb, S.tnpb, S.tlex};
  CUDA_TRY(c, launch_count(c->dim, s, ca, c->stream));
  c->launches++;
  CUDA_TRY(c, launch_scan(S.cnt, row_ptr, S.n_local, S.scan_status, S.tile_ctr, c->stream));
  c->launches++;
  return LOR_OK;
}

lor_status exchange_nccl(lor_ctx c, int s) {
  SpaceDev &S = c->sp[s];
  const size_t rb = (size_t)S.rstride * sizeof(RecEntry);
  if (g_nccl.GroupStart() != ncclSuccess) return fail(c, LOR_ERR_NCCL, "ncclGroupStart");
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) continue;
    if (S.send_count[q] > 0) {
      ncclResult_t r = g_nccl.Send(reinterpret_cast<char *>(S.scratch) + S.send_begin[q] * rb, S.send_count[q] * rb,
                                   ncclUint8, q, c->comm, c->stream);
      if (r != ncclSuccess) { g_nccl.GroupEnd(); return fail(c, LOR_ERR_NCCL, g_nccl.GetErrorString(r)); }
    }
    if (S.recv_count[q] > 0) {
      ncclResult_t r = g_nccl.Recv(reinterpret_cast<char *>(S.scratch) + S.recv_begin[q] * rb, S.recv_count[q] * rb,
                                   ncclUint8, q, c->comm, c->stream);
      if (r != ncclSuccess) { g_nccl.GroupEnd(); return fail(c, LOR_ERR_NCCL, g_nccl.GetErrorString(r)); }
    }
  }
  if (g_nccl.GroupEnd() != ncclSuccess) return fail(c, LOR_ERR_NCCL, "ncclGroupEnd");
  return LOR_OK;
}

lor_status finish(lor_ctx c, int s, lor_csr *out) {
  SpaceDev &S = c->sp[s];
  FinArgs f;
  f.n = S.n_defer;
  f.list = S.defer;
  f.ose = S.ose;
  f.ose_slots = S.ose_slots;
  f.scratch = S.scratch;
  f.rstride = S.rstride;
  f.maxl = S.maxl;
  f.maxu = S.W;
  f.row_begin = S.row_begin;
  f.row_ptr = out->row_ptr;
  f.col = out->col;
  f.val = out->val;
  f.smem_bytes = c->fin_smem;
  CUDA_TRY(c, launch_finalize_list(f, c->stream));
  if (f.n > 0) c->launches++;
  return LOR_OK;
}

XFillArgs xfill_args(lor_ctx c, const SpaceDev &S) {
  XFillArgs x{};
  x.nel_local = c->nel_local;
  x.elem_begin = c->elem_begin;
  x.order = c->order;
  x.xe = S.xe;
  x.xmap = S.xmap;
  x.xhalo = S.xhalo;
  x.X = c->X;
  x.xstride = c->xstride;
  x.row_begin = S.row_begin;
  x.cnt = S.cnt;
  x.pos = S.xpos;
  // keys relative to the lowest column id the rank's extended restriction references (setup)
  const int64_t klo = S.key_lo, khi = S.key_hi;
  x.key_base = (int)klo;
  x.sort32 = (khi - klo < (int64_t(1) << 26) && !(c->dbg & 1)) ? 1 : 0;  // LOR_DBG bit 0: force the rank path
  x.ncx = S.xc[0];
  x.ncy = S.xc[1];
  x.ncz = S.xc[2];
  x.err = c->err;
  x.tstamp = c->tstamp;
  return x;
}

XvArgs xv_args(lor_ctx c, int s) {
  const SpaceDev &H = c->sp[SP_H1];
  const SpaceDev &S = c->sp[s];
  XvArgs x{};
  x.nel_local = c->nel_local;
  x.elem_begin = c->elem_begin;
  x.xe = H.xe;
  x.xhalo = H.xhalo;
  x.topo = c->xtopo ? c->xtopo : c->topo;
  fill_base(S, x.base);
  x.xvmap = S.xvmap;
  x.X = c->X;
  x.xstride = c->xstride;
  x.row_begin = S.row_begin;
  x.cnt = S.cnt;
  x.pos = S.xvpos;
  x.ncx = H.xc[0];
  x.ncy = H.xc[1];
  x.ncz = H.xc[2];
  x.err = c->err;
  const int sb = s == SP_ND ? 6 : 4;  // slot bits of the packed sort keys
  const int64_t klo = S.key_lo, khi = S.key_hi;
  x.key_base = (int)klo;
  x.sort32 = (khi - klo < (int64_t(1) << (31 - sb)) && !(c->dbg & 1)) ? 1 : 0;
  return x;
}

// reuse = true: numeric-only re-assembly into buffers holding the pattern of an earlier full call of
// the same space (NEXT-3): no row lengths, no scan; the extended-frame path
// stores values only.
lor_status vec2d_assemble(lor_ctx c, int sp, double alpha, double beta, lor_quad quad, lor_csr *out);
lor_status assemble(lor_ctx c, int s, double alpha, double beta, lor_quad quad, lor_csr *out, bool reuse = false) {
  if (!c) return LOR_ERR_INVALID_ARGUMENT;
  if (c->dim == 2 && (s == SP_ND || s == SP_RT)) {  // 2D vector spaces (lor_vec2d.cu)
    if (quad != LOR_QUAD_VERTEX && quad != LOR_QUAD_GAUSS2) return fail(c, LOR_ERR_INVALID_ARGUMENT, "bad quadrature");
    return vec2d_assemble(c, s, alpha, beta, quad, out);
  }
  if (s < 0 || s > 2 || !c->sp[s].valid) return fail(c, LOR_ERR_UNSUPPORTED, "space not available for this mesh");
  if (quad != LOR_QUAD_VERTEX && quad != LOR_QUAD_GAUSS2) return fail(c, LOR_ERR_INVALID_ARGUMENT, "bad quadrature");
  SpaceDev &S = c->sp[s];
  if (!out || !out->row_ptr || (S.nnz_local > 0 && (!out->col || !out->val)))
    return fail(c, LOR_ERR_INVALID_ARGUMENT, "null output buffer");
  if (out->cap_nnz < S.nnz_local) return fail(c, LOR_ERR_BUFFER_TOO_SMALL, "cap_nnz < nnz_local");
  CUDA_TRY(c, cudaSetDevice(c->device));
  c->nphase = 0;
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  lor_status st = LOR_OK;
  if (S.rv && !c->vc && quad == LOR_QUAD_VERTEX) {  // p = 1 per-row path of ND / RT (lor_setup)
    RvArgs a{S.n_local, S.rv_off, S.rv_ent, S.emap, S.esgn, S.rv_ea, out->row_ptr, out->col, out->val, S.cnt, c->err};
    if (!reuse) {
      CUDA_TRY(c, launch_rv_rows(s, a, false, c->stream));
      CUDA_TRY(c, launch_scan(S.cnt, out->row_ptr, S.n_local, S.scan_status, S.tile_ctr, c->stream));
      c->launches += 2;
    }
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    CUDA_TRY(c, launch_rv_ea(s, c->nel_local, c->X, c->xstride, alpha, beta, S.rv_ea, c->err, c->stream));
    CUDA_TRY(c, launch_rv_rows(s, a, true, c->stream));
    c->launches += 2;
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    return LOR_OK;
  }
  // variable coefficients on the ND frame would need 2 more E-vector boxes beside 78 KB of resident
  // cells: 1 CTA/SM, slower (7.3 vs 5.2 ms at C4) than the element + merge passes
  if (S.xvok && quad == LOR_QUAD_VERTEX && (!c->vc || ((c->nranks == 1 || c->vc_ghosts) && s == SP_RT))) {  // ND / RT extended frame
    XvArgs x = xv_args(c, s);
    if (!reuse) {
      CUDA_TRY(c, launch_xv_sym(s, c->p, x, c->stream));
      if (c->nel_local > 0) c->launches++;
      CUDA_TRY(c, launch_scan(S.cnt, out->row_ptr, S.n_local, S.scan_status, S.tile_ctr, c->stream));
      c->launches++;
    }
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    x.row_ptr = out->row_ptr;
    x.col = out->col;
    x.val = out->val;
    x.alpha = alpha;
    x.beta = beta;
    x.ca = c->vc ? c->ca : nullptr;
    x.cb = c->vc ? c->cb : nullptr;
    x.values_only = reuse ? 1 : 0;
    CUDA_TRY(c, launch_xv_fill(s, c->p, x, c->stream));
    if (c->nel_local > 0) c->launches++;
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    return LOR_OK;
  }
  if (s == SP_H1 && c->h1_rows && !c->vc && quad == LOR_QUAD_VERTEX) {  // p = 1 per-row path (lor_setup)
    LegArgs a{S.n_local, c->leg_off, c->leg_ent, c->leg_lmap, c->leg_ea, out->row_ptr, out->col, out->val, S.cnt};
    if (!reuse) {
      CUDA_TRY(c, launch_leg_rows(a, false, c->stream));
      CUDA_TRY(c, launch_scan(S.cnt, out->row_ptr, S.n_local, S.scan_status, S.tile_ctr, c->stream));
      c->launches += 2;
    }
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    CUDA_TRY(c, launch_leg_ea(c->leg_ncell, 1, c->leg_lx, alpha, beta, c->leg_ea, c->err, c->stream));
    CUDA_TRY(c, launch_leg_rows(a, true, c->stream));
    c->launches += 2;
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    return LOR_OK;
  }
  // variable coefficients: the extended frames on one rank (the neighbour coefficients come from the
  // local E-vectors), the element + merge passes otherwise
  const bool xpath = S.xok && quad == LOR_QUAD_VERTEX && (!c->vc || c->nranks == 1 || c->vc_ghosts);
  if (!reuse) {  // symbolic part (A2): row lengths per call, then the int64 scan
    if (xpath) {
      XFillArgs x = xfill_args(c, S);
      CUDA_TRY(c, launch_xh1_count(c->p, x, c->stream));
      if (c->nel_local > 0) c->launches++;
      CUDA_TRY(c, launch_scan(S.cnt, out->row_ptr, S.n_local, S.scan_status, S.tile_ctr, c->stream));
      c->launches++;
    } else {
      st = run_count_scan(c, s, out->row_ptr);
      if (st) return st;
    }
  }
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  if (xpath) {  // extended-frame path: every owned row in one pass
    XFillArgs x = xfill_args(c, S);
    x.row_ptr = out->row_ptr;
    x.col = out->col;
    x.val = out->val;
    x.alpha = alpha;
    x.beta = beta;
    x.ca = c->vc ? c->ca : nullptr;
    x.cb = c->vc ? c->cb : nullptr;
    x.values_only = reuse ? 1 : 0;
    CUDA_TRY(c, launch_xh1_fill(c->p, x, c->stream, nullptr));
    if (c->nel_local > 0) c->launches++;
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
    return LOR_OK;
  }
  AsmArgs a;
  a.order = c->order;
  a.nel_local = c->nel_local;
  a.elem_begin = c->elem_begin;
  a.topo = c->topo;
  a.esp = S.esp;
  a.X = c->X;
  a.xstride = c->xstride;
  fill_base(S, a.base);
  a.tabs = Tabs{S.tslot, S.tsize, S.tpb, S.tnpb, S.tlex};
  a.row_begin = S.row_begin;
  a.row_ptr = out->row_ptr;
  a.col = out->col;
  a.val = out->val;
  a.scratch = S.scratch;
  a.rstride = S.rstride;
  a.ose = S.ose;
  a.ose_slots = S.ose_slots;
  a.nval = S.nval;
  a.ose_elem = S.ose_elem;
  a.pbase = S.pbase;
  a.plan = S.plan;
  a.maxl = S.maxl;
  a.plan_mode = 0;
  a.alpha = alpha;
  a.beta = beta;
  a.err = c->err;
  a.tstamp = c->tstamp;
  a.ownbase = S.ownbase;
  a.ownpos = S.ownpos;
  a.dbg = c->dbg;
  a.emap = c->nranks == 1 ? S.emap : nullptr;
  a.esgn = c->nranks == 1 ? S.esgn : nullptr;
  a.ca = c->vc ? c->ca : nullptr;
  a.cb = c->vc ? c->cb : nullptr;
  CUDA_TRY(c, launch_assemble(c->dim, s, c->p, (int)quad, a, c->stream, nullptr));
  if (c->nel_local > 0) c->launches++;
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  if (S.n_mrows > 0) {  // shared rows whose contributors are all local: merge pass
    MergeArgs m{};
    m.n = S.n_mrows;
    m.W = S.W;
    m.W8 = (S.W + 15) / 16 * 16;
    m.rows = S.mrows;
    m.plan = S.plan;
    m.nval = S.nval;
    m.row_ptr = out->row_ptr;
    m.col = out->col;
    m.val = out->val;
    CUDA_TRY(c, launch_merge_rows(m, c->stream));
    c->launches++;
  }
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  if (c->nranks > 1) {
    if (c->exchange_mode == 1) {
      S.pending_exchange = 1;
      return LOR_OK;
    }
    st = exchange_nccl(c, s);
    if (st) return st;
  }
  st = finish(c, s, out);
  if (st) return st;
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  return LOR_OK;
}

// Extended frame on several ranks: the ghost layer's topology records and
// coordinates after the local ones (coordinates from the caller's global E-vector, or interpolated
// from the vertices), and the per-peer lists that refresh the ghost coordinates over NCCL when the
// coordinates change (lor_update_coordinates).  Returns false with a reason if it cannot be built.
bool xframe_ghost_layer(lor_ctx c, const HostPlan &plan, const lor_setup_args &A, const std::vector<int64_t> &xg,
                        std::string &why) {
  const int64_t ng = (int64_t)xg.size();
  c->n_xghost = ng;
  c->xghost_ids = xg;
  if (ng == 0) return true;
  const int np = (A.dim == 3) ? (A.p + 1) * (A.p + 1) * (A.p + 1) : (A.p + 1) * (A.p + 1);
  const int64_t raw = (int64_t)A.dim * np;
  // topology records: local, then ghosts
  std::vector<ElemTopo> xt((size_t)(c->nel_local + ng));
  for (int64_t i = 0; i < c->nel_local; ++i) xt[(size_t)i] = plan.topo[(size_t)i];
  for (int64_t g = 0; g < ng; ++g) xt[(size_t)(c->nel_local + g)] = plan.topo_of(xg[(size_t)g]);
  if (dev_upload(c, &c->xtopo, xt.data(), xt.size()) != cudaSuccess) { why = "ghost topology upload"; return false; }
  // coordinates: grow X by the ghost layer
  double *X2 = nullptr;
  if (cudaMalloc((void **)&X2, sizeof(double) * (size_t)((c->nel_local + ng) * c->xstride)) != cudaSuccess) {
    why = "ghost coordinates allocation";
    return false;
  }
  c->allocs.push_back(X2);
  cudaMemcpy(X2, c->X, sizeof(double) * (size_t)(c->nel_local * c->xstride), cudaMemcpyDeviceToDevice);
  std::vector<double> gh((size_t)(ng * c->xstride), 0.0), tmp;
  for (int64_t g = 0; g < ng; ++g) {
    const double *src;
    if (A.elem_nodes) src = A.elem_nodes + xg[(size_t)g] * raw;
    else {
      interpolate_evector(A.dim, A.p, A.vert_xyz, A.elem_vert, xg[(size_t)g], 1, tmp);
      src = tmp.data();
    }
    memcpy(&gh[(size_t)(g * c->xstride)], src, sizeof(double) * raw);
  }
  cudaMemcpy(X2 + c->nel_local * c->xstride, gh.data(), sizeof(double) * gh.size(), cudaMemcpyHostToDevice);
  c->X = X2;  // the old local-only array stays in allocs (freed at destroy)
  // exchange lists: ghosts held by peer q are a contiguous range of xg (ranks own contiguous
  // element ranges, xg is sorted); this rank sends q the local elements in q's ghost layer
  c->xg_send_count.assign(A.nranks, 0);
  c->xg_recv_begin.assign(A.nranks, 0);
  c->xg_recv_count.assign(A.nranks, 0);
  std::vector<int32_t> sidx;
  for (int q = 0; q < A.nranks; ++q) {
    if (q == A.rank) continue;
    for (int64_t g = 0; g < ng; ++g)
      if (xg[(size_t)g] >= plan.erb[q] && xg[(size_t)g] < plan.erb[q + 1]) {
        if (c->xg_recv_count[q] == 0) c->xg_recv_begin[q] = g;
        ++c->xg_recv_count[q];
      }
    for (int64_t e : xframe_ghosts(plan, q))
      if (e >= plan.elem_begin && e < plan.elem_begin + plan.nel_local) {
        sidx.push_back((int32_t)(e - plan.elem_begin));
        ++c->xg_send_count[q];
      }
  }
  if (!sidx.empty()) {
    if (dev_upload(c, &c->xg_send_idx, sidx.data(), sidx.size()) != cudaSuccess ||
        dev_alloc(c, &c->xg_send_buf, sidx.size() * (size_t)c->xstride) != cudaSuccess) {
      why = "ghost exchange buffers";
      return false;
    }
  }
  return true;
}

// refresh the ghost layer's coordinates from the peers (NCCL, context stream)
lor_status exchange_ghost_coords(lor_ctx c) {
  if (c->n_xghost == 0 || c->nranks == 1 || !c->comm) return LOR_OK;
  int64_t ns = 0;
  for (int64_t v : c->xg_send_count) ns += v;
  if (ns > 0) CUDA_TRY(c, launch_gather_rows(c->X, c->xstride, c->xg_send_idx, ns, c->xg_send_buf, c->stream));
  if (g_nccl.GroupStart() != ncclSuccess) return fail(c, LOR_ERR_NCCL, "ncclGroupStart");
  int64_t so = 0;
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) continue;
    if (c->xg_send_count[q] > 0) {
      if (g_nccl.Send(c->xg_send_buf + so * c->xstride, (size_t)(c->xg_send_count[q] * c->xstride * 8), ncclUint8, q,
                      c->comm, c->stream) != ncclSuccess) { g_nccl.GroupEnd(); return fail(c, LOR_ERR_NCCL, "ncclSend"); }
      so += c->xg_send_count[q];
    }
    if (c->xg_recv_count[q] > 0) {
      if (g_nccl.Recv(c->X + (c->nel_local + c->xg_recv_begin[q]) * c->xstride, (size_t)(c->xg_recv_count[q] * c->xstride * 8),
                      ncclUint8, q, c->comm, c->stream) != ncclSuccess) { g_nccl.GroupEnd(); return fail(c, LOR_ERR_NCCL, "ncclRecv"); }
    }
  }
  if (g_nccl.GroupEnd() != ncclSuccess) return fail(c, LOR_ERR_NCCL, "ncclGroupEnd");
  return LOR_OK;
}

// 2D Nedelec / Raviart-Thomas numbering (reading P-29, one rank): family d of the local
// order holds the lattice edges along d (ND) / normal to d (RT); a dof on coarse edge E has id
// E p + k with k the cell index along the edge's global orientation (min -> max vertex id) and sign
// +-1 for ND by alignment, for RT by the global normal (global tangent turned by +90 degrees)
// against the local normal +e_d; element interiors follow as ne p + el 2p(p-1) + d p(p-1) + lex.
bool vec2d_setup(lor_ctx c, const HostPlan &plan, std::string &why) {
  const int p = c->p, ndpe = 2 * p * (p + 1);
  const int64_t nel = c->nel_local, ne = plan.n_ent[1], ncell = nel * p * p;
  const SpaceDev &H = c->sp[SP_H1];
  if (!H.emap) { why = "needs the H1 element restriction"; return false; }
  for (int sp = SP_ND; sp <= SP_RT; ++sp) {
    lor_ctx_s::Vec2 &V = c->v2[sp];
    V.n = ne * p + nel * 2 * (int64_t)p * (p - 1);
    V.ncell = ncell;
    std::vector<int32_t> map((size_t)nel * ndpe);
    std::vector<int8_t> sgn((size_t)nel * ndpe);
    std::vector<uint8_t> wr((size_t)nel * ndpe);
    for (int64_t e = 0; e < nel; ++e)
      for (int l = 0; l < ndpe; ++l) {
        const int d = l / (p * (p + 1)), r = l % (p * (p + 1));
        const int ext0 = sp == SP_ND ? (d == 0 ? p : p + 1) : (d == 0 ? p + 1 : p);
        const int x[2] = {r % ext0, r / ext0};
        const int along = sp == SP_ND ? d : 1 - d, across = 1 - along;
        int64_t g;
        int sg = 1, w = 1;
        if (x[across] == 0 || x[across] == p) {
          const int le = 2 * along + (x[across] == p);
          const int64_t E = plan.el_edge[e * 4 + le];
          const bool aligned = !plan.el_edge_rev[e * 4 + le];
          g = E * p + (aligned ? x[along] : p - 1 - x[along]);
          sg = (aligned ? 1 : -1) * ((sp == SP_RT && d == 0) ? -1 : 1);
          w = plan.inc_el[1][plan.inc_off[1][E]] == plan.elem_begin + e;
        } else {
          const int lex = sp == SP_ND ? (d == 0 ? x[0] + p * (x[1] - 1) : (x[0] - 1) + (p - 1) * x[1])
                                      : (d == 0 ? (x[0] - 1) + (p - 1) * x[1] : x[0] + p * (x[1] - 1));
          g = ne * p + e * 2 * (int64_t)p * (p - 1) + d * (int64_t)p * (p - 1) + lex;
        }
        map[e * ndpe + l] = (int32_t)g;
        sgn[e * ndpe + l] = (int8_t)sg;
        wr[e * ndpe + l] = (uint8_t)w;
      }
    V.bnd.clear();
    for (int64_t E = 0; E < ne; ++E)
      if (plan.inc_off[1][E + 1] - plan.inc_off[1][E] == 1)
        for (int k = 0; k < p; ++k) V.bnd.push_back((int32_t)(E * p + k));
    if (dev_upload(c, &V.map, map.data(), map.size()) || dev_upload(c, &V.sgn, sgn.data(), sgn.size()) ||
        dev_upload(c, &V.writer, wr.data(), wr.size()) || dev_alloc(c, &V.cmap, ncell * 4) ||
        dev_alloc(c, &V.csgn, ncell * 4) || dev_alloc(c, &V.ent, ncell * 4) || dev_alloc(c, &V.off, V.n + 1) ||
        dev_alloc(c, &V.rp, V.n + 1) || dev_alloc(c, &V.cnt, V.n + 1) || dev_alloc(c, &V.ea, ncell * 16)) {
      why = "out of memory";
      return false;
    }
    const int64_t roff[2] = {0, V.n};
    if (dev_upload(c, &V.droff, roff, 2)) {
      why = "out of memory";
      return false;
    }
    if (launch_v2_cells(sp, p, nel, V.map, V.sgn, V.cmap, V.csgn, c->stream) != cudaSuccess ||
        launch_transpose(V.cmap, ncell * 4, 0, V.n, V.cnt, V.off, V.ent, H.scan_status, H.tile_ctr, c->stream) !=
            cudaSuccess) {
      why = "cells / transpose";
      return false;
    }
    // the pattern is topological: its size once, from the count pass
    V2Rows r{V.n, V.off, V.ent, V.cmap, V.ea, V.rp, nullptr, nullptr, V.cnt};
    if (launch_v2_rows(r, false, c->stream) != cudaSuccess ||
        launch_scan(V.cnt, V.rp, V.n, H.scan_status, H.tile_ctr, c->stream) != cudaSuccess ||
        cudaMemcpyAsync(&V.nnz, V.rp + V.n, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess) {
      why = "pattern size";
      return false;
    }
    V.ok = true;
  }
  return true;
}

lor_status vec2d_assemble(lor_ctx c, int sp, double alpha, double beta, lor_quad quad, lor_csr *out) {
  lor_ctx_s::Vec2 &V = c->v2[sp];
  if (!V.ok) return fail(c, LOR_ERR_UNSUPPORTED, "2D ND / RT: one rank only");
  if (!out || !out->row_ptr || (V.nnz > 0 && (!out->col || !out->val))) return fail(c, LOR_ERR_INVALID_ARGUMENT, "null output buffer");
  if (out->cap_nnz < V.nnz) return fail(c, LOR_ERR_BUFFER_TOO_SMALL, "cap_nnz < nnz_local");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const SpaceDev &H = c->sp[SP_H1];
  c->nphase = 0;
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  V2Args a{c->p, V.ncell, c->X, c->xstride, c->vc ? c->ca : nullptr, c->vc ? c->cb : nullptr, alpha, beta, V.csgn,
           V.ea, c->err};
  CUDA_TRY(c, launch_v2_ea(sp, (int)quad, a, c->stream));
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  V2Rows r{V.n, V.off, V.ent, V.cmap, V.ea, out->row_ptr, out->col, out->val, V.cnt};
  CUDA_TRY(c, launch_v2_rows(r, false, c->stream));
  CUDA_TRY(c, launch_scan(V.cnt, out->row_ptr, V.n, H.scan_status, H.tile_ctr, c->stream));
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  CUDA_TRY(c, launch_v2_rows(r, true, c->stream));
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  c->launches += 4;
  return LOR_OK;
}

lor_status vec2d_discrete(lor_ctx c, int sp, lor_csr *out) {
  lor_ctx_s::Vec2 &V = c->v2[sp];
  if (!V.ok) return fail(c, LOR_ERR_UNSUPPORTED, "2D discrete operators: one rank only");
  if (!out || !out->row_ptr || !out->col || !out->val) return fail(c, LOR_ERR_INVALID_ARGUMENT, "null output buffer");
  if (out->cap_nnz < 2 * V.n) return fail(c, LOR_ERR_BUFFER_TOO_SMALL, "cap_nnz < 2 n_rows");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, launch_rowptr_stride(out->row_ptr, V.n, 2, c->stream));
  V2Disc d{sp, c->p, c->nel_local, 0, V.map, V.sgn, V.writer, c->sp[SP_H1].emap, out->col, out->val};
  CUDA_TRY(c, launch_v2_disc(d, c->stream));
  c->launches += 2;
  return LOR_OK;
}

// Orders at which the one-pass extended frame of a vector space beats the element + merge passes on
// one GPU (full calls, Cartesian N^3-cell meshes, N = 96 / 105, 1xB200, profiles/vector_sweep_r02_v4.jsonl):
// ND at p = 4-5 only (1.2-1.3x faster there; 1.3-2.7x slower at p = 1-3, 6, 7), RT at every order
// but 5 (1.2-1.6x faster; 1.4x slower at p = 5, a tie at 6).
bool xv_preferred(int sv, int p) {
  if (sv == SP_ND) return p == 4 || p == 5;
  return p != 5;
}

}  // namespace

extern "C" {

lor_status lor_nccl_get_unique_id(void *out128) {
  if (!out128) return LOR_ERR_INVALID_ARGUMENT;
  std::string err;
  if (!g_nccl.load(err)) return LOR_ERR_NCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return LOR_ERR_NCCL;
  memcpy(out128, &id, sizeof(id));
  return LOR_OK;
}

lor_status lor_plan_dry_run(const lor_setup_args *args, int64_t *info, int64_t *send_counts, int64_t *recv_counts) {
  if (!args || !info) return LOR_ERR_INVALID_ARGUMENT;
  const lor_setup_args &A = *args;
  if (!(A.dim == 2 || A.dim == 3) || A.p < 1 || A.p > 8 || A.n_vert <= 0 || A.n_elem <= 0 || !A.elem_vert ||
      A.nranks < 1 || A.rank < 0 || A.rank >= A.nranks || (A.nranks > 1 && !A.elem_rank_begin))
    return LOR_ERR_INVALID_ARGUMENT;
  HostPlan plan;
  try {
    PlanInput in;
    in.dim = A.dim;
    in.p = A.p;
    in.rank = A.rank;
    in.nranks = A.nranks;
    in.n_vert = A.n_vert;
    in.n_elem = A.n_elem;
    in.elem_vert = A.elem_vert;
    in.elem_rank_begin = A.elem_rank_begin;
    plan.build(in);
  } catch (const std::exception &ex) {
    g_setup_error = std::string("lor_plan_dry_run: ") + ex.what();
    return LOR_ERR_INVALID_ARGUMENT;
  }
  for (int s = 0; s < 3; ++s) {
    const SpacePlan &P = plan.sp[s];
    int64_t *o = info + 8 * s;
    o[0] = P.valid;
    o[1] = P.n_global;
    o[2] = P.row_begin;
    o[3] = P.n_local;
    o[4] = P.n_records;
    o[5] = (int64_t)P.ose.size();
    o[6] = (int64_t)P.defer.size();
    o[7] = (int64_t)plan.ghost.size();
    for (int q = 0; q < A.nranks; ++q) {
      if (send_counts) send_counts[s * A.nranks + q] = P.valid ? P.send_count[q] : 0;
      if (recv_counts) recv_counts[s * A.nranks + q] = P.valid ? P.recv_count[q] : 0;
    }
  }
  return LOR_OK;
}

lor_status lor_xframe_dry_run(const lor_setup_args *args, int64_t *info, int64_t *send_counts, int64_t *recv_counts) {
  if (!args || !info) return LOR_ERR_INVALID_ARGUMENT;
  const lor_setup_args &A = *args;
  if (A.dim != 3 || A.p < 1 || A.p > 8 || A.n_vert <= 0 || A.n_elem <= 0 || !A.elem_vert || A.nranks < 1 || A.rank < 0 ||
      A.rank >= A.nranks || (A.nranks > 1 && !A.elem_rank_begin))
    return LOR_ERR_INVALID_ARGUMENT;
  HostPlan plan;
  try {
    PlanInput in;
    in.dim = A.dim;
    in.p = A.p;
    in.rank = A.rank;
    in.nranks = A.nranks;
    in.n_vert = A.n_vert;
    in.n_elem = A.n_elem;
    in.elem_vert = A.elem_vert;
    in.elem_rank_begin = A.elem_rank_begin;
    plan.build(in);
  } catch (const std::exception &ex) {
    g_setup_error = std::string("lor_xframe_dry_run: ") + ex.what();
    return LOR_ERR_INVALID_ARGUMENT;
  }
  std::vector<XElem> xe;
  std::vector<int64_t> xg;
  int cmax[3];
  std::string why;
  const bool ok = xframe_build(plan, A.elem_vert, xe, cmax, &why, A.nranks > 1 ? &xg : nullptr);
  info[0] = ok ? 1 : 0;
  info[1] = (int64_t)xg.size();
  info[2] = ok ? std::max(cmax[0], std::max(cmax[1], cmax[2])) : 0;
  info[3] = plan.nel_local;
  for (int q = 0; q < A.nranks; ++q) {
    int64_t sc = 0, rc = 0;
    if (q != A.rank) {
      for (int64_t e : xframe_ghosts(plan, q)) sc += (e >= plan.elem_begin && e < plan.elem_begin + plan.nel_local);
      for (int64_t e : xg) rc += (e >= plan.erb[q] && e < plan.erb[q + 1]);
    }
    if (send_counts) send_counts[q] = sc;
    if (recv_counts) recv_counts[q] = rc;
  }
  if (!ok) g_setup_error = why;
  return LOR_OK;
}

lor_status lor_setup(const lor_setup_args *args, lor_ctx *out) {
  g_setup_error.clear();
  if (!out || !args) {
    g_setup_error = "lor_setup: null args/out";
    return LOR_ERR_INVALID_ARGUMENT;
  }
  *out = nullptr;
  const lor_setup_args &A = *args;
  if (!(A.dim == 2 || A.dim == 3) || A.p < 1 || A.p > 8 || A.n_vert <= 0 || A.n_elem <= 0 || !A.elem_vert ||
      A.nranks < 1 || A.rank < 0 || A.rank >= A.nranks || (!A.elem_nodes && !A.vert_xyz) ||
      (A.nranks > 1 && !A.elem_rank_begin)) {
    g_setup_error = "lor_setup: invalid argument (dim in {2,3}, 1 <= p <= 8, counts > 0, non-null arrays, "
                    "0 <= rank < nranks, elem_rank_begin when nranks > 1)";
    return LOR_ERR_INVALID_ARGUMENT;
  }
  lor_ctx c = new lor_ctx_s();
  c->dim = A.dim;
  c->p = A.p;
  c->rank = A.rank;
  c->nranks = A.nranks;
  c->device = A.device;
  c->stream = reinterpret_cast<cudaStream_t>(A.cuda_stream);
  c->nel = A.n_elem;
  c->dbg = getenv("LOR_DBG") ? atoi(getenv("LOR_DBG")) : 0;
  auto bail = [&](lor_status st, const std::string &msg) {
    cudaError_t ce = cudaGetLastError();
    g_setup_error = "lor_setup: " + msg;
    if (ce != cudaSuccess) g_setup_error += std::string(" (") + cudaGetErrorString(ce) + ")";
    lor_destroy(c);
    return st;
  };
  if (cudaSetDevice(A.device) != cudaSuccess) return bail(LOR_ERR_CUDA, "cudaSetDevice");
  HostPlan plan;
  try {
    PlanInput in;
    in.dim = A.dim;
    in.p = A.p;
    in.rank = A.rank;
    in.nranks = A.nranks;
    in.n_vert = A.n_vert;
    in.n_elem = A.n_elem;
    in.elem_vert = A.elem_vert;
    in.elem_rank_begin = A.elem_rank_begin;
    plan.build(in);
  } catch (const std::exception &ex) {
    return bail(LOR_ERR_INVALID_ARGUMENT, ex.what());
  } catch (...) {
    return bail(LOR_ERR_OUT_OF_MEMORY, "host plan: allocation failure");
  }
  c->elem_begin = plan.elem_begin;
  c->nel_local = plan.nel_local;
  c->ntopo = (int64_t)plan.topo.size();
  // coordinates: local elements, element stride padded to 16 doubles (128 B)
  const int np = (A.dim == 3) ? (A.p + 1) * (A.p + 1) * (A.p + 1) : (A.p + 1) * (A.p + 1);
  const int64_t raw = (int64_t)A.dim * np;
  c->xstride = (raw + 15) / 16 * 16;
  {
    std::vector<double> tmp;
    const double *src = nullptr;
    if (A.elem_nodes) src = A.elem_nodes + plan.elem_begin * raw;
    else {
      interpolate_evector(A.dim, A.p, A.vert_xyz, A.elem_vert, plan.elem_begin, plan.nel_local, tmp);
      src = tmp.data();
    }
    std::vector<double> padded((size_t)(plan.nel_local * c->xstride), 0.0);
    for (int64_t e = 0; e < plan.nel_local; ++e) memcpy(&padded[e * c->xstride], src + e * raw, sizeof(double) * raw);
    // locality-preserving processing order: Morton code of element centroids (neighbours of an
    // element are processed close in time, so partial rows are merged while still in L2)
    const char *ord_env = getenv("LOR_ORDER");  // dev experiments: "natural", "sweep" (default Morton)
    const bool sweep = ord_env && !strcmp(ord_env, "sweep");
    if (!(ord_env && !strcmp(ord_env, "natural"))) {
      const int64_t n = plan.nel_local;
      std::vector<double> cen((size_t)n * 3, 0.0);
      double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
      for (int64_t e = 0; e < n; ++e)
        for (int d = 0; d < A.dim; ++d) {
          double sum = 0.0;
          for (int l = 0; l < np; ++l) sum += src[e * raw + (int64_t)d * np + l];
          const double v = sum / np;
          cen[e * 3 + d] = v;
          lo[d] = std::min(lo[d], v);
          hi[d] = std::max(hi[d], v);
        }
      std::vector<std::pair<uint64_t, int32_t>> key((size_t)n);
      for (int64_t e = 0; e < n; ++e) {
        uint64_t code = 0;
        uint32_t qd[3] = {0, 0, 0};
        for (int d = 0; d < A.dim; ++d) {
          const double t = hi[d] > lo[d] ? (cen[e * 3 + d] - lo[d]) / (hi[d] - lo[d]) : 0.0;
          qd[d] = (uint32_t)std::min(1023.0, std::max(0.0, t * 1023.0 + 0.5));
        }
        if (sweep) {  // plane sweep: z, then y, then x
          for (int d = A.dim - 1; d >= 0; --d) code = (code << 10) | qd[d];
        } else {
          for (int bit = 9; bit >= 0; --bit)
            for (int d = A.dim - 1; d >= 0; --d) code = (code << 1) | ((qd[d] >> bit) & 1u);
        }
        key[e] = {code, (int32_t)e};
      }
      std::stable_sort(key.begin(), key.end(),
                       [](const std::pair<uint64_t, int32_t> &a, const std::pair<uint64_t, int32_t> &b) { return a.first < b.first; });
      std::vector<int32_t> ord((size_t)n);
      for (int64_t e = 0; e < n; ++e) ord[e] = key[e].second;
      if (dev_upload(c, &c->order, ord.data(), ord.size()) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "order");
      c->order_host = ord;
    }
    if (dev_upload(c, &c->X, padded.data(), padded.size()) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "X");
  }
  if (dev_upload(c, &c->topo, plan.topo.data(), plan.topo.size()) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "topo");
  if (dev_alloc(c, &c->err, 4) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "err");
  if (getenv("LOR_PHASE_TIMING") && c->nel_local > 0 &&
      dev_alloc(c, &c->tstamp, (size_t)c->nel_local * 16) != cudaSuccess)
    return bail(LOR_ERR_OUT_OF_MEMORY, "tstamp");
  for (int i = 0; i < 8; ++i) cudaEventCreate(&c->ev[i]);
  int max_smem = 0;
  for (int s = 0; s < 3; ++s) {
    const SpacePlan &P = plan.sp[s];
    SpaceDev &S = c->sp[s];
    S.valid = P.valid && (s == SP_H1 || A.space_mask == 0 || ((A.space_mask >> s) & 1));
    if (!S.valid) continue;
    S.ndpe = P.ndpe;
    S.maxl = P.maxl;
    S.rstride = ((P.maxl + 1) * 16 + 127) / 128 * 8;  // entries + header, padded to whole 128-byte lines
    S.W = (A.dim == 2) ? 9 : (s == SP_H1 ? 27 : (s == SP_ND ? 33 : 11));
    {
      const int64_t ns = tab_slot_entries(A.dim, s), nz = tab_size_entries(A.dim, s);
      const int64_t nk = (A.dim == 2 || s == SP_H1) ? 729 : 3 * 729;
      if (dev_alloc(c, &S.tslot, ns) != cudaSuccess || dev_alloc(c, &S.tsize, nz) != cudaSuccess ||
          dev_alloc(c, &S.tpb, nz) != cudaSuccess || dev_alloc(c, &S.tnpb, nk) != cudaSuccess ||
          dev_alloc(c, &S.tlex, ns * 8) != cudaSuccess)
        return bail(LOR_ERR_OUT_OF_MEMORY, "tables");
      if (launch_build_tables(A.dim, s, A.p, S.tslot, S.tsize, S.tpb, S.tnpb, S.tlex, c->stream) != cudaSuccess)
        return bail(LOR_ERR_CUDA, "tables");
    }
    S.n_global = P.n_global;
    S.row_begin = P.row_begin;
    S.n_local = P.n_local;
    S.n_tr = 0;
    for (int64_t e = 0; e < plan.nel_local; ++e)
      for (int tau = 0; tau < (A.dim == 3 ? 27 : 9); ++tau)
        if (plan.topo[e].flags[tau] & TF_OWNED) S.n_tr += class_rows(A.dim, s, A.p, tau);
    for (int t = 0; t < 4; ++t)
      if (dev_upload(c, &S.base[t], P.base[t].data(), P.base[t].size()) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "base");
    if (dev_upload(c, &S.esp, P.esp.data(), P.esp.size()) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "esp");
    if (dev_upload(c, &S.ose, P.ose.data(), P.ose.size()) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "ose");
    if (dev_upload(c, &S.ose_slots, P.ose_slots.data(), P.ose_slots.size()) != cudaSuccess)
      return bail(LOR_ERR_OUT_OF_MEMORY, "ose_slots");
    if (dev_upload(c, &S.defer, P.defer.data(), P.defer.size()) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "defer");
    S.n_ose = (int)P.ose.size();
    S.n_defer = (int)P.defer.size();
    S.n_records = P.n_records;
    if (P.n_records > 0) {
      cudaError_t e = cudaMalloc((void **)&S.scratch, (size_t)P.n_records * S.rstride * sizeof(RecEntry));
      if (e != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "scratch");
      c->allocs.push_back(S.scratch);
    }
    if (dev_alloc(c, &S.cnt, (size_t)std::max<int64_t>(P.n_local, 1)) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "cnt");
    if (dev_alloc(c, &S.scan_status, (size_t)scan_status_words(P.n_local)) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "scan");
    if (dev_alloc(c, &S.tile_ctr, 1) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "tile");
    S.recv_begin = P.recv_begin;
    S.recv_count = P.recv_count;
    S.send_begin = P.send_begin;
    S.send_count = P.send_count;
    S.rank_off = P.rank_off;
    if (dev_upload(c, &S.droff, P.rank_off.data(), P.rank_off.size()) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "rank_off");
    plan.boundary_rows(s, S.bnd);
    int smem = 0;
    AsmArgs dummy{};
    launch_assemble(A.dim, s, A.p, 0, dummy, c->stream, &smem);
    max_smem = std::max(max_smem, smem);
  }
  c->fin_smem = 48 * 1024;
  // NCCL communicator
  if (A.nranks > 1 && A.nccl_unique_id) {
    std::string err;
    if (!g_nccl.load(err)) return bail(LOR_ERR_NCCL, err);
    ncclUniqueId id;
    memcpy(&id, A.nccl_unique_id, sizeof(id));
    if (g_nccl.CommInitRank(&c->comm, A.nranks, id, A.rank) != ncclSuccess) return bail(LOR_ERR_NCCL, "ncclCommInitRank");
  } else if (A.nranks > 1) {
    c->exchange_mode = 1;  // no communicator: single-process emulation (lor_exchange_copy)
  }
  // the pattern is topological: count + scan once so lor_query can report nnz
  for (int s = 0; s < 3; ++s) {
    SpaceDev &S = c->sp[s];
    if (!S.valid) continue;
    int64_t *rp = nullptr;
    if (cudaMalloc((void **)&rp, sizeof(int64_t) * (S.n_local + 1)) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "rp");
    if (run_count_scan(c, s, rp) != LOR_OK) { cudaFree(rp); return bail(LOR_ERR_CUDA, c->last_error); }
    int64_t nnz = 0;
    cudaStreamSynchronize(c->stream);
    if (cudaMemcpy(&nnz, rp + S.n_local, sizeof(int64_t), cudaMemcpyDeviceToHost) != cudaSuccess) {
      cudaFree(rp);
      return bail(LOR_ERR_CUDA, "nnz readback");
    }
    cudaFree(rp);
    S.nnz_local = nnz;
  }
  // setup merge plan of shared rows (topological): plan-mode assembly writes every shared row's
  // partial-row records, then one merge per owned shared entity records where each block lands
  for (int s = 0; s < 3; ++s) {
    SpaceDev &S = c->sp[s];
    if (!S.valid || S.n_ose == 0) continue;
    const SpacePlan &P = plan.sp[s];
    std::vector<int64_t> pb(P.ose.size());
    std::vector<uint8_t> isdef(P.ose.size(), 0);
    std::vector<int32_t> oel(P.ose_elem.size());
    int64_t nbytes = 0;
    for (size_t i = 0; i < P.ose.size(); ++i) {
      pb[i] = nbytes;
      const int k = P.ose[i].k;
      nbytes += (int64_t)P.ose[i].nrows * plan_row_bytes(k, S.W);
    }
    for (int32_t d : P.defer) isdef[d] = 1;
    for (size_t i = 0; i < oel.size(); ++i) oel[i] = (int32_t)(P.ose_elem[i] - plan.elem_begin);
    std::vector<MergeRow> mr;
    for (size_t i = 0; i < P.ose.size(); ++i) {
      if (isdef[i]) continue;
      const int k = P.ose[i].k;
      for (int r = 0; r < P.ose[i].nrows; ++r)
        mr.push_back(MergeRow{pb[i] + (int64_t)r * plan_row_bytes(k, S.W), (int32_t)(P.ose[i].gid_base + r - S.row_begin), k});
    }
    S.n_mrows = (int64_t)mr.size();
    if (dev_upload(c, &S.mrows, mr.data(), mr.size()) != cudaSuccess) return bail(LOR_ERR_OUT_OF_MEMORY, "mrows");
    const int ndpe_asm = S.ndpe;
    if (dev_upload(c, &S.pbase, pb.data(), pb.size()) != cudaSuccess ||
        dev_upload(c, &S.is_defer, isdef.data(), isdef.size()) != cudaSuccess ||
        dev_upload(c, &S.ose_elem, oel.data(), oel.size()) != cudaSuccess ||
        dev_alloc(c, &S.plan, (size_t)std::max<int64_t>(nbytes, 16)) != cudaSuccess ||
        dev_alloc(c, &S.nval, (size_t)c->nel_local * ndpe_asm * ((S.W + 15) / 16 * 16)) != cudaSuccess)
      return bail(LOR_ERR_OUT_OF_MEMORY, "plan");
    AsmArgs a{};
    a.order = c->order;
    a.nel_local = c->nel_local;
    a.elem_begin = c->elem_begin;
    a.topo = c->topo;
    a.esp = S.esp;
    a.X = c->X;
    a.xstride = c->xstride;
    fill_base(S, a.base);
    a.tabs = Tabs{S.tslot, S.tsize, S.tpb, S.tnpb, S.tlex};
    a.row_begin = S.row_begin;
    a.scratch = S.scratch;
    a.rstride = S.rstride;
    a.ose = S.ose;
    a.ose_slots = S.ose_slots;
      a.maxl = S.maxl;
    a.plan_mode = 1;
    a.alpha = 1.0;
    a.beta = 1.0;
    a.err = c->err;
    if (launch_assemble(A.dim, s, A.p, 0, a, c->stream, nullptr) != cudaSuccess) return bail(LOR_ERR_CUDA, "plan asm");
    PlanArgs pa;
    pa.n = S.n_ose;
    pa.ose = S.ose;
    pa.ose_slots = S.ose_slots;
    pa.is_defer = S.is_defer;
    pa.scratch = S.scratch;
    pa.rstride = S.rstride;
    pa.W = S.W;
    pa.pbase = S.pbase;
    pa.plan = S.plan;
    pa.ose_elem = S.ose_elem;
    pa.ndpe = S.ndpe;
    if (launch_plan_merge(pa, S.n_ose, c->stream) != cudaSuccess) return bail(LOR_ERR_CUDA, "plan merge");
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return bail(LOR_ERR_CUDA, "plan sync");
    int herr[4] = {0, 0, 0, 0};
    cudaMemcpy(herr, c->err, sizeof(herr), cudaMemcpyDeviceToHost);
    if (herr[0]) { cudaMemset(c->err, 0, sizeof(herr)); }  // geometry errors are reported by assembly calls
  }
  // own-row position tables (topological): rows of entities owned by one element alone get the
  // final CSR position of every stencil slot once here, by a position pass of the element kernel
  for (int s = 0; s < 3; ++s) {
    SpaceDev &S = c->sp[s];
    const SpacePlan &P = plan.sp[s];
    if (!S.valid || c->nel_local == 0) continue;
    std::vector<int64_t> ob((size_t)c->nel_local);
    int64_t tot = 0;
    for (int64_t e = 0; e < c->nel_local; ++e) {
      ob[e] = tot;
      for (int tau = 0; tau < 27; ++tau)
        if ((plan.topo[e].flags[tau] & TF_OWNED) && !(P.esp[e].sflags[tau] & SF_SHARED))
          tot += class_rows(A.dim, s, A.p, tau);
    }
    S.n_own = tot;
    if (dev_upload(c, &S.ownbase, ob.data(), ob.size()) != cudaSuccess ||
        dev_alloc(c, &S.ownpos, (size_t)std::max<int64_t>(tot, 1) * own_w(S.W)) != cudaSuccess)
      return bail(LOR_ERR_OUT_OF_MEMORY, "own-row positions");
    AsmArgs a{};
    a.order = c->order;
    a.nel_local = c->nel_local;
    a.elem_begin = c->elem_begin;
    a.topo = c->topo;
    a.esp = S.esp;
    a.X = c->X;
    a.xstride = c->xstride;
    for (int t = 0; t < 4; ++t) a.base[t] = S.base[t];
    a.tabs = Tabs{S.tslot, S.tsize, S.tpb, S.tnpb, S.tlex};
    a.row_begin = S.row_begin;
    a.alpha = 1.0;
    a.beta = 1.0;
    a.err = c->err;
    a.plan_mode = 2;
    a.ownbase = S.ownbase;
    a.ownpos = S.ownpos;
    if (launch_assemble(A.dim, s, A.p, 0, a, c->stream, nullptr) != cudaSuccess) return bail(LOR_ERR_CUDA, "own-row positions");
  }
  // the element restriction of every space, computed once (k_dofmap): read by the discrete
  // operators, and on one rank by the element pass instead of rebuilding its block table per call
  // (LOR_EMAP=0: off)
  if (c->nel_local > 0 && !(getenv("LOR_EMAP") && !atoi(getenv("LOR_EMAP")))) {
    for (int s = 0; s < 3; ++s) {
      SpaceDev &S = c->sp[s];
      if (!S.valid) continue;
      const size_t n = (size_t)c->nel_local * S.ndpe;
      if (dev_alloc(c, &S.emap, n) != cudaSuccess || dev_alloc(c, &S.esgn, n) != cudaSuccess)
        return bail(LOR_ERR_OUT_OF_MEMORY, "element restriction");
      DofmapArgs d;
      d.p = A.p;
      d.ndpe = S.ndpe;
      d.nel_local = c->nel_local;
      d.topo = c->topo;
      fill_base(S, d.base);
      d.map = S.emap;
      d.sign = S.esgn;
      if (launch_dofmap(A.dim, s, d, c->stream) != cudaSuccess) return bail(LOR_ERR_CUDA, "element restriction");
    }
  }
  // extended-frame H1 path: regular-neighbourhood check, element records, box and position tables
  if (A.dim == 3 && c->sp[SP_H1].valid && c->nel_local > 0 && !(getenv("LOR_XFRAME") && !atoi(getenv("LOR_XFRAME")))) {
    SpaceDev &S = c->sp[SP_H1];
    std::vector<XElem> xe;
    std::vector<int64_t> xg;
    std::string why;
    if ((c->nel_local + (A.nranks > 1 ? (int64_t)xframe_ghosts(plan, A.rank).size() : 0)) * c->xstride >= (int64_t(1) << 31)) {
      why = "E-vector index exceeds int32";
    } else if (xframe_build(plan, A.elem_vert, xe, S.xc, &why, A.nranks > 1 ? &xg : nullptr) &&
               !(A.nranks > 1 && !xframe_ghost_layer(c, plan, A, xg, why))) {
      // records in processing order, so a CTA reads its record, restriction and gather list by
      // its own index (one dependent load less)
      {
        std::vector<XElem> xo(xe.size());
        for (size_t b = 0; b < xe.size(); ++b) {
          const int32_t e = c->order_host.empty() ? (int32_t)b : c->order_host[b];
          xo[b] = xe[(size_t)e];
          xo[b].el = e;
        }
        xe.swap(xo);
      }
      if (dev_upload(c, &S.xe, xe.data(), xe.size()) != cudaSuccess ||
          dev_alloc(c, &S.xbox, (size_t)c->nel_local * 125) != cudaSuccess ||
          dev_alloc(c, &S.xmap, (size_t)c->nel_local * xmap_points(A.p, S.xc)) != cudaSuccess ||
          dev_alloc(c, &S.xhalo, (size_t)c->nel_local * (xmap_points(A.p, S.xc) - (int64_t)(A.p + 1) * (A.p + 1) * (A.p + 1))) != cudaSuccess ||
          dev_alloc(c, &S.xpos, (size_t)std::max<int64_t>(S.n_local, 1) * 8) != cudaSuccess)
        return bail(LOR_ERR_OUT_OF_MEMORY, "xframe");
      XSetupArgs xa{};
      xa.nel_local = c->nel_local;
      xa.xe = S.xe;
      xa.topo = c->xtopo ? c->xtopo : c->topo;
      fill_base(S, xa.base);
      xa.row_begin = S.row_begin;
      xa.box = S.xbox;
      xa.nb = xfill_nb(A.p, S.xc);
      xa.xmap = S.xmap;
      xa.xhalo = S.xhalo;
      xa.xstride = c->xstride;
      xa.err = c->err;
      if (cudaMemset(c->err, 0, 4 * sizeof(int)) != cudaSuccess) return bail(LOR_ERR_CUDA, "xframe");
      if (launch_xh1_setup(A.p, xa, c->stream) != cudaSuccess) return bail(LOR_ERR_CUDA, "xframe setup");
      if (cudaStreamSynchronize(c->stream) != cudaSuccess) return bail(LOR_ERR_CUDA, "xframe sync");
      int herr[4] = {0, 0, 0, 0};
      cudaMemcpy(herr, c->err, sizeof(herr), cudaMemcpyDeviceToHost);
      cudaMemset(c->err, 0, sizeof(herr));
      S.xok = herr[0] == 0;
      if (S.xok) {
        // the per-call row lengths of the extended-frame path must equal those of the general
        // minimal-element count (S.cnt still holds them from the nnz pass above)
        int32_t *xc = nullptr;
        std::vector<int32_t> h0((size_t)S.n_local), h1((size_t)S.n_local);
        if (cudaMalloc((void **)&xc, sizeof(int32_t) * std::max<int64_t>(S.n_local, 1)) != cudaSuccess)
          return bail(LOR_ERR_OUT_OF_MEMORY, "xframe check");
        XFillArgs x = xfill_args(c, S);
        x.cnt = xc;
        cudaMemset(xc, 0, sizeof(int32_t) * std::max<int64_t>(S.n_local, 1));
        const bool ok = launch_xh1_count(A.p, x, c->stream) == cudaSuccess && cudaStreamSynchronize(c->stream) == cudaSuccess &&
                        cudaMemcpy(h0.data(), S.cnt, sizeof(int32_t) * S.n_local, cudaMemcpyDeviceToHost) == cudaSuccess &&
                        cudaMemcpy(h1.data(), xc, sizeof(int32_t) * S.n_local, cudaMemcpyDeviceToHost) == cudaSuccess;
        cudaFree(xc);
        if (!ok) return bail(LOR_ERR_CUDA, "xframe check");
        S.xok = h0 == h1;
      }
      if (!S.xok) fprintf(stderr, "lor_setup: extended-frame tables inconsistent, using the element + merge passes\n");
      // ND / RT on the same frame: restriction of the box dofs, checked like H1 (row lengths of the
      // per-call symbolic pass == those of the general minimal-element count)
      for (int sv = SP_ND; S.xok && sv <= SP_RT; ++sv) {
        SpaceDev &V = c->sp[sv];
        // LOR_XV=0 turns the vector-space path off, LOR_XV_ND=0 for ND only (A/B against the
        // element + merge passes)
        const char *xv_env = getenv("LOR_XV"), *xvnd_env = getenv("LOR_XV_ND");
        if (!V.valid || (xv_env && !atoi(xv_env)) || (sv == SP_ND && xvnd_env && !atoi(xvnd_env)) ||
            !xv_supported(sv, A.p, S.xc))
          continue;
        // one rank: the frame only at the orders where it measured faster than the element + merge
        // passes (xv_preferred); several ranks: wherever it fits (it needs no partial-row exchange).
        // LOR_XV=1 forces it at every supported order (tests).
        if (A.nranks == 1 && !(xv_env && atoi(xv_env) == 1) && !xv_preferred(sv, A.p)) continue;
        if (dev_alloc(c, &V.xvmap, (size_t)c->nel_local * xv_map_words(sv, A.p, S.xc)) != cudaSuccess ||
            dev_alloc(c, &V.xvpos, (size_t)std::max<int64_t>(V.n_local, 1) * xv_pos_words(sv)) != cudaSuccess)
          return bail(LOR_ERR_OUT_OF_MEMORY, "xframe (vector spaces)");
        XvArgs x = xv_args(c, sv);
        int32_t *vc = nullptr;
        if (cudaMalloc((void **)&vc, sizeof(int32_t) * std::max<int64_t>(V.n_local, 1)) != cudaSuccess)
          return bail(LOR_ERR_OUT_OF_MEMORY, "xframe check");
        cudaMemset(vc, 0, sizeof(int32_t) * std::max<int64_t>(V.n_local, 1));
        x.cnt = vc;
        std::vector<int32_t> h0((size_t)V.n_local), h1((size_t)V.n_local);
        int herr2[4] = {0, 0, 0, 0};
        bool ok = cudaMemset(c->err, 0, 4 * sizeof(int)) == cudaSuccess && launch_xv_setup(sv, A.p, x, c->stream) == cudaSuccess &&
                  launch_xv_sym(sv, A.p, x, c->stream) == cudaSuccess && cudaStreamSynchronize(c->stream) == cudaSuccess &&
                  cudaMemcpy(herr2, c->err, sizeof(herr2), cudaMemcpyDeviceToHost) == cudaSuccess &&
                  cudaMemcpy(h0.data(), V.cnt, sizeof(int32_t) * V.n_local, cudaMemcpyDeviceToHost) == cudaSuccess &&
                  cudaMemcpy(h1.data(), vc, sizeof(int32_t) * V.n_local, cudaMemcpyDeviceToHost) == cudaSuccess;
        cudaFree(vc);
        cudaMemset(c->err, 0, 4 * sizeof(int));
        if (!ok) return bail(LOR_ERR_CUDA, "xframe setup (vector spaces)");
        V.xvok = herr2[0] == 0 && h0 == h1;
        if (!V.xvok) fprintf(stderr, "lor_setup: extended-frame tables of space %d inconsistent, using the element + merge passes\n", sv);
      }
    } else if (getenv("LOR_XFRAME_VERBOSE")) {
      fprintf(stderr, "lor_setup: extended-frame path off: %s\n", why.c_str());
    }
  }
  // column-id range each extended-frame space references (its restriction): the symbolic pass sorts
  // keys relative to key_lo, packed in 32 bits when the range allows
  for (int s2 = 0; s2 < 3; ++s2) {
    SpaceDev &S2 = c->sp[s2];
    const uint32_t *m = s2 == SP_H1 ? (S2.xok ? reinterpret_cast<const uint32_t *>(S2.xmap) : nullptr)
                                    : (S2.xvok ? S2.xvmap : nullptr);
    if (!m) continue;
    const int64_t words = c->nel_local * (s2 == SP_H1 ? xmap_points(A.p, c->sp[SP_H1].xc)
                                                      : xv_map_words(s2, A.p, c->sp[SP_H1].xc));
    std::vector<uint32_t> h((size_t)words);
    if (cudaMemcpy(h.data(), m, sizeof(uint32_t) * words, cudaMemcpyDeviceToHost) != cudaSuccess)
      return bail(LOR_ERR_CUDA, "key range");
    int64_t lo = INT64_MAX, hi = -1;
    for (uint32_t v : h) {
      if (v == 0xffffffffu) continue;
      const int64_t g = v & 0x7fffffffu;
      lo = std::min(lo, g);
      hi = std::max(hi, g);
    }
    S2.key_lo = hi < 0 ? 0 : lo;
    S2.key_hi = hi + 1;
  }
  if (A.dim == 2 && A.nranks == 1) {
    std::string why2;
    if (!vec2d_setup(c, plan, why2)) return bail(LOR_ERR_CUDA, "2D vector spaces: " + why2);
  }
  // p = 1: a macro-element is a single LOR cell, nothing of its structure is left to exploit, and
  // one CTA per element spends its time on per-element overhead; on one rank the H1 assembly takes
  // the per-row path of lor_legacy.cu instead (dense 8x8 cell matrices, one warp per row over the
  // dof -> cell transpose; 4.4x faster at 96^3 elements). LOR_ROWPATH=0 keeps the extended frame.
  if (A.dim == 3 && A.p == 1 && A.nranks == 1 && c->sp[SP_H1].valid && c->nel_local > 0 &&
      !(getenv("LOR_ROWPATH") && !atoi(getenv("LOR_ROWPATH")))) {
    c->h1_rows = lor_legacy_setup(c) == LOR_OK;
    c->last_error.clear();
  }
  // the same per-row scheme for ND / RT at p = 1 (element = cell; its restriction and signs are the
  // space's own): ND 15.2 -> 4.2 ms (vs the element + merge passes), RT 9.8 -> 2.2 ms (vs the
  // extended frame) at 96^3 elements
  for (int sv = SP_ND; sv <= SP_RT; ++sv) {
    SpaceDev &V = c->sp[sv];
    const int K = rv_dofs_per_cell(sv);
    if (!(A.dim == 3 && A.p == 1 && A.nranks == 1 && V.valid && V.emap && V.esgn && c->nel_local > 0 &&
          c->nel_local * K < (int64_t(1) << 31) && !(getenv("LOR_ROWPATH") && !atoi(getenv("LOR_ROWPATH")))))
      continue;
    if (dev_alloc(c, &V.rv_off, V.n_local + 1) || dev_alloc(c, &V.rv_ent, c->nel_local * K) ||
        dev_alloc(c, &V.rv_ea, c->nel_local * rv_ea_words(sv)))
      return bail(LOR_ERR_OUT_OF_MEMORY, "per-row path (vector spaces)");
    if (launch_transpose(V.emap, c->nel_local * K, V.row_begin, V.n_local, V.cnt, V.rv_off, V.rv_ent, V.scan_status,
                         V.tile_ctr, c->stream) != cudaSuccess)
      return bail(LOR_ERR_CUDA, "per-row path (vector spaces)");
    // a warp ranks <= 64 candidates: dofs in at most 64 / K cells (edges of valence <= 5)
    std::vector<int64_t> ho((size_t)V.n_local + 1);
    if (cudaMemcpy(ho.data(), V.rv_off, sizeof(int64_t) * ho.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
      return bail(LOR_ERR_CUDA, "per-row path (vector spaces)");
    int64_t mx = 0;
    for (int64_t r = 0; r < V.n_local; ++r) mx = std::max(mx, ho[(size_t)r + 1] - ho[(size_t)r]);
    V.rv = mx * K <= 64;
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(LOR_ERR_CUDA, "setup sync");
  *out = c;
  return LOR_OK;
}

lor_status lor_destroy(lor_ctx c) {
  if (!c) return LOR_OK;
  cudaSetDevice(c->device);
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_pack) cudaEventDestroy(c->ev_pack);
  if (c->ev_xchg) cudaEventDestroy(c->ev_xchg);
  for (void *p : c->allocs) cudaFree(p);
  for (int i = 0; i < 8; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  delete c;
  return LOR_OK;
}

lor_status lor_sync(lor_ctx c) {
  if (!c) return LOR_ERR_INVALID_ARGUMENT;
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  int err[4];
  CUDA_TRY(c, cudaMemcpy(err, c->err, sizeof(err), cudaMemcpyDeviceToHost));
  if (err[3]) {
    cudaMemset(c->err, 0, sizeof(err));
    return fail(c, LOR_ERR_INVALID_ARGUMENT, "lor_eliminate_bc: essential dof outside [0, n_rows_local)");
  }
  if (err[0] == 3) {
    cudaMemset(c->err, 0, sizeof(err));
    return fail(c, LOR_ERR_UNSUPPORTED, "per-row path: a dof in more cells than a warp ranks");
  }
  if (err[0]) {
    cudaMemset(c->err, 0, sizeof(err));
    char buf[160];
    snprintf(buf, sizeof buf, "degenerate-geometry(element=%d, cell=%d): det J <= 0", err[1], err[2]);
    return fail(c, LOR_ERR_DEGENERATE_GEOMETRY, buf);
  }
  return LOR_OK;
}

const char *lor_last_error(lor_ctx c) { return c ? c->last_error.c_str() : g_setup_error.c_str(); }

lor_status lor_query(lor_ctx c, lor_space space, int64_t *n_rows_local, int64_t *row_begin, int64_t *n_rows_global,
                     int64_t *nnz_local) {
  if (!c || space < 0 || space > 2) return LOR_ERR_INVALID_ARGUMENT;
  if (c->dim == 2 && space != LOR_H1) {
    const lor_ctx_s::Vec2 &V = c->v2[space];
    if (!V.ok) return fail(c, LOR_ERR_UNSUPPORTED, "2D ND / RT: one rank only");
    if (n_rows_local) *n_rows_local = V.n;
    if (row_begin) *row_begin = 0;
    if (n_rows_global) *n_rows_global = V.n;
    if (nnz_local) *nnz_local = V.nnz;
    return LOR_OK;
  }
  const SpaceDev &S = c->sp[space];
  if (!S.valid) return fail(c, LOR_ERR_UNSUPPORTED, "space not available");
  if (n_rows_local) *n_rows_local = S.n_local;
  if (row_begin) *row_begin = S.row_begin;
  if (n_rows_global) *n_rows_global = S.n_global;
  if (nnz_local) *nnz_local = S.nnz_local;
  return LOR_OK;
}

lor_status lor_query_discrete(lor_ctx c, int which, int64_t *n_rows_local, int64_t *nnz_local, int64_t *n_cols_global) {
  if (!c || which < 0 || which > 2) return LOR_ERR_INVALID_ARGUMENT;
  if (c->dim == 2 && which != 1) {  // 2D: gradient (ND rows) and rotated gradient (RT rows)
    const lor_ctx_s::Vec2 &V = c->v2[which == 0 ? SP_ND : SP_RT];
    if (!V.ok) return fail(c, LOR_ERR_UNSUPPORTED, "2D discrete operators: one rank only");
    if (n_rows_local) *n_rows_local = V.n;
    if (nnz_local) *nnz_local = 2 * V.n;
    if (n_cols_global) *n_cols_global = c->sp[SP_H1].n_global;
    return LOR_OK;
  }
  if (which == 2) return fail(c, LOR_ERR_UNSUPPORTED, "the rotated gradient is 2D");
  if (!c->sp[which == 0 ? SP_ND : SP_RT].valid || !c->sp[which == 0 ? SP_H1 : SP_ND].valid)
    return fail(c, LOR_ERR_UNSUPPORTED, "space not set up (space_mask)");
  if (c->dim != 3) return fail(c, LOR_ERR_UNSUPPORTED, "discrete operators need dim == 3");
  const SpaceDev &R = c->sp[which == 0 ? SP_ND : SP_RT];
  const SpaceDev &C = c->sp[which == 0 ? SP_H1 : SP_ND];
  if (n_rows_local) *n_rows_local = R.n_local;
  if (nnz_local) *nnz_local = R.n_local * (which == 0 ? 2 : 4);
  if (n_cols_global) *n_cols_global = C.n_global;
  return LOR_OK;
}

lor_status lor_assemble_h1(lor_ctx c, double alpha, double beta, lor_quad quad, lor_csr *out) {
  return assemble(c, SP_H1, alpha, beta, quad, out);
}
lor_status lor_assemble_nd(lor_ctx c, double alpha, double beta, lor_quad quad, lor_csr *out) {
  return assemble(c, SP_ND, alpha, beta, quad, out);
}
lor_status lor_assemble_rt(lor_ctx c, double alpha, double beta, lor_quad quad, lor_csr *out) {
  return assemble(c, SP_RT, alpha, beta, quad, out);
}

lor_status lor_reassemble_h1(lor_ctx c, double alpha, double beta, lor_quad quad, lor_csr *out) {
  return assemble(c, SP_H1, alpha, beta, quad, out, true);
}
lor_status lor_reassemble_nd(lor_ctx c, double alpha, double beta, lor_quad quad, lor_csr *out) {
  return assemble(c, SP_ND, alpha, beta, quad, out, true);
}
lor_status lor_reassemble_rt(lor_ctx c, double alpha, double beta, lor_quad quad, lor_csr *out) {
  return assemble(c, SP_RT, alpha, beta, quad, out, true);
}

lor_status lor_update_coordinates(lor_ctx c, const double *elem_nodes) {
  if (!c || !elem_nodes) return LOR_ERR_INVALID_ARGUMENT;
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int np = (c->dim == 3) ? (c->p + 1) * (c->p + 1) * (c->p + 1) : (c->p + 1) * (c->p + 1);
  const size_t raw = (size_t)c->dim * np * sizeof(double);
  if (c->nel_local > 0)
    CUDA_TRY(c, cudaMemcpy2DAsync(c->X, c->xstride * sizeof(double), elem_nodes, raw, raw, (size_t)c->nel_local,
                                  cudaMemcpyDefault, c->stream));
  if (c->leg_lmap)  // the broken LOR coordinates of the per-row path follow
    CUDA_TRY(c, launch_leg_mesh(c->p, c->nel_local, c->sp[SP_H1].emap, c->X, c->xstride, c->leg_lmap, c->leg_lx, c->stream));
  return exchange_ghost_coords(c);  // extended frame on several ranks: the ghost layer follows
}

lor_status lor_set_coefficients(lor_ctx c, const double *alpha_e, const double *beta_e) {
  if (!c || (!alpha_e) != (!beta_e)) return LOR_ERR_INVALID_ARGUMENT;
  CUDA_TRY(c, cudaSetDevice(c->device));
  c->vc_ghosts = false;
  if (c->ca_l) { c->ca = c->ca_l; c->cb = c->cb_l; }  // back to the local-only arrays
  if (!alpha_e) {
    c->vc = false;
    return LOR_OK;
  }
  const int64_t np = (c->dim == 3) ? (int64_t)(c->p + 1) * (c->p + 1) * (c->p + 1) : (int64_t)(c->p + 1) * (c->p + 1);
  const size_t bytes = sizeof(double) * std::max<int64_t>(1, c->nel_local * np);
  if (!c->ca) {
    if (dev_alloc(c, &c->ca, bytes / sizeof(double)) || dev_alloc(c, &c->cb, bytes / sizeof(double)))
      return fail(c, LOR_ERR_OUT_OF_MEMORY, "coefficient E-vectors");
    c->ca_l = c->ca;
    c->cb_l = c->cb;
  }
  if (c->nel_local > 0) {
    CUDA_TRY(c, cudaMemcpyAsync(c->ca, alpha_e, sizeof(double) * c->nel_local * np, cudaMemcpyDefault, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->cb, beta_e, sizeof(double) * c->nel_local * np, cudaMemcpyDefault, c->stream));
  }
  c->vc = true;
  return LOR_OK;
}

lor_status lor_legacy_setup(lor_ctx c) {
  if (!c) return LOR_ERR_INVALID_ARGUMENT;
  if (c->dim != 3 || c->nranks != 1) return fail(c, LOR_ERR_UNSUPPORTED, "legacy comparator: 3D, one rank");
  SpaceDev &S = c->sp[SP_H1];
  if (!S.emap) return fail(c, LOR_ERR_UNSUPPORTED, "legacy comparator needs the H1 element restriction");
  if (c->leg_lmap) return LOR_OK;
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int64_t ncell = c->nel_local * (int64_t)c->p * c->p * c->p;
  if (ncell * 8 >= (int64_t(1) << 31)) return fail(c, LOR_ERR_UNSUPPORTED, "legacy comparator: 8 ncell >= 2^31");
  if (dev_alloc(c, &c->leg_lmap, ncell * 8) || dev_alloc(c, &c->leg_lx, ncell * 24) ||
      dev_alloc(c, &c->leg_ea, ncell * 64) || dev_alloc(c, &c->leg_off, S.n_local + 1) ||
      dev_alloc(c, &c->leg_ent, ncell * 8))
    return fail(c, LOR_ERR_OUT_OF_MEMORY, "legacy comparator workspaces");
  c->leg_ncell = ncell;
  CUDA_TRY(c, launch_leg_mesh(c->p, c->nel_local, S.emap, c->X, c->xstride, c->leg_lmap, c->leg_lx, c->stream));
  CUDA_TRY(c, launch_transpose(c->leg_lmap, ncell * 8, S.row_begin, S.n_local, S.cnt, c->leg_off, c->leg_ent,
                               S.scan_status, S.tile_ctr, c->stream));
  c->launches += 5;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return LOR_OK;
}

lor_status lor_legacy_assemble_h1(lor_ctx c, double alpha, double beta, lor_csr *out) {
  if (!c || !out || !out->row_ptr) return LOR_ERR_INVALID_ARGUMENT;
  if (!c->leg_lmap) return fail(c, LOR_ERR_INVALID_ARGUMENT, "lor_legacy_setup first");
  SpaceDev &S = c->sp[SP_H1];
  if (S.nnz_local > 0 && (!out->col || !out->val)) return fail(c, LOR_ERR_INVALID_ARGUMENT, "null output buffer");
  if (out->cap_nnz < S.nnz_local) return fail(c, LOR_ERR_BUFFER_TOO_SMALL, "cap_nnz < nnz_local");
  CUDA_TRY(c, cudaSetDevice(c->device));
  c->nphase = 0;
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  CUDA_TRY(c, launch_leg_ea(c->leg_ncell, c->p * c->p * c->p, c->leg_lx, alpha, beta, c->leg_ea, c->err, c->stream));
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  LegArgs a{S.n_local, c->leg_off, c->leg_ent, c->leg_lmap, c->leg_ea, out->row_ptr, out->col, out->val, S.cnt};
  CUDA_TRY(c, launch_leg_rows(a, false, c->stream));
  CUDA_TRY(c, launch_scan(S.cnt, out->row_ptr, S.n_local, S.scan_status, S.tile_ctr, c->stream));
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  CUDA_TRY(c, launch_leg_rows(a, true, c->stream));
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  c->launches += 4;
  return LOR_OK;
}

lor_status lor_set_coefficients_global(lor_ctx c, const double *alpha_all, const double *beta_all) {
  if (!c || !alpha_all || !beta_all) return LOR_ERR_INVALID_ARGUMENT;
  const int64_t np = (c->dim == 3) ? (int64_t)(c->p + 1) * (c->p + 1) * (c->p + 1) : (int64_t)(c->p + 1) * (c->p + 1);
  lor_status st = lor_set_coefficients(c, alpha_all + c->elem_begin * np, beta_all + c->elem_begin * np);
  if (st || c->n_xghost == 0) return st;
  // the ghost layer's coefficients after the local ones (the layout of the coordinate array X)
  const int64_t nl = c->nel_local, ng = c->n_xghost;
  if (!c->ca_g && (dev_alloc(c, &c->ca_g, (nl + ng) * np) || dev_alloc(c, &c->cb_g, (nl + ng) * np)))
    return fail(c, LOR_ERR_OUT_OF_MEMORY, "ghost coefficients");
  double *a2 = c->ca_g, *b2 = c->cb_g;
  CUDA_TRY(c, cudaMemcpyAsync(a2, c->ca, sizeof(double) * nl * np, cudaMemcpyDeviceToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(b2, c->cb, sizeof(double) * nl * np, cudaMemcpyDeviceToDevice, c->stream));
  std::vector<double> ga((size_t)(ng * np)), gb((size_t)(ng * np));
  for (int64_t g = 0; g < ng; ++g) {
    memcpy(&ga[(size_t)(g * np)], alpha_all + c->xghost_ids[(size_t)g] * np, sizeof(double) * np);
    memcpy(&gb[(size_t)(g * np)], beta_all + c->xghost_ids[(size_t)g] * np, sizeof(double) * np);
  }
  CUDA_TRY(c, cudaMemcpy(a2 + nl * np, ga.data(), sizeof(double) * ga.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(c, cudaMemcpy(b2 + nl * np, gb.data(), sizeof(double) * gb.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->ca = a2;
  c->cb = b2;
  c->vc_ghosts = true;
  return LOR_OK;
}

lor_status lor_set_exchange(lor_ctx c, int mode) {
  if (!c || (mode != 0 && mode != 1)) return LOR_ERR_INVALID_ARGUMENT;
  if (mode == 0 && c->nranks > 1 && !c->comm) return fail(c, LOR_ERR_NCCL, "no NCCL communicator");
  c->exchange_mode = mode;
  return LOR_OK;
}

lor_status lor_exchange_copy(lor_ctx dst, lor_ctx src, lor_space space) {
  if (!dst || !src || space < 0 || space > 2) return LOR_ERR_INVALID_ARGUMENT;
  SpaceDev &D = dst->sp[space];
  SpaceDev &S = src->sp[space];
  const int q = src->rank, r = dst->rank;
  if (D.recv_count[q] != S.send_count[r]) return fail(dst, LOR_ERR_INVALID_ARGUMENT, "exchange plan mismatch");
  if (D.recv_count[q] == 0) return LOR_OK;
  const size_t rb = (size_t)S.rstride * sizeof(RecEntry);
  CUDA_TRY(dst, cudaStreamSynchronize(src->stream));
  CUDA_TRY(dst, cudaMemcpyAsync(reinterpret_cast<char *>(D.scratch) + D.recv_begin[q] * rb,
                                reinterpret_cast<char *>(S.scratch) + S.send_begin[r] * rb, D.recv_count[q] * rb,
                                cudaMemcpyDeviceToDevice, dst->stream));
  return LOR_OK;
}

lor_status lor_assemble_finish(lor_ctx c, lor_space space, lor_csr *out) {
  if (!c || space < 0 || space > 2 || !out) return LOR_ERR_INVALID_ARGUMENT;
  SpaceDev &S = c->sp[space];
  if (!S.pending_exchange) return LOR_OK;
  S.pending_exchange = 0;
  lor_status st = finish(c, space, out);
  if (st) return st;
  CUDA_TRY(c, cudaEventRecord(c->ev[c->nphase++], c->stream));
  return LOR_OK;
}

lor_status lor_discrete_rotgrad(lor_ctx c, lor_csr *out) {
  if (!c || !out) return LOR_ERR_INVALID_ARGUMENT;
  if (c->dim != 2) return fail(c, LOR_ERR_UNSUPPORTED, "the rotated gradient is 2D");
  return vec2d_discrete(c, SP_RT, out);
}

lor_status lor_discrete_grad(lor_ctx c, lor_csr *out) {
  if (!c || !out) return LOR_ERR_INVALID_ARGUMENT;
  if (c->dim == 2) return vec2d_discrete(c, SP_ND, out);
  if (c->dim != 3) return fail(c, LOR_ERR_UNSUPPORTED, "dim == 3 only");
  const SpaceDev &R = c->sp[SP_ND];
  if (!R.valid) return fail(c, LOR_ERR_UNSUPPORTED, "ND not set up (space_mask)");
  if (out->cap_nnz < 2 * R.n_local) return fail(c, LOR_ERR_BUFFER_TOO_SMALL, "cap_nnz < 2 n_rows");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const SpaceDev &Cs = c->sp[SP_H1];
  if (R.emap && Cs.emap) {  // one pass: columns, values and the stride row pointer
    DiscMapArgs m{c->p, c->nel_local, c->topo, R.emap, R.esgn, Cs.emap, Cs.esgn, R.row_begin, out->col, out->val,
                  out->row_ptr, R.n_local};
    if (R.n_local == 0) CUDA_TRY(c, launch_rowptr_stride(out->row_ptr, 0, 2, c->stream));
    CUDA_TRY(c, launch_discrete_map(0, m, c->stream));
    c->launches--;  // no separate row-pointer kernel
  } else {
    CUDA_TRY(c, launch_rowptr_stride(out->row_ptr, R.n_local, 2, c->stream));
    DiscArgs a;
    a.p = c->p;
    a.nel_local = c->nel_local;
    a.topo = c->topo;
    fill_base(R, a.base_row);
    fill_base(c->sp[SP_H1], a.base_col);
    a.row_begin = R.row_begin;
    a.col = out->col;
    a.val = out->val;
    CUDA_TRY(c, launch_discrete(0, a, c->stream));
  }
  c->launches += 2;
  return LOR_OK;
}

lor_status lor_discrete_curl(lor_ctx c, lor_csr *out) {
  if (!c || !out) return LOR_ERR_INVALID_ARGUMENT;
  if (c->dim != 3) return fail(c, LOR_ERR_UNSUPPORTED, "dim == 3 only");
  const SpaceDev &R = c->sp[SP_RT];
  if (!R.valid || !c->sp[SP_ND].valid) return fail(c, LOR_ERR_UNSUPPORTED, "RT / ND not set up (space_mask)");
  if (out->cap_nnz < 4 * R.n_local) return fail(c, LOR_ERR_BUFFER_TOO_SMALL, "cap_nnz < 4 n_rows");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const SpaceDev &Cs = c->sp[SP_ND];
  if (R.emap && Cs.emap) {  // one pass: columns, values and the stride row pointer
    DiscMapArgs m{c->p, c->nel_local, c->topo, R.emap, R.esgn, Cs.emap, Cs.esgn, R.row_begin, out->col, out->val,
                  out->row_ptr, R.n_local};
    if (R.n_local == 0) CUDA_TRY(c, launch_rowptr_stride(out->row_ptr, 0, 4, c->stream));
    CUDA_TRY(c, launch_discrete_map(1, m, c->stream));
    c->launches--;
  } else {
    CUDA_TRY(c, launch_rowptr_stride(out->row_ptr, R.n_local, 4, c->stream));
    DiscArgs a;
    a.p = c->p;
    a.nel_local = c->nel_local;
    a.topo = c->topo;
    fill_base(R, a.base_row);
    fill_base(c->sp[SP_ND], a.base_col);
    a.row_begin = R.row_begin;
    a.col = out->col;
    a.val = out->val;
    CUDA_TRY(c, launch_discrete(1, a, c->stream));
  }
  c->launches += 2;
  return LOR_OK;
}

lor_status lor_dof_map(lor_ctx c, lor_space space, int32_t *elem_dofs, int8_t *signs) {
  if (!c || space < 0 || space > 2 || !elem_dofs) return LOR_ERR_INVALID_ARGUMENT;
  if (c->dim == 2 && space != LOR_H1) {
    const lor_ctx_s::Vec2 &V = c->v2[space];
    if (!V.ok) return fail(c, LOR_ERR_UNSUPPORTED, "2D ND / RT: one rank only");
    const size_t n = (size_t)c->nel_local * 2 * c->p * (c->p + 1);
    CUDA_TRY(c, cudaMemcpyAsync(elem_dofs, V.map, n * 4, cudaMemcpyDeviceToDevice, c->stream));
    if (signs) CUDA_TRY(c, cudaMemcpyAsync(signs, V.sgn, n, cudaMemcpyDeviceToDevice, c->stream));
    return LOR_OK;
  }
  const SpaceDev &S = c->sp[space];
  if (!S.valid) return fail(c, LOR_ERR_UNSUPPORTED, "space not available");
  CUDA_TRY(c, cudaSetDevice(c->device));
  DofmapArgs a;
  a.p = c->p;
  a.ndpe = S.ndpe;
  a.nel_local = c->nel_local;
  a.topo = c->topo;
  fill_base(S, a.base);
  a.map = elem_dofs;
  a.sign = signs;
  CUDA_TRY(c, launch_dofmap(c->dim, space, a, c->stream));
  c->launches++;
  return LOR_OK;
}

lor_status lor_query_transpose(lor_ctx c, lor_space space, int64_t *n_entries) {
  if (!c || space < 0 || space > 2 || !n_entries) return LOR_ERR_INVALID_ARGUMENT;
  const SpaceDev &S = c->sp[space];
  if (!S.valid) return fail(c, LOR_ERR_UNSUPPORTED, "space not available");
  *n_entries = S.n_tr;
  return LOR_OK;
}

lor_status lor_dof_transpose(lor_ctx c, lor_space space, int64_t *offsets, int32_t *entries, int64_t cap_entries) {
  if (!c || space < 0 || space > 2 || !offsets || (!entries && cap_entries > 0)) return LOR_ERR_INVALID_ARGUMENT;
  SpaceDev &S = c->sp[space];
  if (!S.valid) return fail(c, LOR_ERR_UNSUPPORTED, "space not available");
  if (cap_entries < S.n_tr) return fail(c, LOR_ERR_BUFFER_TOO_SMALL, "cap_entries < lor_query_transpose");
  if ((int64_t)c->nel_local * S.ndpe >= (int64_t(1) << 31))
    return fail(c, LOR_ERR_INVALID_ARGUMENT, "n_elem_local * ndof_per_el exceeds int32");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int32_t *map = S.emap;
  if (!map) {  // element restriction of this rank's elements into a context workspace
    if (!S.trmap) {
      CUDA_TRY(c, cudaMalloc((void **)&S.trmap, sizeof(int32_t) * std::max<int64_t>(1, c->nel_local * S.ndpe)));
      c->allocs.push_back(S.trmap);
    }
    DofmapArgs a;
    a.p = c->p;
    a.ndpe = S.ndpe;
    a.nel_local = c->nel_local;
    a.topo = c->topo;
    fill_base(S, a.base);
    a.map = S.trmap;
    a.sign = nullptr;
    CUDA_TRY(c, launch_dofmap(c->dim, space, a, c->stream));
    c->launches++;
    map = S.trmap;
  }
  CUDA_TRY(c, launch_transpose(map, c->nel_local * S.ndpe, S.row_begin, S.n_local, S.cnt, offsets, entries,
                               S.scan_status, S.tile_ctr, c->stream));
  c->launches += 4;
  return LOR_OK;
}

lor_status lor_coordinates(lor_ctx c, double *xyz) {
  if (!c || !xyz) return LOR_ERR_INVALID_ARGUMENT;
  const SpaceDev &S = c->sp[SP_H1];
  CUDA_TRY(c, cudaSetDevice(c->device));
  CoordArgs a;
  a.p = c->p;
  a.nel_local = c->nel_local;
  a.topo = c->topo;
  fill_base(S, a.base);
  a.X = c->X;
  a.xstride = c->xstride;
  a.row_begin = S.row_begin;
  a.n_local = S.n_local;
  a.out = xyz;
  a.emap = S.emap;
  CUDA_TRY(c, launch_coords(c->dim, a, c->stream));
  if (c->nel_local > 0) c->launches++;
  return LOR_OK;
}

lor_status lor_query_elements(lor_ctx c, int64_t *elem_begin, int64_t *n_elem_local, int *nh1, int *nnd, int *nrt) {
  if (!c) return LOR_ERR_INVALID_ARGUMENT;
  if (elem_begin) *elem_begin = c->elem_begin;
  if (n_elem_local) *n_elem_local = c->nel_local;
  const int nv2 = c->dim == 2 ? 2 * c->p * (c->p + 1) : 0;  // 2D ND / RT: lattice edges
  if (nh1) *nh1 = c->sp[0].ndpe;
  if (nnd) *nnd = c->dim == 2 ? nv2 : c->sp[1].ndpe;
  if (nrt) *nrt = c->dim == 2 ? nv2 : c->sp[2].ndpe;
  return LOR_OK;
}

int64_t lor_kernel_launches(lor_ctx c) { return c ? c->launches : 0; }

int64_t lor_debug_dump(lor_ctx c, int what, lor_space space, void *host_out, int64_t cap) {
  if (!c || space < 0 || space > 2 || !host_out || !c->sp[space].valid) return 0;
  const SpaceDev &S = c->sp[space];
  int64_t bytes = 0;
  const void *src = nullptr;
  if (what == 0) { bytes = tab_slot_entries(c->dim, space) * 4; src = S.tslot; }
  else if (what == 1) { bytes = tab_size_entries(c->dim, space); src = S.tsize; }
  else if (what == 2 && c->tstamp) { bytes = c->nel_local * 16 * 8; src = c->tstamp; }
  else return 0;
  if (bytes > cap) return 0;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (cudaMemcpy(host_out, src, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return bytes;
}

int lor_fill_path(lor_ctx c, lor_space space) {
  if (!c || space < 0 || space > 2 || !c->sp[space].valid) return -1;
  if (((space == LOR_H1 && c->h1_rows) || c->sp[space].rv) && !c->vc) return 2;
  if (c->vc)
    return ((c->sp[space].xok || (space == LOR_RT && c->sp[space].xvok)) && (c->nranks == 1 || c->vc_ghosts)) ? 1 : 0;
  return (c->sp[space].xok || c->sp[space].xvok) ? 1 : 0;
}

int lor_last_phase_ms(lor_ctx c, float *ms, int cap) {
  if (!c || !ms) return 0;
  int n = 0;
  for (int i = 0; i + 1 < c->nphase && n < cap; ++i) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, c->ev[i], c->ev[i + 1]) != cudaSuccess) t = -1.f;
    ms[n++] = t;
  }
  return n;
}

}  // extern "C"
// ------------------------------------------------------------------ ParCSR split + BC elimination
namespace {

// rows / columns of operator op: 0..2 the space's matrix (square), 3 discrete gradient (ND x H1),
// 4 discrete curl (RT x ND)
bool op_spaces(lor_ctx c, int op, int &rs, int &cs) {
  if (op >= 0 && op <= 2) { rs = cs = op; }
  else if (op == 3) { rs = SP_ND; cs = SP_H1; }
  else if (op == 4) { rs = SP_RT; cs = SP_ND; }
  else if (op == 5) { rs = SP_RT; cs = SP_H1; }
  else return false;
  if (c->dim == 2) {  // 2D: ND / RT from lor_vec2d (one rank); gradient and rotated gradient
    if (op == 4) return false;
    auto ok = [&](int sp) { return sp == SP_H1 ? c->sp[SP_H1].valid : c->v2[sp].ok; };
    return ok(rs) && ok(cs);
  }
  return op != 5 && c->sp[rs].valid && c->sp[cs].valid;
}

// rows / columns of an operator: local rows, first row, owned column range, global columns and the
// device rank ranges of the column space
void op_dims(lor_ctx c, int rs, int cs, int64_t &n, int64_t &rb, int64_t &cb, int64_t &cn, int64_t &ng,
             const int64_t *&croff) {
  if (c->dim == 2 && rs != SP_H1) { n = c->v2[rs].n; rb = 0; }
  else { n = c->sp[rs].n_local; rb = c->sp[rs].row_begin; }
  if (c->dim == 2 && cs != SP_H1) { cb = 0; cn = ng = c->v2[cs].n; croff = c->v2[cs].droff; }
  else { cb = c->sp[cs].row_begin; cn = c->sp[cs].n_local; ng = c->sp[cs].n_global; croff = c->sp[cs].droff; }
}

template <class T>
cudaError_t grow(lor_ctx c, T **p, int64_t &cap, int64_t need) {
  if (*p && cap >= need) return cudaSuccess;
  if (*p) {
    c->allocs.erase(std::find(c->allocs.begin(), c->allocs.end(), (void *)*p));
    cudaFree(*p);
    *p = nullptr;
  }
  cap = std::max<int64_t>(need, 1);
  cudaError_t e = cudaMalloc((void **)p, sizeof(T) * cap);
  if (e == cudaSuccess) c->allocs.push_back(*p);
  return e;
}

lor_status side_stream(lor_ctx c) {
  if (c->side) return LOR_OK;
  CUDA_TRY(c, cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming));
  CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_xchg, cudaEventDisableTiming));
  return LOR_OK;
}

PcArgs pc_args(lor_ctx c, PcState &P, const lor_csr *A) {
  PcArgs a{};
  a.n = P.n;
  a.rp = A->row_ptr;
  a.col = A->col;
  a.val = A->val;
  a.cb = P.cb;
  a.ce = P.ce;
  a.row_begin = P.row_begin;
  a.square = P.square;
  a.croff = P.croff;
  a.nranks = c->nranks;
  a.ncols = P.ncols;
  a.bitmap = P.bitmap;
  a.wpre = P.wpre;
  a.cnt_d = P.cnt_d;
  a.cnt_o = P.cnt_o;
  a.rowmask = P.rowmask;
  a.err = c->err + 3;
  return a;
}

}  // namespace
extern "C" {

lor_status lor_parcsr_prepare(lor_ctx c, int op, const lor_csr *A, int64_t *nnz_diag, int64_t *nnz_offd,
                              int64_t *n_col_offd) {
  int rs, cs;
  if (!c || !A || !A->row_ptr) return LOR_ERR_INVALID_ARGUMENT;
  if (!op_spaces(c, op, rs, cs)) return fail(c, LOR_ERR_UNSUPPORTED, "operator not available for this mesh");
  if (c->nranks > 32) return fail(c, LOR_ERR_UNSUPPORTED, "ParCSR split: nranks > 32");
  PcState &P = c->pc[op];
  CUDA_TRY(c, cudaSetDevice(c->device));
  P.ready = false;
  P.pending = 0;
  int64_t cn = 0;
  op_dims(c, rs, cs, P.n, P.row_begin, P.cb, cn, P.ncols, P.croff);
  P.ce = P.cb + cn;
  P.square = op <= 2;
  P.nw = (P.ncols + 31) / 32;
  const int64_t n1 = P.n + 1;
  if (!P.bitmap) {  // sizes are topological: allocated once per operator
    if (dev_alloc(c, &P.bitmap, P.nw + 1) || dev_alloc(c, &P.rowmask, n1) || dev_alloc(c, &P.cnt_d, n1) ||
        dev_alloc(c, &P.cnt_o, n1) || dev_alloc(c, &P.flag, n1) || dev_alloc(c, &P.pc, P.nw + 1) ||
        dev_alloc(c, &P.wpre, P.nw + 2) || dev_alloc(c, &P.drp, n1) || dev_alloc(c, &P.orp, n1) ||
        dev_alloc(c, &P.pos, std::max(n1, P.nw + 2)) ||
        dev_alloc(c, &P.status, scan_status_words(std::max(P.n, P.nw))) || dev_alloc(c, &P.tile_ctr, 1) ||
        (P.square && dev_alloc(c, &P.marker, n1)))
      return fail(c, LOR_ERR_OUT_OF_MEMORY, "parcsr workspace");
  }
  CUDA_TRY(c, cudaMemsetAsync(P.bitmap, 0, sizeof(uint32_t) * (P.nw + 1), c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->err + 3, 0, sizeof(int), c->stream));
  PcArgs a = pc_args(c, P, A);
  CUDA_TRY(c, launch_pc_count(a, c->stream));
  CUDA_TRY(c, launch_scan(P.cnt_d, P.drp, P.n, P.status, P.tile_ctr, c->stream));
  CUDA_TRY(c, launch_scan(P.cnt_o, P.orp, P.n, P.status, P.tile_ctr, c->stream));
  CUDA_TRY(c, launch_pc_popc(P.bitmap, P.nw, P.pc, c->stream));
  CUDA_TRY(c, launch_scan(P.pc, P.wpre, P.nw, P.status, P.tile_ctr, c->stream));
  c->launches += 5;
  int64_t tot[3] = {0, 0, 0};
  CUDA_TRY(c, cudaMemcpyAsync(&tot[0], P.drp + P.n, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(&tot[1], P.orp + P.n, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(&tot[2], P.wpre + P.nw, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  int bad = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&bad, c->err + 3, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (bad == 1) return fail(c, LOR_ERR_INVALID_ARGUMENT, "ParCSR split: a row of a square operator lacks its diagonal");
  if (bad) return fail(c, LOR_ERR_INVALID_ARGUMENT, "ParCSR split: column id outside [0, n_cols_global)");
  P.nnz_d = tot[0];
  P.nnz_o = tot[1];
  P.n_col_offd = tot[2];
  // marker exchange plan (square operators on several ranks): peer q's segment of col_map_offd and
  // the owned rows whose offd columns q owns -- by structural symmetry exactly the rows q's
  // col_map_offd holds from this rank, in the same (ascending) order
  P.send_off.assign(c->nranks + 1, 0);
  P.send_cnt.assign(c->nranks, 0);
  P.recv_lo.assign(c->nranks + 1, 0);
  if (P.square && c->nranks > 1) {
    CUDA_TRY(c, launch_pc_peer_lo(P.bitmap, P.wpre, P.nw, P.croff, c->nranks, P.pos, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(P.recv_lo.data(), P.pos, sizeof(int64_t) * (c->nranks + 1), cudaMemcpyDeviceToHost,
                                c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    for (int pass = 0; pass < 2; ++pass) {  // 0: counts per peer, 1: the lists
      for (int q = 0; q < c->nranks; ++q) {
        if (q == c->rank) continue;
        CUDA_TRY(c, launch_pc_flag(P.rowmask, P.n, q, P.flag, c->stream));
        CUDA_TRY(c, launch_scan(P.flag, P.pos, P.n, P.status, P.tile_ctr, c->stream));
        c->launches += 2;
        if (pass == 0) {
          CUDA_TRY(c, cudaMemcpyAsync(&P.send_cnt[q], P.pos + P.n, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
        } else if (P.send_cnt[q] > 0) {
          CUDA_TRY(c, launch_pc_scatter(P.rowmask, P.pos, P.n, q, P.send_list + P.send_off[q], c->stream));
          c->launches++;
        }
      }
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      if (pass == 0) {
        for (int q = 0; q < c->nranks; ++q) P.send_off[q + 1] = P.send_off[q] + P.send_cnt[q];
        if (P.send_off[c->nranks] > P.cap_send) {
          if (grow(c, &P.send_list, P.cap_send, P.send_off[c->nranks]) ||
              grow(c, &P.sbuf, P.cap_send_b, P.send_off[c->nranks]))
            return fail(c, LOR_ERR_OUT_OF_MEMORY, "parcsr send lists");
        }
      }
    }
  }
  if (P.square && grow(c, &P.omark, P.cap_omark, P.n_col_offd + 1)) return fail(c, LOR_ERR_OUT_OF_MEMORY, "parcsr markers");
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  P.ready = true;
  if (nnz_diag) *nnz_diag = P.nnz_d;
  if (nnz_offd) *nnz_offd = P.nnz_o;
  if (n_col_offd) *n_col_offd = P.n_col_offd;
  return LOR_OK;
}

lor_status lor_parcsr_fill(lor_ctx c, int op, const lor_csr *A, lor_parcsr *M) {
  int rs, cs;
  if (!c || !A || !M || !A->row_ptr) return LOR_ERR_INVALID_ARGUMENT;
  if (!op_spaces(c, op, rs, cs)) return fail(c, LOR_ERR_UNSUPPORTED, "operator not available for this mesh");
  PcState &P = c->pc[op];
  if (!P.ready) return fail(c, LOR_ERR_INVALID_ARGUMENT, "lor_parcsr_fill before lor_parcsr_prepare");
  if (!M->diag_row_ptr || !M->offd_row_ptr || (P.nnz_d > 0 && (!M->diag_col || !M->diag_val)) ||
      (P.nnz_o > 0 && (!M->offd_col || !M->offd_val)) || (P.n_col_offd > 0 && !M->col_map_offd))
    return fail(c, LOR_ERR_INVALID_ARGUMENT, "null ParCSR buffer");
  if (M->cap_diag < P.nnz_d || M->cap_offd < P.nnz_o || M->cap_col_map < P.n_col_offd)
    return fail(c, LOR_ERR_BUFFER_TOO_SMALL, "ParCSR buffers smaller than lor_parcsr_prepare's sizes");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaMemcpyAsync(M->diag_row_ptr, P.drp, sizeof(int64_t) * (P.n + 1), cudaMemcpyDeviceToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(M->offd_row_ptr, P.orp, sizeof(int64_t) * (P.n + 1), cudaMemcpyDeviceToDevice, c->stream));
  PcArgs a = pc_args(c, P, A);
  PcOut o{P.drp, P.orp, M->diag_col, M->offd_col, M->diag_val, M->offd_val};
  CUDA_TRY(c, launch_pc_fill(a, o, P.nnz_o > 0, c->stream));
  c->launches += P.nnz_o > 0 ? 2 : 1;
  if (P.n_col_offd > 0) {
    CUDA_TRY(c, launch_pc_colmap(P.bitmap, P.wpre, P.nw, M->col_map_offd, c->stream));
    c->launches++;
  }
  return LOR_OK;
}

lor_status lor_boundary_dofs(lor_ctx c, lor_space space, int32_t *rows, int64_t cap, int64_t *n) {
  if (!c || space < 0 || space > 2 || !n) return LOR_ERR_INVALID_ARGUMENT;
  const bool v2 = c->dim == 2 && space != LOR_H1;
  if (v2 && !c->v2[space].ok) return fail(c, LOR_ERR_UNSUPPORTED, "2D ND / RT: one rank only");
  if (!v2 && !c->sp[space].valid) return fail(c, LOR_ERR_UNSUPPORTED, "space not available");
  const std::vector<int32_t> &B = v2 ? c->v2[space].bnd : c->sp[space].bnd;
  *n = (int64_t)B.size();
  if (!rows) return LOR_OK;
  if (cap < *n) return fail(c, LOR_ERR_BUFFER_TOO_SMALL, "cap < number of boundary dofs");
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (*n > 0) CUDA_TRY(c, cudaMemcpy(rows, B.data(), sizeof(int32_t) * *n, cudaMemcpyHostToDevice));
  return LOR_OK;
}

lor_status lor_eliminate_bc(lor_ctx c, lor_space space, const int32_t *ess, int64_t n_ess, lor_parcsr *M) {
  if (!c || space < 0 || space > 2 || !M || (n_ess > 0 && !ess) || n_ess < 0) return LOR_ERR_INVALID_ARGUMENT;
  PcState &P = c->pc[space];
  if (!P.ready) return fail(c, LOR_ERR_INVALID_ARGUMENT, "lor_eliminate_bc before lor_parcsr_prepare/fill");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaMemsetAsync(P.marker, 0, P.n + 1, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->err + 3, 0, sizeof(int), c->stream));
  CUDA_TRY(c, launch_bc_mark(ess, n_ess, P.n, P.marker, c->err + 3, c->stream));
  c->launches++;
  const int64_t nsend = P.send_off.empty() ? 0 : P.send_off[c->nranks];
  const bool remote = c->nranks > 1 && P.n_col_offd > 0;
  if (c->nranks > 1) {
    CUDA_TRY(c, launch_bc_pack(P.marker, P.send_list, nsend, P.sbuf, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(P.omark, 0, P.n_col_offd + 1, c->stream));
    if (nsend > 0) c->launches++;
  }
  const bool use_nccl = c->nranks > 1 && c->exchange_mode == 0;
  if (use_nccl) {  // the marker exchange starts first and overlaps the diag / offd-row elimination
    lor_status st = side_stream(c);
    if (st) return st;
    CUDA_TRY(c, cudaEventRecord(c->ev_pack, c->stream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->side, c->ev_pack, 0));
    if (g_nccl.GroupStart() != ncclSuccess) return fail(c, LOR_ERR_NCCL, "ncclGroupStart");
    for (int q = 0; q < c->nranks; ++q) {
      if (q == c->rank) continue;
      ncclResult_t r = ncclSuccess;
      if (P.send_cnt[q] > 0)
        r = g_nccl.Send(P.sbuf + P.send_off[q], P.send_cnt[q], ncclUint8, q, c->comm, c->side);
      if (r == ncclSuccess && P.recv_lo[q + 1] > P.recv_lo[q])
        r = g_nccl.Recv(P.omark + P.recv_lo[q], P.recv_lo[q + 1] - P.recv_lo[q], ncclUint8, q, c->comm, c->side);
      if (r != ncclSuccess) { g_nccl.GroupEnd(); return fail(c, LOR_ERR_NCCL, g_nccl.GetErrorString(r)); }
    }
    if (g_nccl.GroupEnd() != ncclSuccess) return fail(c, LOR_ERR_NCCL, "ncclGroupEnd");
    CUDA_TRY(c, cudaEventRecord(c->ev_xchg, c->side));
  }
  BcArgs b{P.n, M->diag_row_ptr, M->offd_row_ptr, M->diag_col, M->diag_val, M->offd_val};
  CUDA_TRY(c, launch_bc_rows(ess, n_ess, b, c->stream));
  if (n_ess > 0) c->launches++;
  if (!remote) {
    // the sends may still be in flight: later work on the context stream (the next pack) waits
    if (use_nccl) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_xchg, 0));
    return LOR_OK;
  }
  if (!use_nccl) {
    P.pending = 1;
    return LOR_OK;
  }
  CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_xchg, 0));
  CUDA_TRY(c, launch_bc_offd_cols(M->offd_col, P.nnz_o, P.omark, M->offd_val, c->stream));
  if (P.nnz_o > 0) c->launches++;
  return LOR_OK;
}

lor_status lor_bc_exchange_copy(lor_ctx dst, lor_ctx src, lor_space space) {
  if (!dst || !src || space < 0 || space > 2) return LOR_ERR_INVALID_ARGUMENT;
  PcState &D = dst->pc[space], &S = src->pc[space];
  if (!D.ready || !S.ready) return fail(dst, LOR_ERR_INVALID_ARGUMENT, "ParCSR not prepared");
  const int q = src->rank, r = dst->rank;
  const int64_t want = D.recv_lo[q + 1] - D.recv_lo[q];
  if (want != S.send_cnt[r]) return fail(dst, LOR_ERR_INVALID_ARGUMENT, "marker exchange plan mismatch");
  if (want == 0) return LOR_OK;
  CUDA_TRY(dst, cudaStreamSynchronize(src->stream));
  CUDA_TRY(dst, cudaMemcpyAsync(D.omark + D.recv_lo[q], S.sbuf + S.send_off[r], want, cudaMemcpyDeviceToDevice,
                                dst->stream));
  return LOR_OK;
}

lor_status lor_eliminate_bc_finish(lor_ctx c, lor_space space, lor_parcsr *M) {
  if (!c || space < 0 || space > 2 || !M) return LOR_ERR_INVALID_ARGUMENT;
  PcState &P = c->pc[space];
  if (!P.pending) return LOR_OK;
  P.pending = 0;
  CUDA_TRY(c, launch_bc_offd_cols(M->offd_col, P.nnz_o, P.omark, M->offd_val, c->stream));
  if (P.nnz_o > 0) c->launches++;
  return LOR_OK;
}

lor_status lor_parcsr_exchange_counts(lor_ctx c, lor_space space, int64_t *send_counts, int64_t *recv_counts) {
  if (!c || space < 0 || space > 2) return LOR_ERR_INVALID_ARGUMENT;
  const PcState &P = c->pc[space];
  if (!P.ready) return fail(c, LOR_ERR_INVALID_ARGUMENT, "ParCSR not prepared");
  for (int q = 0; q < c->nranks; ++q) {
    if (send_counts) send_counts[q] = P.send_cnt.empty() ? 0 : P.send_cnt[q];
    if (recv_counts) recv_counts[q] = P.recv_lo.empty() ? 0 : P.recv_lo[q + 1] - P.recv_lo[q];
  }
  return LOR_OK;
}

}  // extern "C"
