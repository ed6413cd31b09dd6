// lor_plan.h -- host-side setup plan (see lor_plan.cpp).
#pragma once
#include <stdint.h>

#include <vector>

#include "lor_internal.h"

namespace lorb {

struct PlanInput {
  int dim, p, rank, nranks;
  int64_t n_vert, n_elem;
  const int64_t *elem_vert;
  const int64_t *elem_rank_begin;
};

struct SpacePlan {
  int space = 0;
  bool valid = false;
  int ndpe = 0, maxl = 0;
  int64_t n_global = 0, row_begin = 0, n_local = 0;
  std::vector<int64_t> rank_off;          // [nranks+1]
  std::vector<int32_t> base[4];           // global id of first dof per entity (vertex, edge, face, interior)
  std::vector<ElemSpace> esp;             // per local element
  std::vector<Ose> ose;                   // owned shared entities
  std::vector<int32_t> ose_slots;         // record base per slot
  std::vector<int32_t> ose_elem;          // global element id per slot
  std::vector<int32_t> defer;             // OSE indices finalized after the exchange
  int64_t n_records = 0;                  // scratch records (MAXL entries each)
  std::vector<int64_t> recv_begin, recv_count, send_begin, send_count;  // per peer, in records
};

struct HostPlan {
  int dim = 0, p = 0, rank = 0, nranks = 1;
  int64_t nv = 0, ne = 0, nf = 0, nel = 0;
  int64_t elem_begin = 0, nel_local = 0;
  int64_t n_ent[4] = {0, 0, 0, 0};
  std::vector<int64_t> erb;
  std::vector<int> elem_rank;
  std::vector<int32_t> el_edge, el_face;
  std::vector<uint8_t> el_edge_rev, el_face_code;
  std::vector<int64_t> inc_off[3];
  std::vector<int32_t> inc_el[3];
  std::vector<int64_t> ghost;      // ghost element ids (topology records after the local ones)
  std::vector<ElemTopo> topo;      // local elements, then ghosts
  SpacePlan sp[3];
  const int64_t *EVp = nullptr;    // the caller's elem_vert (valid during lor_setup)

  void build(const PlanInput &in);
  ElemTopo topo_of(int64_t e) const;
  // local rows (ascending) of the owned dofs of space s on the domain boundary: the dofs of every
  // coarse entity lying on a boundary facet (a face -- an edge in 2D -- of exactly one element);
  // the essential dofs of a Dirichlet / tangential / normal trace condition.
  void boundary_rows(int s, std::vector<int32_t> &out) const;
};

int maxl_of(int dim, int space);
int ndpe_of(int dim, int p, int space);
void entity_ndofs(int dim, int p, int space, int64_t nd[4]);
void slot_entity(int dim, int tau, int &type, int &lidx);
void interpolate_evector(int dim, int p, const double *vert, const int64_t *ev, int64_t e0, int64_t n,
                         std::vector<double> &X);

}  // namespace lorb
