// lor_plan.cpp -- host-side setup of the B200 LOR library (native C++, runs once in lor_setup).
//
// Computes, for one rank, everything the assembly kernels treat as setup-time topology (the
// paper reuses the high-order element restriction):
//   * coarse entities: edges keyed by sorted vertex pairs, faces by sorted vertex 4-tuples;
//     edge orientation (min -> max vertex id) and face frames;
//   * entity incidence (sorted element lists): valence, minimal element, slot of each element;
//   * ownership: owner(entity) = rank of its minimal element;
//   * per space, the rank-major global numbering of each entity's dofs (App. A.4/A.6), stored as
//     the global id of each entity's first dof (an entity's dofs are consecutive);
//   * per element topology records (ElemTopo) for local and ghost elements, per element space
//     records (ElemSpace) and the scratch/exchange plan for rows shared by several elements.
// Nothing here is per-assembly work; assembly-time work (counts, scan, sub-cell matrices, CSR
// fill, merge of shared rows, exchange) runs in the CUDA kernels.
#include "lor_plan.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <stdexcept>

namespace lorb {

namespace {

inline int local_edge_3d(int d, int b1, int b2) { return 4 * d + b1 + 2 * b2; }

// corners (tail, head) of local edge le (3D: 4d + b1 + 2b2; 2D: 2d + b1)
inline void edge_ends(int dim, int le, int &tail, int &head) {
  int d;
  if (dim == 3) {
    d = le / 4;
    int b1 = le & 1, b2 = (le >> 1) & 1;
    int u = (d == 0) ? 1 : 0, v = (d == 2) ? 1 : 2;
    tail = (b1 << u) | (b2 << v);
  } else {
    d = le / 2;
    tail = (le & 1) << (1 - d);
  }
  head = tail | (1 << d);
}

// corners of local face lf = 2n + side indexed by (alpha, beta) along the in-face axes (u < v)
inline void face_quad(int lf, int fc[2][2]) {
  int n = lf / 2, side = lf & 1;
  int u = (n == 0) ? 1 : 0, v = (n == 2) ? 1 : 2;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) fc[a][b] = (side << n) | (a << u) | (b << v);
}

struct Key2 {
  uint64_t a, b;
  bool operator<(const Key2 &o) const { return a < o.a || (a == o.a && b < o.b); }
  bool operator==(const Key2 &o) const { return a == o.a && b == o.b; }
};

}  // namespace

int maxl_of(int dim, int space) {
  if (space == SP_H1) return dim == 3 ? 18 : 6;
  if (space == SP_ND) return 20;
  return 6;
}

int ndpe_of(int dim, int p, int space) {
  if (space == SP_H1) return dim == 3 ? (p + 1) * (p + 1) * (p + 1) : (p + 1) * (p + 1);
  if (space == SP_ND) return 3 * p * (p + 1) * (p + 1);
  return 3 * p * p * (p + 1);
}

// dofs per entity type [vertex, edge, face, interior]
void entity_ndofs(int dim, int p, int space, int64_t nd[4]) {
  if (space == SP_H1) {
    nd[0] = 1;
    nd[1] = p - 1;
    nd[2] = (dim == 3) ? (int64_t)(p - 1) * (p - 1) : 0;
    nd[3] = (dim == 3) ? (int64_t)(p - 1) * (p - 1) * (p - 1) : (int64_t)(p - 1) * (p - 1);
  } else if (space == SP_ND) {
    nd[0] = 0;
    nd[1] = p;
    nd[2] = 2 * (int64_t)p * (p - 1);
    nd[3] = 3 * (int64_t)p * (p - 1) * (p - 1);
  } else {
    nd[0] = 0;
    nd[1] = 0;
    nd[2] = (int64_t)p * p;
    nd[3] = 3 * (int64_t)p * p * (p - 1);
  }
}

// entity type of slot tau: 0 vertex, 1 edge, 2 face, 3 interior; and the local entity index
void slot_entity(int dim, int tau, int &type, int &lidx) {
  int c[3] = {tau % 3, (tau / 3) % 3, tau / 9};
  int nI = 0;
  for (int a = 0; a < dim; ++a) nI += (c[a] == 1);
  if (nI == dim) { type = 3; lidx = 0; return; }
  if (nI == 0) {
    type = 0;
    lidx = 0;
    for (int a = 0; a < dim; ++a) lidx |= (c[a] == 2) << a;
    return;
  }
  if (dim == 2) { // nI == 1: edge along the I axis
    int d = (c[0] == 1) ? 0 : 1;
    type = 1;
    lidx = 2 * d + (c[1 - d] == 2);
    return;
  }
  if (nI == 1) {
    int d = (c[0] == 1) ? 0 : (c[1] == 1 ? 1 : 2);
    int u = (d == 0) ? 1 : 0, v = (d == 2) ? 1 : 2;
    type = 1;
    lidx = local_edge_3d(d, c[u] == 2, c[v] == 2);
    return;
  }
  int n = (c[0] != 1) ? 0 : (c[1] != 1 ? 1 : 2);
  type = 2;
  lidx = 2 * n + (c[n] == 2);
}

// topology record of any element e (entity ids, orientation codes, valences, TF_MIN / TF_OWNED
// for this rank); valid after build()
void HostPlan::boundary_rows(int s, std::vector<int32_t> &out) const {
  out.clear();
  const SpacePlan &S = sp[s];
  if (!S.valid) return;
  int64_t nd[4];
  entity_ndofs(dim, p, s, nd);
  const int nc = 1 << dim, nle = (dim == 3) ? 12 : 4, nslot = (dim == 3) ? 27 : 9, ft = dim - 1;
  std::vector<char> bnd[3];
  for (int t = 0; t < 3; ++t) bnd[t].assign(n_ent[t], 0);
  auto ent_id = [&](int64_t e, int type, int lidx) -> int64_t {
    if (type == 0) return EVp[e * nc + lidx];
    if (type == 1) return el_edge[e * nle + lidx];
    return el_face[e * 6 + lidx];
  };
  for (int64_t e = 0; e < nel; ++e)
    for (int tau = 0; tau < nslot; ++tau) {
      int type, lidx;
      slot_entity(dim, tau, type, lidx);
      if (type != ft) continue;
      const int64_t id = ent_id(e, type, lidx);
      if (inc_off[type][id + 1] - inc_off[type][id] != 1) continue;  // shared facet: interior
      const int cls[3] = {tau % 3, (tau / 3) % 3, tau / 9};
      int n = 0;
      while (cls[n] == 1) ++n;  // the facet's normal axis (its one non-interior class)
      for (int t2 = 0; t2 < nslot; ++t2) {
        const int c2[3] = {t2 % 3, (t2 / 3) % 3, t2 / 9};
        if (c2[n] != cls[n]) continue;  // not on this facet
        int ty2, l2;
        slot_entity(dim, t2, ty2, l2);
        if (ty2 < 3) bnd[ty2][ent_id(e, ty2, l2)] = 1;
      }
    }
  for (int t = 0; t < 3; ++t) {
    if (nd[t] == 0) continue;
    for (int64_t id = 0; id < n_ent[t]; ++id) {
      if (!bnd[t][id]) continue;
      const int64_t g = S.base[t][id];
      if (g < S.row_begin || g >= S.row_begin + S.n_local) continue;
      for (int64_t k = 0; k < nd[t]; ++k) out.push_back((int32_t)(g - S.row_begin + k));
    }
  }
  std::sort(out.begin(), out.end());
}

ElemTopo HostPlan::topo_of(int64_t e) const {
  const int nc = 1 << dim, nle = (dim == 3) ? 12 : 4;
  const int nslot = (dim == 3) ? 27 : 9;
  auto owner = [&](int type, int64_t id) -> int {
    if (type == 3) return elem_rank[id];
    return elem_rank[inc_el[type][inc_off[type][id]]];
  };
  ElemTopo T;
  for (int tau = 0; tau < 27; ++tau) {
    T.ent[tau] = -1;
    T.orient[tau] = 0;
    T.val[tau] = 0;
    T.flags[tau] = 0;
  }
  for (int i = 0; i < 3; ++i) T.pad[i] = 0;
  for (int tau = 0; tau < nslot; ++tau) {
    int type, lidx;
    slot_entity(dim, tau, type, lidx);
    uint8_t orient = 0;
    int64_t id;
    if (type == 0) id = EVp[e * nc + lidx];
    else if (type == 1) { id = el_edge[e * nle + lidx]; orient = el_edge_rev[e * nle + lidx]; }
    else if (type == 2) { id = el_face[e * 6 + lidx]; orient = el_face_code[e * 6 + lidx]; }
    else id = e;
    T.ent[tau] = (int32_t)id;
    T.orient[tau] = orient;
    if (type == 3) {
      T.val[tau] = 1;
      T.flags[tau] = TF_MIN | (elem_rank[e] == rank ? TF_OWNED : 0);
    } else {
      const int64_t k0 = inc_off[type][id], k1 = inc_off[type][id + 1];
      T.val[tau] = (uint8_t)std::min<int64_t>(k1 - k0, 255);
      T.flags[tau] = (inc_el[type][k0] == e ? TF_MIN : 0) | (owner(type, id) == rank ? TF_OWNED : 0);
    }
  }
  return T;
}

void HostPlan::build(const PlanInput &in) {
  dim = in.dim;
  p = in.p;
  rank = in.rank;
  nranks = in.nranks;
  nv = in.n_vert;
  nel = in.n_elem;
  const int nc = 1 << dim, nle = (dim == 3) ? 12 : 4, nlf = (dim == 3) ? 6 : 0;
  const int nslot = (dim == 3) ? 27 : 9;
  if (nv >= (int64_t(1) << 31) || nel >= (int64_t(1) << 31)) throw std::invalid_argument("mesh too large");
  erb.resize(nranks + 1);
  if (in.elem_rank_begin) {
    for (int r = 0; r <= nranks; ++r) erb[r] = in.elem_rank_begin[r];
  } else {
    if (nranks != 1) throw std::invalid_argument("elem_rank_begin required when nranks > 1");
    erb[0] = 0;
    erb[1] = nel;
  }
  if (erb[0] != 0 || erb[nranks] != nel) throw std::invalid_argument("elem_rank_begin must span [0, n_elem]");
  for (int r = 0; r < nranks; ++r)
    if (erb[r + 1] < erb[r]) throw std::invalid_argument("elem_rank_begin not monotone");
  elem_begin = erb[rank];
  nel_local = erb[rank + 1] - erb[rank];
  elem_rank.resize(nel);
  for (int r = 0; r < nranks; ++r)
    for (int64_t e = erb[r]; e < erb[r + 1]; ++e) elem_rank[e] = r;
  const int64_t *EV = in.elem_vert;
  for (int64_t i = 0; i < nel * nc; ++i)
    if (EV[i] < 0 || EV[i] >= nv) throw std::invalid_argument("vertex index out of range");

  // ---- coarse edges -------------------------------------------------------------------------
  {
    std::vector<uint64_t> keys(nel * nle);
    for (int64_t e = 0; e < nel; ++e)
      for (int le = 0; le < nle; ++le) {
        int t, h;
        edge_ends(dim, le, t, h);
        uint64_t a = EV[e * nc + t], b = EV[e * nc + h];
        if (a == b) throw std::invalid_argument("degenerate edge");
        keys[e * nle + le] = std::min(a, b) * (uint64_t)nv + std::max(a, b);
      }
    std::vector<uint64_t> uk(keys);
    std::sort(uk.begin(), uk.end());
    uk.erase(std::unique(uk.begin(), uk.end()), uk.end());
    ne = (int64_t)uk.size();
    el_edge.resize(nel * nle);
    el_edge_rev.resize(nel * nle);
    for (int64_t e = 0; e < nel; ++e)
      for (int le = 0; le < nle; ++le) {
        el_edge[e * nle + le] = (int32_t)(std::lower_bound(uk.begin(), uk.end(), keys[e * nle + le]) - uk.begin());
        int t, h;
        edge_ends(dim, le, t, h);
        el_edge_rev[e * nle + le] = EV[e * nc + t] > EV[e * nc + h];
      }
  }
  // ---- coarse faces (3D) + frames (App. A.2/A.4) ------------------------------------------------
  nf = 0;
  if (dim == 3) {
    std::vector<Key2> keys(nel * 6);
    for (int64_t e = 0; e < nel; ++e)
      for (int lf = 0; lf < 6; ++lf) {
        int fc[2][2];
        face_quad(lf, fc);
        uint64_t v[4] = {(uint64_t)EV[e * 8 + fc[0][0]], (uint64_t)EV[e * 8 + fc[1][0]], (uint64_t)EV[e * 8 + fc[0][1]],
                         (uint64_t)EV[e * 8 + fc[1][1]]};
        std::sort(v, v + 4);
        keys[e * 6 + lf] = Key2{v[0] * (uint64_t)nv + v[1], v[2] * (uint64_t)nv + v[3]};
      }
    std::vector<Key2> uk(keys);
    std::sort(uk.begin(), uk.end());
    uk.erase(std::unique(uk.begin(), uk.end()), uk.end());
    nf = (int64_t)uk.size();
    el_face.resize(nel * 6);
    el_face_code.resize(nel * 6);
    for (int64_t e = 0; e < nel; ++e)
      for (int lf = 0; lf < 6; ++lf) {
        el_face[e * 6 + lf] = (int32_t)(std::lower_bound(uk.begin(), uk.end(), keys[e * 6 + lf]) - uk.begin());
        int fc[2][2];
        face_quad(lf, fc);
        int a0 = 0, b0 = 0;
        int64_t best = EV[e * 8 + fc[0][0]];
        for (int a = 0; a < 2; ++a)
          for (int b = 0; b < 2; ++b)
            if (EV[e * 8 + fc[a][b]] < best) { best = EV[e * 8 + fc[a][b]]; a0 = a; b0 = b; }
        int64_t nu = EV[e * 8 + fc[1 - a0][b0]], nvv = EV[e * 8 + fc[a0][1 - b0]];
        int swap, s1neg, s2neg;
        if (nu < nvv) { swap = 0; s1neg = a0; s2neg = b0; }   // axis1 <-> u
        else { swap = 1; s1neg = b0; s2neg = a0; }             // axis1 <-> v
        el_face_code[e * 6 + lf] = (uint8_t)(swap | (s1neg << 1) | (s2neg << 2));
      }
  }
  // ---- incidence (elements per entity, ascending) ---------------------------------------------
  auto build_inc = [&](int64_t n_ent, int per, auto get, std::vector<int64_t> &off, std::vector<int32_t> &lst) {
    off.assign(n_ent + 1, 0);
    for (int64_t e = 0; e < nel; ++e)
      for (int i = 0; i < per; ++i) off[get(e, i) + 1]++;
    for (int64_t k = 0; k < n_ent; ++k) off[k + 1] += off[k];
    lst.resize(off[n_ent]);
    std::vector<int64_t> fill(off.begin(), off.end() - 1);
    for (int64_t e = 0; e < nel; ++e)
      for (int i = 0; i < per; ++i) lst[fill[get(e, i)]++] = (int32_t)e;
  };
  build_inc(nv, nc, [&](int64_t e, int i) { return EV[e * nc + i]; }, inc_off[0], inc_el[0]);
  build_inc(ne, nle, [&](int64_t e, int i) { return (int64_t)el_edge[e * nle + i]; }, inc_off[1], inc_el[1]);
  if (dim == 3) build_inc(nf, 6, [&](int64_t e, int i) { return (int64_t)el_face[e * 6 + i]; }, inc_off[2], inc_el[2]);
  else inc_off[2].assign(1, 0);
  for (int t = 0; t < 3; ++t)
    for (size_t k = 0; k + 1 < inc_off[t].size(); ++k)
      if (inc_off[t][k + 1] - inc_off[t][k] > MAX_VALENCE)
        throw std::invalid_argument("entity valence exceeds 16 (unsupported)");
  n_ent[0] = nv;
  n_ent[1] = ne;
  n_ent[2] = nf;
  n_ent[3] = nel;
  auto owner = [&](int type, int64_t id) -> int {
    if (type == 3) return elem_rank[id];
    return elem_rank[inc_el[type][inc_off[type][id]]];
  };

  // ---- ghost elements: elements of other ranks that contain an entity owned by this rank ---------
  {
    std::vector<char> is_ghost(nel, 0);
    for (int t = 0; t < 3; ++t)
      for (int64_t id = 0; id + 1 < (int64_t)inc_off[t].size(); ++id) {
        if (owner(t, id) != rank) continue;
        for (int64_t k = inc_off[t][id]; k < inc_off[t][id + 1]; ++k) {
          int64_t e = inc_el[t][k];
          if (elem_rank[e] != rank) is_ghost[e] = 1;
        }
      }
    ghost.clear();
    for (int64_t e = 0; e < nel; ++e)
      if (is_ghost[e]) ghost.push_back(e);
  }
  // ---- topology records (local elements, then ghosts) -------------------------------------------
  EVp = EV;
  const int64_t ntop = nel_local + (int64_t)ghost.size();
  topo.assign(ntop, ElemTopo{});
  for (int64_t i = 0; i < ntop; ++i) topo[i] = topo_of((i < nel_local) ? elem_begin + i : ghost[i - nel_local]);

  // ---- per space numbering, rows, shared-row plan -------------------------------------------------
  for (int s = 0; s < 3; ++s) {
    SpacePlan &S = sp[s];
    S = SpacePlan{};
    S.space = s;
    S.valid = (dim == 3) || (s == SP_H1);
    if (!S.valid) continue;
    S.ndpe = ndpe_of(dim, p, s);
    S.maxl = maxl_of(dim, s);
    int64_t nd[4];
    entity_ndofs(dim, p, s, nd);
    // per-owner totals in canonical entity order: vertices, edges, faces, interiors
    std::vector<int64_t> tot(nranks, 0);
    for (int t = 0; t < 4; ++t) {
      if (nd[t] == 0) continue;
      for (int64_t id = 0; id < n_ent[t]; ++id) tot[owner(t, id)] += nd[t];
    }
    S.rank_off.assign(nranks + 1, 0);
    for (int r = 0; r < nranks; ++r) S.rank_off[r + 1] = S.rank_off[r] + tot[r];
    S.n_global = S.rank_off[nranks];
    if (S.n_global >= (int64_t(1) << 31) - 1) throw std::invalid_argument("n_global >= 2^31");
    S.row_begin = S.rank_off[rank];
    S.n_local = S.rank_off[rank + 1] - S.rank_off[rank];
    std::vector<int64_t> cur(S.rank_off.begin(), S.rank_off.end() - 1);
    for (int t = 0; t < 4; ++t) {
      S.base[t].assign(n_ent[t], -1);
      if (nd[t] == 0) continue;
      for (int64_t id = 0; id < n_ent[t]; ++id) {
        int o = owner(t, id);
        S.base[t][id] = (int32_t)cur[o];
        cur[o] += nd[t];
      }
    }
    // owned shared entities (OSE) in canonical order, with slots in element order
    std::vector<int64_t> recv_cnt(nranks, 0), send_cnt(nranks, 0);
    std::vector<std::vector<int64_t>> ose_of(3);  // entity id -> ose index (per type), -1
    int64_t local_recs = 0;
    struct Slot { int64_t ose; int peer; int64_t rel; };  // rel: relative record within region
    std::vector<Slot> slots;
    for (int t = 0; t < 3; ++t) {
      ose_of[t].assign(n_ent[t], -1);
      if (nd[t] == 0) continue;
      for (int64_t id = 0; id < n_ent[t]; ++id) {
        int64_t k0 = inc_off[t][id], k1 = inc_off[t][id + 1];
        if (owner(t, id) != rank || k1 - k0 < 2) continue;
        Ose o;
        o.gid_base = S.base[t][id];
        o.nrows = (int32_t)nd[t];
        o.k = (int32_t)(k1 - k0);
        o.slot_off = (int32_t)S.ose_slots.size();
        bool remote = false;
        int64_t oi = (int64_t)S.ose.size();
        for (int64_t k = k0; k < k1; ++k) {
          int64_t e = inc_el[t][k];
          int q = elem_rank[e];
          Slot sl;
          sl.ose = oi;
          sl.peer = q;
          if (q == rank) { sl.rel = local_recs; local_recs += nd[t]; }
          else { sl.rel = recv_cnt[q]; recv_cnt[q] += nd[t]; remote = true; }
          slots.push_back(sl);
          S.ose_slots.push_back(0);
          S.ose_elem.push_back((int32_t)e);
        }
        if (remote) S.defer.push_back((int32_t)oi);
        ose_of[t][id] = oi;
        S.ose.push_back(o);
      }
    }
    // send side: entities owned by other ranks touched by local elements
    // (canonical entity order, then local elements in order)
    std::vector<std::vector<int64_t>> send_rel(3);
    for (int t = 0; t < 3; ++t) {
      send_rel[t].clear();
      if (nd[t] == 0) continue;
      // map entity -> first send record of (entity, first local element); consecutive per element
      send_rel[t].assign(n_ent[t], -1);
      for (int64_t id = 0; id < n_ent[t]; ++id) {
        int o = owner(t, id);
        if (o == rank) continue;
        int64_t k0 = inc_off[t][id], k1 = inc_off[t][id + 1];
        bool touched = false;
        for (int64_t k = k0; k < k1; ++k) touched |= (elem_rank[inc_el[t][k]] == rank);
        if (!touched) continue;
        send_rel[t][id] = send_cnt[o];
        for (int64_t k = k0; k < k1; ++k)
          if (elem_rank[inc_el[t][k]] == rank) send_cnt[o] += nd[t];
      }
    }
    // region layout: [local][recv peer 0..][send peer 0..]
    S.recv_begin.assign(nranks, 0);
    S.recv_count.assign(nranks, 0);
    S.send_begin.assign(nranks, 0);
    S.send_count.assign(nranks, 0);
    int64_t off = local_recs;
    for (int q = 0; q < nranks; ++q) { S.recv_begin[q] = off; S.recv_count[q] = recv_cnt[q]; off += recv_cnt[q]; }
    for (int q = 0; q < nranks; ++q) { S.send_begin[q] = off; S.send_count[q] = send_cnt[q]; off += send_cnt[q]; }
    S.n_records = off;
    if (S.n_records >= (int64_t(1) << 31)) throw std::invalid_argument("scratch too large");
    for (size_t i = 0; i < slots.size(); ++i) {
      const Slot &sl = slots[i];
      S.ose_slots[i] = (int32_t)(sl.peer == rank ? sl.rel : S.recv_begin[sl.peer] + sl.rel);
    }
    // element space records (local elements only)
    S.esp.assign(nel_local, ElemSpace{});
    for (int64_t i = 0; i < nel_local; ++i) {
      int64_t e = elem_begin + i;
      ElemSpace &R = S.esp[i];
      for (int tau = 0; tau < 27; ++tau) { R.rec[tau] = -1; R.ose[tau] = -1; R.ebase[tau] = -1; R.sflags[tau] = 0; }
      for (int tau = 0; tau < nslot; ++tau) {
        int type, lidx;
        slot_entity(dim, tau, type, lidx);
        const int64_t id = topo[(size_t)i].ent[tau];
        R.ebase[tau] = S.base[type].empty() ? -1 : S.base[type][id];
        if (type == 3 || nd[type] == 0) continue;
        int64_t k0 = inc_off[type][id], k1 = inc_off[type][id + 1];
        if (k1 - k0 < 2) continue;  // exclusive rows: written directly
        R.sflags[tau] |= SF_SHARED;
        int o = owner(type, id);
        if (o == rank) {
          int64_t oi = ose_of[type][id];
          R.ose[tau] = (int32_t)oi;
          const Ose &O = S.ose[oi];
          for (int64_t k = k0; k < k1; ++k)
            if (inc_el[type][k] == e) R.rec[tau] = S.ose_slots[O.slot_off + (k - k0)];
          bool remote = false;
          for (int64_t k = k0; k < k1; ++k) remote |= (elem_rank[inc_el[type][k]] != rank);
          if (remote) R.sflags[tau] |= SF_DEFER;
        } else {
          R.sflags[tau] |= SF_SEND;
          int64_t rel = send_rel[type][id];
          for (int64_t k = k0; k < k1; ++k) {
            int64_t ek = inc_el[type][k];
            if (elem_rank[ek] != rank) continue;
            if (ek == e) break;
            rel += nd[type];
          }
          R.rec[tau] = (int32_t)(S.send_begin[o] + rel);
        }
      }
    }
  }
}

// ---- Gauss-Lobatto points (for elem_nodes == NULL): Newton on P_p'(x) in long double ------------
static void gll01(int p, std::vector<double> &s) {
  s.resize(p + 1);
  for (int i = 0; i <= p; ++i) {
    long double x = -std::cos(3.14159265358979323846264338327950288L * i / p);
    if (i > 0 && i < p) {
      for (int it = 0; it < 60; ++it) {
        long double p0 = 1, p1 = x;
        for (int k = 2; k <= p; ++k) {
          long double p2 = ((2.0L * k - 1) * x * p1 - (k - 1.0L) * p0) / k;
          p0 = p1;
          p1 = p2;
        }
        long double dP = p * (x * p1 - p0) / (x * x - 1);
        long double d2P = (2 * x * dP - p * (p + 1.0L) * p1) / (1 - x * x);
        long double dx = dP / d2P;
        x -= dx;
        if (std::fabs((double)dx) < 1e-30) break;
      }
    }
    s[i] = (double)((x + 1) / 2);
  }
}

void interpolate_evector(int dim, int p, const double *vert, const int64_t *ev, int64_t e0, int64_t n,
                         std::vector<double> &X) {
  std::vector<double> s;
  gll01(p, s);
  int np = (dim == 3) ? (p + 1) * (p + 1) * (p + 1) : (p + 1) * (p + 1);
  int nc = 1 << dim;
  X.assign(n * dim * np, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t *c = ev + (e0 + i) * nc;
    for (int l = 0; l < np; ++l) {
      int ix = l % (p + 1), iy = (l / (p + 1)) % (p + 1), iz = (dim == 3) ? l / ((p + 1) * (p + 1)) : 0;
      double w[2][3] = {{1 - s[ix], 1 - s[iy], 1 - s[iz]}, {s[ix], s[iy], s[iz]}};
      for (int q = 0; q < nc; ++q) {
        double wt = w[q & 1][0] * w[(q >> 1) & 1][1] * (dim == 3 ? w[(q >> 2) & 1][2] : 1.0);
        for (int d = 0; d < dim; ++d) X[(i * dim + d) * np + l] += wt * vert[c[q] * dim + d];
      }
    }
  }
}

}  // namespace lorb
