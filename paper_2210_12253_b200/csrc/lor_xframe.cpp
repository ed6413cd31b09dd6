// lor_xframe.cpp -- host setup of the extended-frame H1 fill path (lor_xframe.h).
//
// For every local element e: the elements of its 3x3x3 coarse neighbourhood and, for each, the map
// from e's extended lattice frame to the neighbour's local lattice.  The neighbourhood is walked by
// face adjacency only (face incidence of the plan); a mesh qualifies when every walk agrees:
//   * a diagonal neighbour reached through different face neighbours is the same element with
//     the same frame map, and it exists exactly when all its face components exist;
//   * the coarse vertices of the block ({-1,0,1,2}^3 in e's frame) carry one vertex id each and
//     distinct positions carry distinct ids.
// Then the LOR cells around every row e owns are exactly the cells of a box [clo, chi]^3 of the
// extended frame, which is what k_xh1 computes.
#include "lor_xframe.h"

#include <algorithm>
#include <cstring>
#include <map>

#include "lor_plan.h"

namespace lorb {

namespace {

struct XMap {
  int64_t el = -1;   // global element id
  int P[8][3];       // extended coarse position of each local corner (a + 2b + 4c)
};

bool same_map(const XMap &a, const XMap &b) {
  if (a.el != b.el) return false;
  for (int v = 0; v < 8; ++v)
    for (int k = 0; k < 3; ++k)
      if (a.P[v][k] != b.P[v][k]) return false;
  return true;
}

// local axis of f running along extended axis k (and its sign), -1 if none
int axis_along(const XMap &f, int k, int &sgn) {
  for (int a = 0; a < 3; ++a) {
    const int d = f.P[1 << a][k] - f.P[0][k];
    if (d != 0) { sgn = d; return a; }
  }
  return -1;
}

// the map is an axis-aligned unit cube: P[v] = P[0] + sum_a v_a * (signed unit vector of axis a)
bool is_unit_cube(const XMap &f) {
  int used = 0;
  for (int a = 0; a < 3; ++a) {
    int nz = 0, k0 = -1;
    for (int k = 0; k < 3; ++k) {
      const int d = f.P[1 << a][k] - f.P[0][k];
      if (d != 0) { ++nz; k0 = k; if (d != 1 && d != -1) return false; }
    }
    if (nz != 1 || (used >> k0) & 1) return false;
    used |= 1 << k0;
  }
  for (int v = 0; v < 8; ++v)
    for (int k = 0; k < 3; ++k) {
      int x = f.P[0][k];
      for (int a = 0; a < 3; ++a)
        if ((v >> a) & 1) x += f.P[1 << a][k] - f.P[0][k];
      if (x != f.P[v][k]) return false;
    }
  return true;
}

}  // namespace

// non-local elements sharing a coarse vertex with a local element (sorted): the ghost layer of the
// extended frame on several ranks (every element of a 3x3x3 neighbourhood shares a vertex with its
// centre); the same rule applied to another rank gives the elements this rank sends it
std::vector<int64_t> xframe_ghosts(const HostPlan &plan, int rank) {
  const int64_t *EV = plan.EVp;
  std::vector<char> mark((size_t)plan.nel, 0);
  for (int64_t e = plan.erb[rank]; e < plan.erb[rank + 1]; ++e)
    for (int v = 0; v < 8; ++v) {
      const int64_t vid = EV[e * 8 + v];
      for (int64_t k = plan.inc_off[0][vid]; k < plan.inc_off[0][vid + 1]; ++k) {
        const int64_t o = plan.inc_el[0][k];
        if (plan.elem_rank[o] != rank) mark[(size_t)o] = 1;
      }
    }
  std::vector<int64_t> g;
  for (int64_t e = 0; e < plan.nel; ++e)
    if (mark[(size_t)e]) g.push_back(e);
  return g;
}

bool xframe_build(const HostPlan &plan, const int64_t *EV, std::vector<XElem> &out, int cmax[3], std::string *why,
                  std::vector<int64_t> *xghost) {
  auto no = [&](const char *m) {
    if (why) *why = m;
    return false;
  };
  if (plan.dim != 3) return no("dim != 3");
  if (!xghost && plan.nranks != 1) return no("nranks > 1 without a ghost layer");
  std::vector<int64_t> gl;
  if (plan.nranks > 1) gl = xframe_ghosts(plan, plan.rank);
  if (xghost) *xghost = gl;
  const int p = plan.p;
  const int64_t n = plan.nel_local;
  out.assign((size_t)n, XElem{});
  cmax[0] = cmax[1] = cmax[2] = 0;
  // face neighbour of f across the local face that faces extended direction dir * e_k
  auto face_nb = [&](const XMap &f, int k, int dir, XMap &g, bool &bad) -> bool {
    int sgn = 0;
    const int a = axis_along(f, k, sgn);
    if (a < 0) { bad = true; return false; }
    const int side = (dir * sgn > 0) ? 1 : 0;
    const int lf = 2 * a + side;
    const int32_t fid = plan.el_face[f.el * 6 + lf];
    const int64_t k0 = plan.inc_off[2][fid], k1 = plan.inc_off[2][fid + 1];
    if (k1 - k0 == 1) return false;  // boundary face
    if (k1 - k0 != 2) { bad = true; return false; }
    const int64_t o = plan.inc_el[2][k0] == f.el ? plan.inc_el[2][k0 + 1] : plan.inc_el[2][k0];
    int lf2 = -1;
    for (int q = 0; q < 6; ++q)
      if (plan.el_face[o * 6 + q] == fid) lf2 = q;
    if (lf2 < 0) { bad = true; return false; }
    const int n2 = lf2 / 2, side2 = lf2 & 1;
    g.el = o;
    int found = 0;
    for (int v2 = 0; v2 < 8; ++v2) {
      if (((v2 >> n2) & 1) != side2) continue;
      int vf = -1;
      for (int v = 0; v < 8; ++v)
        if (((v >> a) & 1) == side && EV[f.el * 8 + v] == EV[o * 8 + v2]) vf = v;
      if (vf < 0) { bad = true; return false; }
      const int vin = vf ^ (1 << a);
      const int v2o = v2 ^ (1 << n2);
      for (int kk = 0; kk < 3; ++kk) {
        g.P[v2][kk] = f.P[vf][kk];
        g.P[v2o][kk] = 2 * f.P[vf][kk] - f.P[vin][kk];
      }
      ++found;
    }
    if (found != 4 || !is_unit_cube(g)) { bad = true; return false; }
    return true;
  };
  for (int64_t le = 0; le < n; ++le) {
    const int64_t e = plan.elem_begin + le;
    XMap m[27];
    bool ex[27];
    for (int i = 0; i < 27; ++i) ex[i] = false;
    m[13].el = e;
    for (int v = 0; v < 8; ++v)
      for (int k = 0; k < 3; ++k) m[13].P[v][k] = (v >> k) & 1;
    ex[13] = true;
    // walk by number of non-zero delta components
    for (int nzc = 1; nzc <= 3; ++nzc)
      for (int i = 0; i < 27; ++i) {
        const int d[3] = {i % 3 - 1, (i / 3) % 3 - 1, i / 9 - 1};
        if ((d[0] != 0) + (d[1] != 0) + (d[2] != 0) != nzc) continue;
        bool expect = true;  // exists iff every face component exists
        if (nzc > 1)
          for (int k = 0; k < 3; ++k)
            if (d[k] != 0) {
            const int fi = 13 + (k == 0 ? d[0] : k == 1 ? 3 * d[1] : 9 * d[2]);
              expect = expect && ex[fi];
            }
        bool first = true;
        for (int k = 0; k < 3; ++k) {
          if (d[k] == 0) continue;
          const int from = i - (k == 0 ? d[0] : k == 1 ? 3 * d[1] : 9 * d[2]);
          if (!ex[from]) continue;
          XMap g;
          bool bad = false;
          const bool got = face_nb(m[from], k, d[k], g, bad);
          if (bad) return no("non-conforming face adjacency");
          if (nzc == 1) expect = got;
          if (got != expect) return no("irregular neighbourhood (edge/vertex valence)");
          if (!got) continue;
          if (first) { m[i] = g; first = false; }
          else if (!same_map(m[i], g)) return no("neighbourhood walks disagree");
        }
        ex[i] = expect && !first;
        if (expect && first) return no("irregular neighbourhood");
      }
    // coarse vertex ids of the block: consistent and injective
    {
      int64_t vid[64];
      for (int i = 0; i < 64; ++i) vid[i] = -1;
      for (int i = 0; i < 27; ++i) {
        if (!ex[i]) continue;
        for (int v = 0; v < 8; ++v) {
          const int q = (m[i].P[v][0] + 1) + 4 * (m[i].P[v][1] + 1) + 16 * (m[i].P[v][2] + 1);
          const int64_t id = EV[m[i].el * 8 + v];
          if (vid[q] >= 0 && vid[q] != id) return no("inconsistent vertex ids");
          vid[q] = id;
        }
      }
      std::map<int64_t, int> seen;
      for (int i = 0; i < 64; ++i)
        if (vid[i] >= 0 && seen[vid[i]]++) return no("vertex repeated in a neighbourhood");
    }
    XElem &X = out[(size_t)le];
    memset(&X, 0, sizeof(X));
    const ElemTopo &T = plan.topo[(size_t)le];
    // every coarse entity this element owns (minimal element, this rank), whether or not the space
    // has dofs on it (H1 has none on edges / faces / interiors at p = 1; ND / RT do): the cell box
    // must hold the cells around the rows of every space (lor_xv.cuh shares it)
    for (int tau = 0; tau < 27; ++tau)
      if ((T.flags[tau] & TF_MIN) && (T.flags[tau] & TF_OWNED)) X.own |= 1u << tau;
    for (int a = 0; a < 3; ++a) {
      bool lo = false, hi = false;
      for (int tau = 0; tau < 27; ++tau) {
        if (!((X.own >> tau) & 1)) continue;
        const int c = a == 0 ? tau % 3 : a == 1 ? (tau / 3) % 3 : tau / 9;
        lo = lo || c == 0;
        hi = hi || c == 2;
      }
      const int fm = 13 - (a == 0 ? 1 : a == 1 ? 3 : 9), fp = 13 + (a == 0 ? 1 : a == 1 ? 3 : 9);
      X.clo[a] = (int8_t)((lo && ex[fm]) ? -1 : 0);
      X.chi[a] = (int8_t)((hi && ex[fp]) ? p : p - 1);
      cmax[a] = std::max(cmax[a], X.chi[a] - X.clo[a] + 1);
      // owned-row bounding box along a (class 0 -> x = 0, 1 -> [1, p-1], 2 -> x = p)
      bool c1 = false;
      for (int tau = 0; tau < 27; ++tau)
        if ((X.own >> tau) & 1) c1 = c1 || (a == 0 ? tau % 3 : a == 1 ? (tau / 3) % 3 : tau / 9) == 1;
      X.olo[a] = (int8_t)(lo ? 0 : (c1 ? 1 : p));
      X.ohi[a] = (int8_t)(hi ? p : (c1 ? p - 1 : 0));
    }
    for (int i = 0; i < 27; ++i) {
      X.nbr[i].el = -1;
      X.nbr[i].code = 0;
      if (!ex[i] || i == 13) continue;
      const XMap &g = m[i];
      uint32_t code = 0;
      for (int a = 0; a < 3; ++a) {
        int k = -1, s = 0;
        for (int kk = 0; kk < 3; ++kk) {
          const int dd = g.P[1 << a][kk] - g.P[0][kk];
          if (dd) { k = kk; s = dd; }
        }
        code |= (uint32_t)k << (2 * a);
        if (s < 0) code |= 1u << (6 + a);
      }
      for (int k = 0; k < 3; ++k) code |= (uint32_t)(g.P[0][k] + 1) << (9 + 2 * k);
      if (g.el >= plan.elem_begin && g.el < plan.elem_begin + n) {
        X.nbr[i].el = (int32_t)(g.el - plan.elem_begin);
      } else {  // ghost layer: indices after the local elements
        const auto it = std::lower_bound(gl.begin(), gl.end(), g.el);
        if (it == gl.end() || *it != g.el) return no("neighbour outside the ghost layer");
        X.nbr[i].el = (int32_t)(n + (it - gl.begin()));
      }
      X.nbr[i].code = code;
    }
  }
  return true;
}

}  // namespace lorb
