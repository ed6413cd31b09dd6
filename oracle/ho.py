"""Dense HIGH-ORDER matrices on tiny meshes -- TEST INFRASTRUCTURE ONLY (method-level pin).

Used only by the spectral-equivalence self-check of the oracle: kappa(A_LOR^{-1} A_HO) must stay
bounded as p grows ("A_{V_h} and A_{V_p} are spectrally equivalent, independent
of p"; l.138 for mass; l.148 for the interpolation-histopolation ND/RT bases).

H1: GLL-Lagrange tensor basis ("Lagrange interpolating polynomials defined at the
Cartesian product of the Gauss--Lobatto quadrature points"), integrated with a q = p+2 point
Gauss rule on the (trilinear) element map, assembled with the oracle's own H1 dof map.
ND / RT (3D): the interpolation--histopolation bases (l.142-150, SPEC closed form of the
histopolants, reading P-13), covariant / contravariant Piola maps, same quadrature, assembled with
the oracle's ND / RT dof maps and signs (ho_vector_matrix).

Pins (tests/test_oracle_pins.py): histopolation delta property and derivative identity; p = 1
equals the textbook lowest-order matrices (l.150); K_ND G = 0 and K_RT C = 0 (commuting de Rham
sequence); kappa(A_LOR^-1 A_HO) bounded for p = 1..8 (2D H1), 1..5 (3D H1), 1..4 (3D ND, RT).
"""
from __future__ import annotations

import numpy as np


def gauss(q):
    x, w = np.polynomial.legendre.leggauss(q)
    return (x + 1) / 2, w / 2  # on [0,1]


def lagrange_1d(nodes, x):
    """B[i, j] = l_j(x_i), D[i, j] = l_j'(x_i) for Lagrange polynomials on `nodes`."""
    n = len(nodes)
    B = np.ones((len(x), n))
    D = np.zeros((len(x), n))
    for j in range(n):
        for m in range(n):
            if m == j:
                continue
            B[:, j] *= (x - nodes[m]) / (nodes[j] - nodes[m])
        for k in range(n):
            if k == j:
                continue
            term = np.ones(len(x)) / (nodes[j] - nodes[k])
            for m in range(n):
                if m == j or m == k:
                    continue
                term *= (x - nodes[m]) / (nodes[j] - nodes[m])
            D[:, j] += term
    return B, D


def ho_h1_matrix(mesh, gll_nodes_01, h1_map, n, alpha=1.0, beta=1.0, q=None):
    """Dense degree-p H1 stiffness(alpha) + mass(beta) on the mesh's (bi/tri)linear element maps."""
    dim, p = mesh.dim, mesh.p
    q = q or p + 2
    xq, wq = gauss(q)
    B, D = lagrange_1d(np.asarray(gll_nodes_01), xq)   # [q, p+1]
    A = np.zeros((n, n))
    corners = mesh.vert[mesh.elem]  # [nel, 2^d, d]
    if dim == 2:
        # basis index l = i + (p+1) j ; point (a, b)
        phi = np.einsum("ai,bj->abji", B, B).reshape(q, q, -1)
        gx = np.einsum("ai,bj->abji", D, B).reshape(q, q, -1)
        gy = np.einsum("ai,bj->abji", B, D).reshape(q, q, -1)
        for e in range(mesh.nel):
            C = corners[e]
            Ae = np.zeros(((p + 1) ** 2,) * 2)
            for a in range(q):
                for b in range(q):
                    x = np.array([xq[a], xq[b]])
                    J = np.zeros((2, 2))
                    for v in range(4):
                        bits = [(v >> d) & 1 for d in range(2)]
                        f = [x[d] if bits[d] else 1 - x[d] for d in range(2)]
                        df = [1.0 if bits[d] else -1.0 for d in range(2)]
                        J[:, 0] += C[v] * df[0] * f[1]
                        J[:, 1] += C[v] * f[0] * df[1]
                    det = np.linalg.det(J)
                    Ji = np.linalg.inv(J)
                    G = np.stack([gx[a, b], gy[a, b]], axis=0)  # [2, nb] reference gradients
                    Gp = Ji.T @ G
                    w = wq[a] * wq[b] * det
                    Ae += w * (alpha * Gp.T @ Gp + beta * np.outer(phi[a, b], phi[a, b]))
            idx = h1_map[e]
            A[np.ix_(idx, idx)] += Ae
        return A
    phi = np.einsum("ai,bj,ck->abckji", B, B, B).reshape(q, q, q, -1)
    g0 = np.einsum("ai,bj,ck->abckji", D, B, B).reshape(q, q, q, -1)
    g1 = np.einsum("ai,bj,ck->abckji", B, D, B).reshape(q, q, q, -1)
    g2 = np.einsum("ai,bj,ck->abckji", B, B, D).reshape(q, q, q, -1)
    for e in range(mesh.nel):
        C = corners[e]
        Ae = np.zeros(((p + 1) ** 3,) * 2)
        for a in range(q):
            for b in range(q):
                for c in range(q):
                    x = np.array([xq[a], xq[b], xq[c]])
                    J = np.zeros((3, 3))
                    for v in range(8):
                        bits = [(v >> d) & 1 for d in range(3)]
                        f = [x[d] if bits[d] else 1 - x[d] for d in range(3)]
                        df = [1.0 if bits[d] else -1.0 for d in range(3)]
                        J[:, 0] += C[v] * df[0] * f[1] * f[2]
                        J[:, 1] += C[v] * f[0] * df[1] * f[2]
                        J[:, 2] += C[v] * f[0] * f[1] * df[2]
                    det = np.linalg.det(J)
                    Ji = np.linalg.inv(J)
                    G = np.stack([g0[a, b, c], g1[a, b, c], g2[a, b, c]], axis=0)
                    Gp = Ji.T @ G
                    w = wq[a] * wq[b] * wq[c] * det
                    Ae += w * (alpha * Gp.T @ Gp + beta * np.outer(phi[a, b, c], phi[a, b, c]))
        idx = h1_map[e]
        A[np.ix_(idx, idx)] += Ae
    return A


# ------------------------------------------------------------------------------------------------
# Interpolation--histopolation H(curl) / H(div) bases (SPEC histopolation
# closed form h_j = -sum_{k<j} l'_k, reading P-13).  On [0,1]: nodes s_0..s_p (GLL), l_k the
# degree-p Lagrange polynomials, h_j (j = 1..p) the degree-(p-1) histopolants with
# int_{s_{i-1}}^{s_i} h_j = delta_ij.  Reference ND functions (edge along axis a, lattice x):
#   x-edges: e_x h_{i+1}(xi) l_j(eta) l_k(zeta), local index nd_lidx(a=0, (i, j, k)), and cyclic;
# reference RT functions (face normal a):
#   x-faces: e_x l_i(xi) h_{j+1}(eta) h_{k+1}(zeta), local index rt_lidx(a=0, (i, j, k)).
# Their degrees of freedom are tangential integrals over sub-edges / fluxes through sub-faces of
# the Gauss-Lobatto lattice: the same functionals as the lowest-order LOR Nedelec / Raviart-Thomas
# dofs (covariant / contravariant Piola preserve them), so the HO and LOR matrices share the
# oracle's numbering and signs, and "the lowest-order case ... reduces exactly to the standard
# lowest-order Nedelec and Raviart-Thomas elements" (l.150).
# ------------------------------------------------------------------------------------------------
def histopolation_1d(nodes, x):
    """H[i, j-1] = h_j(x_i), j = 1..p, h_j = -sum_{k<j} l_k' (SPEC closed form)."""
    _, D = lagrange_1d(nodes, x)
    return -np.cumsum(D, axis=1)[:, :-1]


def _nd_index(p, a, x):
    ext = [p if b == a else p + 1 for b in range(3)]
    return a * p * (p + 1) * (p + 1) + x[0] + ext[0] * (x[1] + ext[1] * x[2])


def _rt_index(p, a, x):
    ext = [p + 1 if b == a else p for b in range(3)]
    return a * (p + 1) * p * p + x[0] + ext[0] * (x[1] + ext[1] * x[2])


def _ref_vector_basis(space, p, xq):
    """values [Q, n, 3] and curl (ND) [Q, n, 3] / div (RT) [Q, n] at the tensor points xq^3."""
    s = None
    B, D = lagrange_1d(np.asarray(_nodes_cache[p]), xq)   # l_k, l_k'
    H = histopolation_1d(np.asarray(_nodes_cache[p]), xq)  # h_j
    _, Dh = _hist_deriv(p, xq)
    q = len(xq)
    n = 3 * p * (p + 1) ** 2 if space == "nd" else 3 * p * p * (p + 1)
    val = np.zeros((q, q, q, n, 3))
    der = np.zeros((q, q, q, n, 3)) if space == "nd" else np.zeros((q, q, q, n))
    for a in range(3):
        ext = [(p if b == a else p + 1) if space == "nd" else (p + 1 if b == a else p) for b in range(3)]
        for x2 in range(ext[2]):
            for x1 in range(ext[1]):
                for x0 in range(ext[0]):
                    x = (x0, x1, x2)
                    f, df = [], []
                    for b in range(3):
                        hist = (b == a) if space == "nd" else (b != a)
                        if hist:
                            f.append(H[:, x[b]])
                            df.append(Dh[:, x[b]])
                        else:
                            f.append(B[:, x[b]])
                            df.append(D[:, x[b]])
                    F = np.einsum("a,b,c->abc", f[0], f[1], f[2])
                    gF = [np.einsum("a,b,c->abc", df[0], f[1], f[2]), np.einsum("a,b,c->abc", f[0], df[1], f[2]),
                          np.einsum("a,b,c->abc", f[0], f[1], df[2])]
                    if space == "nd":
                        i = _nd_index(p, a, x)
                        val[:, :, :, i, a] = F
                        # curl(e_a F) = grad F x e_a
                        ea = np.zeros(3)
                        ea[a] = 1.0
                        g = np.stack(gF, axis=-1)
                        der[:, :, :, i, :] = np.cross(g, ea)
                    else:
                        i = _rt_index(p, a, x)
                        val[:, :, :, i, a] = F
                        der[:, :, :, i] = gF[a]
    # point index Q = xi + q eta + q^2 zeta  (array axes were (xi, eta, zeta))
    val = val.transpose(2, 1, 0, 3, 4).reshape(q ** 3, n, 3)
    der = der.transpose(2, 1, 0, 3, 4).reshape(q ** 3, n, 3) if space == "nd" else \
        der.transpose(2, 1, 0, 3).reshape(q ** 3, n)
    return val, der


_nodes_cache = {}


def _hist_deriv(p, x):
    """h_j and h_j' at x: h_j' = -sum_{k<j} l_k'' (second derivatives by the product rule)."""
    nodes = np.asarray(_nodes_cache[p])
    n = len(nodes)
    D2 = np.zeros((len(x), n))
    for j in range(n):
        for k in range(n):
            if k == j:
                continue
            for m in range(n):
                if m == j or m == k:
                    continue
                term = np.ones(len(x)) / ((nodes[j] - nodes[k]) * (nodes[j] - nodes[m]))
                for r in range(n):
                    if r in (j, k, m):
                        continue
                    term *= (x - nodes[r]) / (nodes[j] - nodes[r])
                D2[:, j] += term
    H = histopolation_1d(nodes, x)
    return H, -np.cumsum(D2, axis=1)[:, :-1]


def ho_vector_matrix(mesh, space, gll_nodes_01, vmap, vsign, n, alpha=1.0, beta=1.0, q=None):
    """Dense degree-p interpolation--histopolation ND (alpha curl.curl + beta mass) or RT
    (alpha div.div + beta mass) matrix on the (tri)linear element maps, 3D, q = p+2 Gauss points,
    assembled with the oracle's ND/RT dof map and orientation signs."""
    assert mesh.dim == 3 and space in ("nd", "rt")
    p = mesh.p
    q = q or p + 2
    _nodes_cache[p] = np.asarray(gll_nodes_01, dtype=float)
    xq, wq = gauss(q)
    val, der = _ref_vector_basis(space, p, xq)
    W = np.einsum("a,b,c->cba", wq, wq, wq).reshape(-1)        # weight of point xi + q eta + q^2 zeta
    pts = np.stack(np.meshgrid(xq, xq, xq, indexing="ij"), axis=-1)  # [xi, eta, zeta, 3]
    pts = pts.transpose(2, 1, 0, 3).reshape(-1, 3)
    corners = mesh.vert[mesh.elem]
    A = np.zeros((n, n))
    for e in range(mesh.nel):
        C = corners[e]
        J = np.zeros((len(pts), 3, 3))
        for v in range(8):
            bits = [(v >> d) & 1 for d in range(3)]
            f = np.stack([pts[:, d] if bits[d] else 1 - pts[:, d] for d in range(3)], axis=1)
            df = [1.0 if bits[d] else -1.0 for d in range(3)]
            g = np.stack([df[0] * f[:, 1] * f[:, 2], f[:, 0] * df[1] * f[:, 2], f[:, 0] * f[:, 1] * df[2]], axis=1)
            J += np.einsum("k,qd->qkd", C[v], g)
        det = np.linalg.det(J)
        Ji = np.linalg.inv(J)
        if space == "nd":
            phi = np.einsum("qdk,qnd->qnk", Ji, val)                 # J^{-T} phi-hat
            cu = np.einsum("qkd,qnd->qnk", J, der) / det[:, None, None]  # J curl-hat / det
            wd = W * det
            Ae = alpha * np.einsum("q,qnk,qmk->nm", wd, cu, cu) + beta * np.einsum("q,qnk,qmk->nm", wd, phi, phi)
        else:
            phi = np.einsum("qkd,qnd->qnk", J, val) / det[:, None, None]  # J phi-hat / det
            dv = der / det[:, None]
            wd = W * det
            Ae = alpha * np.einsum("q,qn,qm->nm", wd, dv, dv) + beta * np.einsum("q,qnk,qmk->nm", wd, phi, phi)
        idx = vmap[e]
        sg = vsign[e].astype(float)
        A[np.ix_(idx, idx)] += Ae * np.outer(sg, sg)
    return A


def ho_vector_matrix_2d(mesh, space, gll_nodes_01, vmap, vsign, n, alpha=1.0, beta=1.0, q=None):
    """2D analogue of ho_vector_matrix (reading P-29 local order): ND family a = e_a h(t_a) l(t_o)
    with scalar curl, RT family a = e_a l(t_a) h(t_o) with divergence (the interpolation--histopolation
    bases of l.142-150 on quadrilaterals), covariant / contravariant Piola maps, q = p+2 Gauss points,
    assembled with the oracle's 2D ND / RT dof map and signs."""
    assert mesh.dim == 2 and space in ("nd", "rt")
    p = mesh.p
    q = q or p + 2
    nodes = np.asarray(gll_nodes_01, dtype=float)
    _nodes_cache[p] = nodes
    xq, wq = gauss(q)
    B, D = lagrange_1d(nodes, xq)
    H, Dh = _hist_deriv(p, xq)
    nb = 2 * p * (p + 1)
    val = np.zeros((q, q, nb, 2))   # [point along x, point along y, basis, component]
    der = np.zeros((q, q, nb))
    for a in range(2):
        o = 1 - a
        ext = [(p if b == a else p + 1) if space == "nd" else (p + 1 if b == a else p) for b in range(2)]
        for x1 in range(ext[1]):
            for x0 in range(ext[0]):
                x = (x0, x1)
                i = a * p * (p + 1) + x0 + ext[0] * x1
                # factor along each axis: histopolant along the edge (ND: a; RT: o), Lagrange across
                hist_axis = a if space == "nd" else o
                f = [H[:, x[b]] if b == hist_axis else B[:, x[b]] for b in range(2)]
                df = [Dh[:, x[b]] if b == hist_axis else D[:, x[b]] for b in range(2)]
                val[:, :, i, a] = np.outer(f[0], f[1])
                if space == "nd":  # curl (F e_a) = d(F)/dx for a = y, -d(F)/dy for a = x
                    der[:, :, i] = np.outer(df[0], f[1]) if a == 1 else -np.outer(f[0], df[1])
                else:              # div (F e_a) = dF/dx_a
                    der[:, :, i] = np.outer(df[0], f[1]) if a == 0 else np.outer(f[0], df[1])
    corners = mesh.vert[mesh.elem]
    A = np.zeros((n, n))
    for e in range(mesh.nel):
        C = corners[e]
        Ae = np.zeros((nb, nb))
        for ia in range(q):
            for ib in range(q):
                t = (xq[ia], xq[ib])
                J = np.zeros((2, 2))
                for v in range(4):
                    bits = [(v >> d) & 1 for d in range(2)]
                    f = [t[d] if bits[d] else 1 - t[d] for d in range(2)]
                    dfv = [1.0 if bits[d] else -1.0 for d in range(2)]
                    J[:, 0] += C[v] * dfv[0] * f[1]
                    J[:, 1] += C[v] * f[0] * dfv[1]
                det = np.linalg.det(J)
                ph = val[ia, ib]                                   # [nb, 2] reference
                phi = ph @ np.linalg.inv(J) if space == "nd" else ph @ J.T / det   # J^{-T} / J phi / det
                s = der[ia, ib] / det
                w = wq[ia] * wq[ib] * det
                Ae += w * (alpha * np.outer(s, s) + beta * phi @ phi.T)
        idx = vmap[e]
        sg = vsign[e].astype(float)
        A[np.ix_(idx, idx)] += Ae * np.outer(sg, sg)
    return A
