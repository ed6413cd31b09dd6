"""Dense HIGH-ORDER matrices on tiny meshes -- TEST INFRASTRUCTURE ONLY (method-level pin).

Used only by the spectral-equivalence self-check of the oracle: kappa(A_LOR^{-1} A_HO) must stay
bounded as p grows ("A_{V_h} and A_{V_p} are spectrally equivalent, independent
of p"; l.138 for mass; l.148 for the interpolation-histopolation ND/RT bases).

H1: GLL-Lagrange tensor basis ("Lagrange interpolating polynomials defined at the
Cartesian product of the Gauss--Lobatto quadrature points"), integrated with a q = p+2 point
Gauss rule on the (trilinear) element map, assembled with the oracle's own H1 dof map.
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
