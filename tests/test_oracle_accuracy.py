"""Rounding accuracy of the oracle against an extended-precision (x87 long double, 64-bit
mantissa) evaluation of the same definition -- the evidence behind the parity tolerance P-10b
(tests/parity.py): on the hardest case met by the parity tests (Gauss-2 rule,
p = 8, jittered and orientation-scrambled cells, entries down to 1e-5 of their row max) every
oracle entry is within 1e-13 relative of the extended-precision value when it is >= 7e-3 of its
row max, and within 32 u * row max (half the P-10b bound) otherwise.  Two independently rounded
fp64 evaluations therefore differ by at most 64 u * row max.  This is not a correctness pin (the
formula is the textbook Q1 one restated); it measures rounding only."""
import numpy as np
import pytest

from paper_2210_12253_b200 import meshgen as mg

LD = np.longdouble
U = 2.0 ** -53


def h1_cell_ld(C, quad, alpha, beta):
    if quad == "gauss2":
        g = (LD(1) / 2 - LD(1) / (2 * np.sqrt(LD(3))), LD(1) / 2 + LD(1) / (2 * np.sqrt(LD(3))))
    else:
        g = (LD(0), LD(1))
    A = np.zeros((8, 8), dtype=LD)
    for q in range(8):
        t = [g[(q >> d) & 1] for d in range(3)]
        N = np.zeros(8, dtype=LD)
        G = np.zeros((8, 3), dtype=LD)
        for v in range(8):
            f = [t[a] if (v >> a) & 1 else 1 - t[a] for a in range(3)]
            df = [LD(1) if (v >> a) & 1 else LD(-1) for a in range(3)]
            N[v] = f[0] * f[1] * f[2]
            G[v] = [df[0] * f[1] * f[2], f[0] * df[1] * f[2], f[0] * f[1] * df[2]]
        J = C.T @ G  # J[k][d] = sum_v X_v[k] dN_v/dx_d
        c = np.zeros((3, 3), dtype=LD)
        for i in range(3):
            for j in range(3):
                i1, i2, j1, j2 = (i + 1) % 3, (i + 2) % 3, (j + 1) % 3, (j + 2) % 3
                c[i, j] = J[i1, j1] * J[i2, j2] - J[i1, j2] * J[i2, j1]
        det = J[0, 0] * c[0, 0] + J[0, 1] * c[0, 1] + J[0, 2] * c[0, 2]
        gp = G @ (c.T / det)
        A += (alpha * (gp @ gp.T) + beta * np.outer(N, N)) * det / 8
    return A


def row_ld(m, om, r, quad, alpha, beta):
    out = {}
    p, P = m.p, m.p + 1
    for e in range(m.nel):
        for l in np.flatnonzero(om[e] == r):
            x = (l % P, (l // P) % P, l // (P * P))
            for o in range(8):
                k = [x[a] - ((o >> a) & 1) for a in range(3)]
                if min(k) < 0 or max(k) >= p:
                    continue
                lid = [(k[0] + (v & 1)) + P * ((k[1] + ((v >> 1) & 1)) + P * (k[2] + (v >> 2))) for v in range(8)]
                C = np.array([[LD(m.X[e, d, li]) for d in range(3)] for li in lid], dtype=LD)
                A = h1_cell_ld(C, quad, LD(alpha), LD(beta))
                for v in range(8):
                    cc = int(om[e, lid[v]])
                    out[cc] = out.get(cc, LD(0)) + A[o, v]
    return out


@pytest.mark.parametrize("quad,p", [("gauss2", 8), ("gauss2", 5), ("vertex", 8)])
def test_oracle_rounding_vs_long_double(oracle_lib, quad, p):
    m = mg.box_mesh(3, (2, 2, 2), p, jitter=True, scramble=True)
    om, _ = oracle_lib.dof_map(m, "h1")
    ref = oracle_lib.assemble(m, "h1", quad, 1.3, 0.7)
    rows = [0, 2, 1 + (p + 1), int(om[0, (p + 1) ** 3 // 2]), ref.row_ptr.shape[0] - 2]
    worst_small = 0.0
    for r in rows:
        ex = row_ld(m, om, r, quad, 1.3, 0.7)
        s, e = ref.row_ptr[r], ref.row_ptr[r + 1]
        rm = float(np.abs(ref.val[s:e]).max())
        for c, v in zip(ref.col[s:e], ref.val[s:e]):
            err = float(abs(LD(v) - ex[int(c)]))
            if abs(v) >= 64 * U / 1e-12 * rm:
                assert err <= 1e-13 * abs(v), (r, c, v, float(ex[int(c)]))
            else:
                assert err <= 32 * U * rm, (r, c, v, float(ex[int(c)]), err / rm)
                worst_small = max(worst_small, err / rm / U)
    print(f"{quad} p={p}: worst sub-floor error {worst_small:.1f} u x row max")
