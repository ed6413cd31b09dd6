"""Bank-conflict-free thread/slot schedule of the 5x5x5 cell box of k_xh1_fill<4, 5>.

Each box cell c = (x, y, z) gets a storage slot s(c) = 16 * h(c) + rho(c), computed by thread s(c):
  * cell phase: the 16 lanes of half-warp h read the E-vector box at (x + 7 y + 43 z) mod 16 (the
    XR = 7, XS = 43 layout) -> distinct within every half-warp (reads conflict free), and write
    slot s = thread (writes conflict free);
  * row gather: the rows of an interior element (4 x 4 per z layer per half-warp) read the cells of a
    4 x 4 window at offsets {0, 1}^2 -> rho must be injective on every such window;
  * rho = a per-layer relabelling of (x mod 4) + 4 (y mod 4) (injective on every 4 x 4 window),
    chosen so that every rho class has <= 8 cells; h = a proper 8-edge-colouring (Koenig) of the
    bipartite multigraph (E-vector residue class, rho class) whose edges are the cells.
Prints the C initialiser of perm[128] (slot -> cell id, 255 = none)."""
import itertools

NB, XR, XS = 5, 7, 43
cells = [(x, y, z) for z in range(NB) for y in range(NB) for x in range(NB)]
cid = lambda x, y, z: x + NB * (y + NB * z)
base = lambda x, y: (x % 4) + 4 * (y % 4)

# per-layer relabelling (base class sizes per layer: one 4, six 2, nine 1): layer z sends its 4-class
# to colour z, its six 2-classes round-robin to colours 5..15 (so each gets 2 or 3 of them over
# the five layers), its 1-classes to the remaining colours -> every colour holds 7 or 8 cells
size = [0] * 16
for y in range(NB):
    for x in range(NB):
        size[base(x, y)] += 1
tot, relabel = [0] * 16, []
for z in range(NB):
    four = [b for b in range(16) if size[b] == 4]
    twos = [b for b in range(16) if size[b] == 2]
    ones = [b for b in range(16) if size[b] == 1]
    m = {four[0]: z}
    tcols = [5 + (6 * z + i) % 11 for i in range(6)]
    for b, c in zip(twos, tcols):
        m[b] = c
    rest = [c for c in range(16) if c not in m.values()]
    for b, c in zip(ones, rest):
        m[b] = c
    for b, c in m.items():
        tot[c] += size[b]
    relabel.append(m)
assert max(tot) <= 8, tot
rho = {c: relabel[c[2]][base(c[0], c[1])] for c in cells}
e = {c: (c[0] + XR * c[1] + XS * c[2]) % 16 for c in cells}

# Koenig edge colouring with 8 colours (alternating-path recolouring)
L = [[None] * 8 for _ in range(16)]  # L[e][colour] = cell
R = [[None] * 8 for _ in range(16)]  # R[rho][colour] = cell
col = {}
for c in cells:
    u, v = e[c], rho[c]
    a = next(k for k in range(8) if L[u][k] is None)
    b = next(k for k in range(8) if R[v][k] is None)
    if a != b and R[v][a] is not None:
        # flip the a/b alternating path starting at v (via its a-edge)
        path, side, node, k = [], 'R', v, a
        while True:
            edge = (R if side == 'R' else L)[node][k]
            if edge is None:
                break
            path.append(edge)
            node = e[edge] if side == 'R' else rho[edge]
            side = 'L' if side == 'R' else 'R'
            k = b if k == a else a
        for ed in path:
            L[e[ed]][col[ed]] = None; R[rho[ed]][col[ed]] = None
        for ed in path:
            col[ed] = b if col[ed] == a else a
            L[e[ed]][col[ed]] = ed; R[rho[ed]][col[ed]] = ed
    col[c] = a
    L[u][a] = c; R[v][a] = c

slot = {c: 16 * col[c] + rho[c] for c in cells}
assert len(set(slot.values())) == len(cells)
perm = [255] * 128
for c in cells:
    perm[slot[c]] = cid(*c)
for h in range(8):  # checks
    grp = [c for c in cells if slot[c] // 16 == h]
    assert len({e[c] for c in grp}) == len(grp)
for z in range(NB):
    for a, b in itertools.product((0, 1), repeat=2):
        w = [(x, y, z) for x in range(a, a + 4) for y in range(b, b + 4)]
        assert len({rho[c] for c in w}) == 16
print("{" + ", ".join(str(v) for v in perm) + "}")
