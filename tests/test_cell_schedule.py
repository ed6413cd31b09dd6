"""The precomputed thread/slot schedule of the 5^3 cell box (scripts/gen_cell_schedule.py, embedded in
lor_xh1.cu as k545) is a bijection onto slots 0..127 with the bank properties DESIGN.md §4 states.
Host-only: no GPU needed."""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _table_from_source():
    src = open(os.path.join(ROOT, "paper_2210_12253_b200", "csrc", "lor_xh1.cu")).read()
    m = re.search(r"k545\[128\] = \{([^}]*)\}", src)
    assert m, "k545 table not found"
    return [int(v) for v in m.group(1).split(",")]


def test_embedded_table_matches_generator():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "gen_cell_schedule.py")],
                         capture_output=True, text=True, check=True).stdout.strip()
    gen = [int(v) for v in out.strip("{}").split(",")]
    assert gen == _table_from_source()


def test_schedule_properties():
    perm = _table_from_source()
    NB, XR, XS = 5, 7, 43
    cells = [c for c in perm if c != 255]
    assert sorted(cells) == list(range(NB ** 3))                 # every box cell exactly once
    for h in range(8):                                          # half-warp h = threads 16h..16h+15
        grp = [c for c in perm[16 * h:16 * h + 16] if c != 255]
        e = [(c % NB + XR * ((c // NB) % NB) + XS * (c // (NB * NB))) % 16 for c in grp]
        assert len(set(e)) == len(grp)                          # E-vector loads: distinct banks
    slot = {c: t for t, c in enumerate(perm) if c != 255}
    for z in range(NB):                                         # interior row gather: 4 x 4 windows
        for a in (0, 1):
            for b in (0, 1):
                w = [slot[x + NB * (y + NB * z)] % 16 for x in range(a, a + 4) for y in range(b, b + 4)]
                assert len(set(w)) == 16
