"""Per-phase share of warp-stall samples and executed instructions of k_xh1_fill (ncu source page).
usage: python scripts/ncu_phases.py REP   (phase boundaries = marker comments in lor_xh1.cu)"""
import collections, csv, os, re, subprocess, sys

src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2210_12253_b200", "csrc", "lor_xh1.cu")).read().splitlines()
marks = []  # (line, phase) from '// @phase NAME' markers
for i, l in enumerate(src, 1):
    m = re.search(r"// @phase (\w+)", l)
    if m:
        marks.append((i, m.group(1)))
def phase(ln):
    ph = "pre"
    for i, n in marks:
        if ln >= i:
            ph = n
    return ph
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr = f = None
agg = collections.defaultdict(lambda: [0, 0])
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and r and r[0].isdigit() and f == "lor_xh1.cu":
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")].replace(",", "") or 0)
            n = int(r[hdr.index("Instructions Executed")].replace(",", "") or 0)
        except ValueError:
            continue
        a = agg[phase(int(r[0]))]; a[0] += s; a[1] += n
ts = sum(v[0] for v in agg.values()) or 1; ti = sum(v[1] for v in agg.values()) or 1
for k, v in agg.items():
    print(f"{k:12s} stall {100*v[0]/ts:5.1f}%  inst {100*v[1]/ti:5.1f}%  {v[1]:12d}")
