"""Aggregate an ncu source page (cuda,sass) per source line / line range.
usage: python scripts/ncu_lines.py REP [topN]"""
import csv, subprocess, sys, collections

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
f = None
agg = collections.defaultdict(lambda: [0, 0, ""])
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")].replace(",", "") or 0)
            n = int(r[hdr.index("Instructions Executed")].replace(",", "") or 0)
        except ValueError:
            s, n = 0, 0
        a = agg[(f, int(r[0]))]
        a[0] += s; a[1] += n; a[2] = r[1][:70]
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {ts}  warp-instr {ti}")
for (f, ln), (s, n, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f}:{ln:5d} stall {100*s/ts:5.1f}%  inst {100*n/ti:5.1f}%  {src}")
