"""Per-source-line stall samples / instructions from an ncu report (compile with -lineinfo).
usage: ncu_lines.py REP [TOP]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, 0, ""]); fname = None; hdr = None; line = None; src = ""
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; hdr = None; continue
    if len(r) == 2 and r[0] == "Function Name":
        continue
    if hdr is None:
        hdr = r; continue
    if r[0]:
        line, src = r[0], r[1]
    try:
        s = int(r[4] or 0); ie = int(r[7] or 0)
    except (ValueError, IndexError):
        continue
    a = agg[(fname, line)]
    a[0] += s; a[1] += ie; a[2] = src.strip()[:90]
tot = sum(v[0] for v in agg.values()) or 1; toti = sum(v[1] for v in agg.values()) or 1
for (f, ln), (s, ie, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{s/tot*100:5.1f}% stall {ie/toti*100:5.1f}% inst  {f}:{ln}  {src}")
