"""Rebuild profiles/ncu_summary.json from the round's `ncu --set full` raw CSV
exports (profiles/r02/s6_*_raw.csv, the last evidence pass of the round): per config the dominant kernel's
duration and DRAM bytes next to its algorithmic bytes (bench.py reads the
C2 entry's traffic for roofline.traffic)."""
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALG = {"c2_matrix": 100745240, "c1_residual": 14712864, "c3_residual": 103852584, "c3_matrix": 556384800,
       "c4_elasticity": 1076350560, "c5_blocks": 1279402064}
SRC = {"c2_matrix": "s6_c2_ring", "c1_residual": "s6_cfg1", "c3_residual": "s6_cfg3r", "c3_matrix": "s6_cfg3m",
       "c4_elasticity": "s6_cfg4", "c5_blocks": "s6_cfg5"}
out = {}
for tag, stem in SRC.items():
    path = os.path.join(ROOT, "profiles", "r02", stem + "_raw.csv")
    rows = list(csv.reader(open(path)))
    hdr, unit, vals = rows[0], rows[1], rows[2]
    def get(name, scale=None):
        i = hdr.index(name)
        v = float(vals[i].replace(",", ""))
        u = unit[i]
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
                "nsecond": 1e-9, "msecond": 1e-3, "ms": 1e-3}.get(u, 1)
        return v * mult
    dur = get("gpu__time_duration.sum")
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    e = {"kernel": vals[hdr.index("Kernel Name")], "source": f"profiles/r02/{stem}.txt (ncu --set full --clock-control none, "
         "tools/evidence_r02.sh)", "duration_s": dur, "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes": rd + wr}
    if tag in ALG:
        e["algorithmic_bytes"] = ALG[tag]
        e["achieved_GBps_alg"] = ALG[tag] / dur / 1e9
    out[tag] = e
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
for k, v in out.items():
    print(k, f"{v['duration_s']*1e6:.1f} us", f"dram {v['dram_bytes']/1e6:.1f} MB", f"{v.get('achieved_GBps_alg', 0):.0f} GB/s")
