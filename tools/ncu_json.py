"""Update profiles/ncu_summary.json with one kernel's ncu numbers.

usage: python tools/ncu_json.py TAG REPORT.ncu-rep|RAW.csv ALGORITHMIC_BYTES "source label"
(RAW.csv = `ncu -i REPORT --page raw --csv` output)
Per-launch DRAM traffic (dram__bytes_read + write) and duration of the first
kernel in the report; bench.py reads the traffic back as roofline.traffic."""
import csv, io, json, os, subprocess, sys

tag, rep, alg, label = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
raw = open(rep).read() if rep.endswith(".csv") else \
    subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]


def num(name):
    i = hdr.index(name)
    v = float(vals[i].replace(",", ""))
    u = units[i]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}.get(u, 1)
    return v * scale


d = num("gpu__time_duration.sum")
r, w = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_summary.json")
js = json.load(open(path)) if os.path.exists(path) else {}
js[tag] = {"kernel": vals[hdr.index("Kernel Name")][:110], "source": label, "duration_s": d,
           "dram_read_bytes": r, "dram_write_bytes": w, "dram_bytes": r + w, "algorithmic_bytes": alg,
           "achieved_GBps_alg": alg / d / 1e9}
json.dump(js, open(path, "w"), indent=1)
print(tag, js[tag])
