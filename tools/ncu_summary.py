"""Summarise an ncu report: key metrics, stall reasons, hottest SASS lines."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    print("kernel:", vals[hdr.index("Kernel Name")][:110])
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.per_cycle_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__waves_per_multiprocessor",
            "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
            "launch__shared_mem_per_block_dynamic"]
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w:60s} {vals[i]:>14s} {units[i]}")
    st = [(h, vals[i]) for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("_per_issue_active.ratio")]
    st = sorted(st, key=lambda x: -float(x[1] or 0))[:6]
    print("  stalls/issue:", ", ".join(f"{h.split('stalled_')[1].split('_per')[0]}={float(v):.1f}" for h, v in st))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src)))
if len(r) > 2:
    h = r[1]; body = r[2:]
    i_src, i_s = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(x[i_s] or 0) for x in body)
    print("  hottest SASS (share of stall samples):")
    for x in sorted(body, key=lambda x: -int(x[i_s] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
        print(f"   {int(x[i_s])/tot*100:5.1f}%  {x[i_src].strip()[:90]}")
