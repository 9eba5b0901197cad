import json, sys
for l in open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/all_configs.jsonl'):
    r = json.loads(l)
    if 'error' in r:
        print(r); continue
    print(f"C{r['config']}{'' if r['part'] is None else r['part'][0]:1} {r['strategy']:7s} ms={r['ms']:8.3f} "
          f"cells/s={r['cells_per_s']:.3e} GB/s={r['GB_s']:7.1f} frac={r['frac_of_measured_peak']:.3f} "
          f"launches={r['launches_per_step']:.0f} first={r['first_call_s']:.2f}s")
