for e in X=0 LOAM_GPU_NO_STAR=1; do
env $e ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_star|k_ring|k_cell|k_tile" --csv python bench.py --all-configs --configs 1 --strategies auto --steps 3 2>/dev/null | grep -v "^{" | python -c "
import sys,csv
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
print('$e', [(r[ki][:40], r[vi]) for r in rows[1:]][-4:])
"
done
