# developer sweep of the canonical pair-tile plan parameters (pairs seg slots runs per tile)
for cfg in ${PT_CFGS:-"768 4096 1024 48" "384 2048 512 48" "384 4096 1024 48" "1536 4096 1024 64" "512 3072 768 48" "256 2048 512 32"}; do
  set -- $cfg
  LOAM_GPU_PT_PAIRS=$1 LOAM_GPU_PT_SEG=$2 LOAM_GPU_PT_SLOTS=$3 LOAM_GPU_PT_RUNS=$4 timeout 300 \
    python bench.py --all-configs --configs ${PT_CONFIGS:-3m,5} --strategies auto --steps 5 2>/dev/null | \
    python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$cfg', 'C%s%s' % (d['config'], d['part'] or ''), round(d['ms'],4), round(d['frac_of_measured_peak'],3), round(d['first_call_s'],2))
"
done
