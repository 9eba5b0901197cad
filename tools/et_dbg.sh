for d in 0 1 2 3 4 7; do
  LOAM_GPU_ET_DBG=$d LOAM_GPU_ET_STAGES=${ST:-2} LOAM_GPU_ET_ROWS=${ROWS:-64} timeout 300 python bench.py --all-configs --configs 3m --strategies auto --steps 10 2>/dev/null | python tools/table.py /dev/stdin | sed "s/^/dbg=$d /"
done
