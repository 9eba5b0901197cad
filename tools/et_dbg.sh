for d in ${DBGS:-0 8 1}; do
  LOAM_GPU_ET_DBG=$d timeout 300 python bench.py --all-configs --configs 3m --strategies auto --steps 10 2>/dev/null | python tools/table.py /dev/stdin | sed "s/^/dbg=$d /"
done
