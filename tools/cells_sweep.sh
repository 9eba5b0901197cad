for b in ${CELLS:-512 1024 2048}; do
  LOAM_GPU_PATCH_CELLS=$b timeout 600 python bench.py --all-configs --steps 10 --strategies patch --configs ${CFGS:-3r} 2>/dev/null | sed "s/^/{\"budget\": $b, \"r\": /; s/\$/}/"
done >> gpurun_out/sweep.jsonl
