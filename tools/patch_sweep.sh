# budget sweep of the patch kernel: CFGS configs, BUDGETS list, appends to gpurun_out/sweep.jsonl
for b in ${BUDGETS:-1024 2048 3072 4096}; do
  LOAM_GPU_PATCH_BUDGET=$b timeout 600 python bench.py --all-configs --steps 10 --strategies patch --configs ${CFGS:-3m} 2>/dev/null | sed "s/^/{\"budget\": $b, \"r\": /; s/\$/}/"
done >> gpurun_out/sweep.jsonl
echo done
