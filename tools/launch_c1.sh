python bench.py --all-configs --configs 1 --strategies auto,atomic --steps 5 > gpurun_out/c1_plain.jsonl 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.per_cycle_active --clock-control none -k regex:"k_ring|k_cell|memset" --csv python bench.py --all-configs --configs 1 --strategies auto,atomic --steps 5 > gpurun_out/c1_ncu.csv 2>/dev/null
echo rc=$?
