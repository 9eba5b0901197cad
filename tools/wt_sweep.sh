# Developer: link-walk tiles (C3 matrix): tests of the path, then rows-per-tile / stages sweep and an ncu capture.
O=gpurun_out/${TAG:-wts}; mkdir -p $O
timeout 600 python -m pytest tests/test_wtile_gpu.py -x -q 2>&1 | tail -5
for st in 2 1; do for rows in 128 96 64; do
LOAM_GPU_WT_STAGES=$st LOAM_GPU_WT_ROWS=$rows LOAM_GPU_WT_INFO=1 python tools/cfg_probe.py 3 matrix "st=$st rows=$rows" 2>&1 | grep -E "wtile:|cfg" | sort -u | tail -2
done; done
ncu --set full --clock-control none --import-source on -k regex:k_wtile -s 2 -c 1 -o $O/wt python bench.py --all-configs --configs 3m --strategies auto --steps 3 > $O/ncu.log 2>&1; echo ncu_rc=$?
python tools/ncu_summary.py $O/wt.ncu-rep 20 > $O/wt.txt 2>&1; python tools/ncu_lines.py $O/wt.ncu-rep 40 >> $O/wt.txt 2>&1
ncu -i $O/wt.ncu-rep --page raw --csv 2>/dev/null > $O/wt_raw.csv; rm -f $O/wt.ncu-rep
