O=gpurun_out/${TAG:-ntn}; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:k_ntile -s 2 -c 1 -o $O/nt python bench.py --all-configs --configs 4 --strategies auto --steps 3 > $O/ncu.log 2>&1; echo ncu_rc=$?
python tools/ncu_summary.py $O/nt.ncu-rep 12 > $O/nt.txt 2>&1; python tools/ncu_lines.py $O/nt.ncu-rep 30 >> $O/nt.txt 2>&1
ncu -i $O/nt.ncu-rep --page raw --csv 2>/dev/null > $O/nt_raw.csv
