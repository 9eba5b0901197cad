O=gpurun_out/${TAG:-c5n}; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:k_etile -s 1 -c 1 -o $O/et python tools/c5_split.py > $O/ncu.log 2>&1; echo ncu_rc=$?
python tools/ncu_summary.py $O/et.ncu-rep 12 > $O/et.txt 2>&1; python tools/ncu_lines.py $O/et.ncu-rep 25 >> $O/et.txt 2>&1
ncu -i $O/et.ncu-rep --page raw --csv 2>/dev/null > $O/et_raw.csv
