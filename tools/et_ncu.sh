# ncu full capture of the edge-tile kernel (C3 matrix); env passes through (LOAM_GPU_ET_*)
O=gpurun_out/${TAG:-en}; mkdir -p $O
python bench.py --all-configs --configs 3m --strategies auto --steps 3 > $O/plain.log 2>&1; echo plain_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_etile -s 2 -c 1 -o $O/et python bench.py --all-configs --configs 3m --strategies auto --steps 3 > $O/ncu.log 2>&1; echo ncu_rc=$?
python tools/ncu_summary.py $O/et.ncu-rep 20 > $O/et.txt 2>&1; python tools/ncu_lines.py $O/et.ncu-rep 40 >> $O/et.txt 2>&1
ncu -i $O/et.ncu-rep --page raw --csv 2>/dev/null > $O/et_raw.csv
