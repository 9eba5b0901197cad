# Developer: ncu --set full capture of the fused Taylor-Hood kernel (config 5), after a plain run.
O=gpurun_out/${TAG:-thn}; mkdir -p $O
python bench.py --all-configs --configs 5 --strategies auto --steps 3 > $O/plain.log 2>&1; echo plain_rc=$?; tail -2 $O/plain.log
ncu --set full --clock-control none --import-source on -k regex:k_thtile -s 2 -c 1 -o $O/th python bench.py --all-configs --configs 5 --strategies auto --steps 3 > $O/ncu.log 2>&1; echo ncu_rc=$?
python tools/ncu_summary.py $O/th.ncu-rep 20 > $O/th.txt 2>&1; python tools/ncu_lines.py $O/th.ncu-rep 40 >> $O/th.txt 2>&1
ncu -i $O/th.ncu-rep --page raw --csv 2>/dev/null > $O/th_raw.csv; rm -f $O/th.ncu-rep
