# edge-tile sweep (C3 matrix): parity check, rows x stages table, optional ncu capture (NCU=1)
O=gpurun_out/${TAG:-e3}; mkdir -p $O
timeout 300 python tools/etile_check.py > $O/check.log 2>&1; echo check_rc=$?; tail -4 $O/check.log
for st in ${STAGES:-1 2}; do for rows in ${ROWS:-128 64}; do
  LOAM_GPU_ET_STAGES=$st LOAM_GPU_ET_ROWS=$rows timeout 300 python bench.py --all-configs --configs ${CFG:-3m} --strategies auto --steps 10 2>/dev/null | python tools/table.py /dev/stdin | sed "s/^/st=$st rows=$rows /"
done; done
if [ -n "$NCU" ]; then
ncu --set full --clock-control none --import-source on -k regex:k_etile -s 2 -c 1 -o $O/et python bench.py --all-configs --configs 3m --strategies auto --steps 3 > $O/ncu.log 2>&1; echo ncu_rc=$?
python tools/ncu_summary.py $O/et.ncu-rep 20 > $O/et.txt 2>&1; python tools/ncu_lines.py $O/et.ncu-rep 30 >> $O/et.txt 2>&1
fi
