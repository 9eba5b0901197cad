# Round evidence: tests, smoke, contract bench line, reference arm, per-config strategy
# table, ncu launch list of the bench, full ncu captures of the edge-tile kernels.
O=gpurun_out/ev; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.jsonl 2> $O/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_arm.jsonl 2> $O/bench_ref.err; echo ref_rc=$?
timeout 1500 python bench.py --all-configs --steps 10 ${STRATS:+--strategies $STRATS} > $O/strategies_all_configs.jsonl 2> $O/all.err; echo all_rc=$?
python tools/table.py $O/strategies_all_configs.jsonl > $O/strategies_all_configs.txt
python tools/c5_split.py > $O/c5_split.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $O/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-config-table > $O/ncu_launch.log 2>&1; echo launch_rc=$?
summ() { python tools/ncu_summary.py $1.ncu-rep 20 > $1.txt 2>&1; python tools/ncu_lines.py $1.ncu-rep 25 >> $1.txt 2>&1; ncu -i $1.ncu-rep --page raw --csv > $1_raw.csv 2>/dev/null; rm -f $1.ncu-rep; }
ncu --set full --clock-control none --import-source on -k regex:k_etile -s 2 -c 1 -o $O/cfg3m python bench.py --all-configs --configs 3m --strategies auto --steps 3 > $O/ncu_cfg3m.log 2>&1; echo ncu_3m_rc=$?
summ $O/cfg3m
ncu --set full --clock-control none --import-source on -k regex:k_etile -s 1 -c 1 -o $O/cfg5a python tools/c5_split.py > $O/ncu_cfg5a.log 2>&1; echo ncu_5a_rc=$?
summ $O/cfg5a
ncu --set full --clock-control none --import-source on -k regex:k_ntile -s 2 -c 1 -o $O/cfg4 python bench.py --all-configs --configs 4 --strategies auto --steps 3 > $O/ncu_cfg4.log 2>&1; echo ncu_4_rc=$?
summ $O/cfg4
ncu --set full --clock-control none --import-source on -k regex:k_rtile -s 1 -c 1 -o $O/cfg5b python tools/c5_split.py > $O/ncu_cfg5b.log 2>&1; echo ncu_5b_rc=$?
summ $O/cfg5b
ncu --set full --clock-control none --import-source on -k regex:k_star -s 2 -c 1 -o $O/cfg1 python bench.py --all-configs --configs 1 --strategies auto --steps 3 > $O/ncu_cfg1.log 2>&1; echo ncu_1_rc=$?
summ $O/cfg1
ncu --set full --clock-control none --import-source on -k regex:k_ring -s 5 -c 1 -o $O/c2_ring python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-config-table > $O/ncu_c2.log 2>&1; echo ncu_c2_rc=$?
summ $O/c2_ring
ncu --set full --clock-control none --import-source on -k regex:k_cell -s 2 -c 1 -o $O/cfg3r python bench.py --all-configs --configs 3r --strategies auto --steps 3 > $O/ncu_cfg3r.log 2>&1; echo ncu_3r_rc=$?
summ $O/cfg3r
