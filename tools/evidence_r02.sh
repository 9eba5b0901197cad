# Round-2 evidence: GPU tests, smoke, the contract bench line, the reference
# arm, per-config protocol table (rotation / flushed, default and
# deterministic), plan-build phases, the ncu launch list of the bench command
# and one --set full capture per config's dominant kernel (every profiled
# command first exits 0 without ncu).  Outputs under gpurun_out/ev2/.
O=gpurun_out/${EV:-ev2}; mkdir -p $O
summ() { python tools/ncu_summary.py $1.ncu-rep 20 > $1.txt 2>&1; python tools/ncu_lines.py $1.ncu-rep 25 >> $1.txt 2>&1; ncu -i $1.ncu-rep --page raw --csv > $1_raw.csv 2>/dev/null; rm -f $1.ncu-rep; }
timeout 1100 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.jsonl 2> $O/bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_arm.jsonl 2> $O/bench_ref.err; echo ref_rc=$?
python tools/rot_probe.py > $O/protocol_table.txt 2>&1; echo rot_rc=$?
DET=1 python tools/rot_probe.py 2>&1 | grep config > $O/protocol_table_deterministic.txt; echo det_rc=$?
python tools/plan_probe.py > $O/plan_phases.txt 2>&1; echo plan_rc=$?
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-config-table > $O/plain_bench.jsonl 2> $O/plain_bench.err; echo plain_rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file $O/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-config-table > $O/ncu_launch.log 2>&1; echo launch_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_ring -s 12 -c 1 -o $O/c2_ring python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-config-table > $O/ncu_c2.log 2>&1; echo ncu_c2_rc=$?
summ $O/c2_ring
for c in 1 3r 3m 4 5; do
  case $c in 1) k=k_star;; 3r) k=k_cell;; 3m) k=k_wtile;; 4) k=k_ltile;; 5) k=k_thtile;; esac
  python bench.py --all-configs --configs $c --strategies auto --steps 3 > $O/plain_cfg$c.log 2>&1; echo plain_$c rc=$?
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/cfg$c python bench.py --all-configs --configs $c --strategies auto --steps 3 > $O/ncu_cfg$c.log 2>&1; echo ncu_$c rc=$?
  summ $O/cfg$c
done
