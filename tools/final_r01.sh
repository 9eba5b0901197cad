# Round-1 evidence run: tests, contract bench line, reference arm, strategy
# table, solver / wave lines, ncu launch list and full captures of the top
# kernels.  Outputs under gpurun_out/final/ (copied to profiles/r01/ after review).
set -x
O=gpurun_out/final
SKIP=${SKIP:-}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.jsonl 2> $O/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_arm.jsonl 2> $O/bench_ref.err; echo ref_rc=$?
timeout 1200 python bench.py --all-configs --steps 10 > $O/strategies_all_configs.jsonl 2> $O/all.err; echo all_rc=$?
timeout 600 python bench.py --solver --steps 10 > $O/solver_bench.jsonl 2> $O/solver.err; echo solver_rc=$?
timeout 600 python bench.py --wave --steps 200 > $O/wave_bench.jsonl 2> $O/wave.err; echo wave_rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $O/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo launch_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_ring -s 5 -c 1 -o $O/c2_ring python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_c2.log 2>&1; echo ncu_c2_rc=$?
summ() { python tools/ncu_summary.py $1.ncu-rep 20 > $1.txt 2>&1; python tools/ncu_lines.py $1.ncu-rep 25 >> $1.txt 2>&1; ncu -i $1.ncu-rep --page raw --csv > $1_raw.csv 2>/dev/null; }
summ $O/c2_ring
for c in 1 3m 3r 4 5; do
  case $c in 1) k=k_star;; 3m) k=k_ptile;; 3r) k=k_cell;; 4) k=k_owner;; 5) k=k_ptile;; esac
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/cfg$c python bench.py --all-configs --configs $c --strategies auto --steps 3 > $O/ncu_cfg$c.log 2>&1; echo ncu_$c rc=$?
  summ $O/cfg$c; rm -f $O/cfg$c.ncu-rep
done
