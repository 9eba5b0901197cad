# Round-2 check: GPU tests, smoke, contract bench line, reference arm, per-config table.
O=gpurun_out/r02; mkdir -p $O
timeout 1100 python -m pytest tests -m gpu -q --durations=25 > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.jsonl 2> $O/bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_arm.jsonl 2> $O/bench_ref.err; echo ref_rc=$?
timeout 1200 python bench.py --all-configs --steps 10 > $O/strategies_all_configs.jsonl 2> $O/all.err; echo all_rc=$?
python tools/table.py $O/strategies_all_configs.jsonl > $O/strategies_all_configs.txt 2>&1
