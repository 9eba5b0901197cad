timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --all-configs --steps 10 > gpurun_out/all_configs.jsonl 2> gpurun_out/all_configs.err; echo allcfg_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err; echo ref_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
