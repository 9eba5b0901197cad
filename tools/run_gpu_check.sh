# tests + per-config table on one B200 (used during development)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --all-configs --steps 5 ${CFGS:+--configs $CFGS} > gpurun_out/all_configs.jsonl 2> gpurun_out/all_configs.err; echo allcfg_rc=$?
tail -3 gpurun_out/all_configs.err
