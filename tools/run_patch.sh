# patch-kernel parity + table (development)
timeout 600 python -m pytest tests/test_configs_gpu.py -x -q -k "patch" > gpurun_out/pytest_patch.log 2>&1; echo pytest_rc=$?; tail -15 gpurun_out/pytest_patch.log
timeout 900 python bench.py --all-configs --steps 10 --strategies ${STRATS:-auto,patch} ${CFGS:+--configs $CFGS} > gpurun_out/all_patch.jsonl 2> gpurun_out/all_patch.err; echo allcfg_rc=$?
tail -3 gpurun_out/all_patch.err
