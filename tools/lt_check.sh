# Developer: link tiles (config 4) -- parity tests, then timing (flushed steps).
O=gpurun_out/${TAG:-lt}; mkdir -p $O
timeout 900 python -m pytest tests/test_configs_gpu.py tests/test_submesh_gpu.py tests/test_graph_gpu.py tests/test_deterministic_gpu.py -k "c4 or elasticity or cfg4 or 4" -x -q > $O/pytest.log 2>&1; echo pytest_rc=$?; tail -3 $O/pytest.log
python tools/cfg_probe.py 4 - static 2>&1 | tail -1
LOAM_GPU_LT_STAGES=3 python tools/cfg_probe.py 4 - "static st=3" 2>&1 | tail -1
