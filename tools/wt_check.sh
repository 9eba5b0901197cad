# Developer: link-walk tiles (C3 matrix) -- parity tests, then timing (flushed steps) vs the edge tiles.
O=gpurun_out/${TAG:-wt}; mkdir -p $O
timeout 1000 python -m pytest tests/test_configs_gpu.py tests/test_etile_gpu.py tests/test_submesh_gpu.py tests/test_deterministic_gpu.py tests/test_graph_gpu.py tests/test_irregular_gpu.py -x -q > $O/pytest.log 2>&1; echo pytest_rc=$?; tail -12 $O/pytest.log
LOAM_GPU_WT_INFO=1 LOAM_GPU_PLAN_TIMING=1 python tools/cfg_probe.py 3 matrix wtile 2>&1 | grep -E "wtile|cfg|walk" | sort -u | tail -6
LOAM_GPU_NO_WTILE=1 python tools/cfg_probe.py 3 matrix etile 2>&1 | tail -1
