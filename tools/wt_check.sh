# Developer: link-walk tiles (C3 matrix) -- parity tests, then timing (flushed steps).
timeout 1000 python -m pytest tests/test_wtile_gpu.py tests/test_configs_gpu.py tests/test_etile_gpu.py tests/test_submesh_gpu.py tests/test_graph_gpu.py -x -q -k "not c1 and not c2" 2>&1 | tail -4
LOAM_GPU_WT_INFO=1 python tools/cfg_probe.py 3 matrix wtile 2>&1 | grep -E "wtile|cfg" | sort -u | tail -3
