# Developer: row-owner sparsity build -- bit-exactness tests, then build times (row-owner vs radix) per config.
O=gpurun_out/${TAG:-sp}; mkdir -p $O
timeout 1000 python -m pytest tests/test_topology_data_gpu.py tests/test_configs_gpu.py tests/test_fullsize_gpu.py tests/test_submesh_gpu.py tests/test_thtile_gpu.py -x -q > $O/pytest.log 2>&1; echo pytest_rc=$?; tail -3 $O/pytest.log
python tools/sp_probe.py 2>&1 | tail -8
LOAM_GPU_SPARSITY_SORT=1 python tools/sp_probe.py 2>&1 | tail -8
