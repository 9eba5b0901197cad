# Developer: fused Taylor-Hood launch -- parity tests, then timing (flushed steps) fused vs separate.
O=gpurun_out/${TAG:-th}; mkdir -p $O
timeout 900 python -m pytest tests/test_thtile_gpu.py tests/test_configs_gpu.py -k "thtile or c5" -x -q > $O/pytest.log 2>&1; echo pytest_rc=$?; tail -15 $O/pytest.log
LOAM_GPU_TH_INFO=1 LOAM_GPU_PLAN_TIMING=1 python tools/cfg_probe.py 5 - fused > $O/probe.log 2>&1; tail -12 $O/probe.log
LOAM_GPU_NO_THTILE=1 python tools/cfg_probe.py 5 - separate 2>&1 | tail -1
