# Developer: fused Taylor-Hood launch -- parity tests, then timing (flushed steps) fused vs separate.
O=gpurun_out/${TAG:-th}; mkdir -p $O
timeout 900 python -m pytest tests/test_thtile_gpu.py tests/test_configs_gpu.py -k "thtile or c5" -x -q > $O/pytest.log 2>&1; echo pytest_rc=$?; tail -5 $O/pytest.log
for st in 2 3; do for ed in 64 96; do
LOAM_GPU_TH_STAGES=$st LOAM_GPU_TH_EDGES=$ed python tools/cfg_probe.py 5 - "st=$st ed=$ed" 2>&1 | tail -1
done; done
