# Developer: tile-size / stage sweep of the fused Taylor-Hood kernel (flushed steps, config 5).
for st in 2 3; do for sp in 64 96 128; do for ed in 48 64 96 128; do
LOAM_GPU_TH_STAGES=$st LOAM_GPU_TH_SPOKES=$sp LOAM_GPU_TH_EDGES=$ed python tools/cfg_probe.py 5 - "st=$st sp=$sp ed=$ed" 2>&1 | tail -1
done; done; done
