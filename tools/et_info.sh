# Developer: edge-tile footprint (C3 matrix) and time for tile caps.
for cells in 512 384 320 256; do for seg in 4096 3072; do
LOAM_GPU_ET_INFO=1 LOAM_GPU_ET_CELLS=$cells LOAM_GPU_ET_SEG=$seg python tools/cfg_probe.py 3 matrix "cells=$cells seg=$seg" 2>&1 | grep -E "etile:|cfg" | sort -u | tail -2
done; done
