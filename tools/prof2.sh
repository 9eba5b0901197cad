# two ncu captures: C3 matrix and C3 residual under one strategy
for c in ${CFGS:-3m 3r}; do
python bench.py --all-configs --configs $c --strategies ${STRAT:-patch} --steps 3 > gpurun_out/plain_$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_patch} -s 2 -c 1 -o gpurun_out/${OUT:-patch}_$c python bench.py --all-configs --configs $c --strategies ${STRAT:-patch} --steps 3 > gpurun_out/ncu_$c.log 2>&1
echo ncu_$c rc=$?
done
