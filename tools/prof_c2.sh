python bench.py --all-configs --configs 2 --strategies ${STRAT:-auto} --steps 3 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_nbr_mat} -s 3 -c 1 -o gpurun_out/${OUT:-c2_nbr} python bench.py --all-configs --configs 2 --strategies ${STRAT:-auto} --steps 3 > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$?
