# usage: CFG=3m KREGEX=k_owner_mat OUT=name bash tools/prof_cfg.sh
python bench.py --all-configs --configs ${CFG} --strategies ${STRAT:-auto} --steps 3 > gpurun_out/plain_${OUT}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${SKIP:-2} -c 1 -o gpurun_out/${OUT} python bench.py --all-configs --configs ${CFG} --strategies ${STRAT:-auto} --steps 3 > gpurun_out/ncu_${OUT}.log 2>&1
echo ncu_rc=$?
