set -x
timeout 900 python bench.py --all-configs --steps 5 > gpurun_out/all_configs.jsonl 2> gpurun_out/all_configs.err
echo allcfg_rc=$?
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_owner_mat -s 4 -c 1 -o gpurun_out/c2_owner python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo ncu2_rc=$?
