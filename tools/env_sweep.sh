# run the all-configs table under several env settings: ENVS="A=1 B=2;C=3" (';'-separated)
IFS=';' read -ra SETS <<< "${ENVS}"
for e in "${SETS[@]}"; do
  env $e timeout 600 python bench.py --all-configs --steps 10 --strategies ${STRATS:-auto} --configs ${CFGS:-3m} 2>/dev/null | sed "s/^/{\"env\": \"$e\", \"r\": /; s/\$/}/"
done >> gpurun_out/sweep.jsonl
