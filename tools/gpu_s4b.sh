mkdir -p gpurun_out
timeout 300 python tools/prof_apply.py --config green_cubes_n256 --reps 2 > gpurun_out/s4b_plain.log 2>&1 || { tail gpurun_out/s4b_plain.log; exit 1; }
for pair in "0 v0" "1 v1" "4 p1" "5 u0"; do
  set -- $pair
  OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_box -s $1 -c 1 -f -o gpurun_out/s4b_box_$2 python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/s4b_ncu_$2.log 2>&1
  tail -n 1 gpurun_out/s4b_ncu_$2.log
done
timeout 600 python tools/shard_balance.py green_cubes_n64 green_cubes_n256 > gpurun_out/s4b_balance.jsonl 2> gpurun_out/s4b_balance.err
cat gpurun_out/s4b_balance.jsonl; tail -3 gpurun_out/s4b_balance.err
