# launch list of the bench command (apply kernels) and ncu --set full of the first V / last U level and the GEMV
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none -k regex:"k_box|k_gemv" -c 28 --csv --log-file gpurun_out/cap_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/cap_ncu.log 2>&1
tail -c 200 gpurun_out/cap_ncu.log
for pair in "0 v0" "1 v1" "4 p1" "5 u0"; do
  set -- $pair
  OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_box -s $1 -c 1 -f -o gpurun_out/cap_box_$2 python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/cap_ncu_$2.log 2>&1
done
ls gpurun_out/cap_*.ncu-rep
