mkdir -p gpurun_out
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/s4s_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/s4s_tests.log
python bench.py > gpurun_out/s4s_bench.json 2> gpurun_out/s4s_bench.err
echo "bench rc=$?"; tail -c 400 gpurun_out/s4s_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none -k regex:"k_box|k_gemv" -c 28 --csv --log-file gpurun_out/s4s_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/s4s_ncu.log 2>&1
tail -2 gpurun_out/s4s_ncu.log
for pair in "0 v0" "4 p1" "5 u0"; do
  set -- $pair
  OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_box -s $1 -c 1 -f -o gpurun_out/s4s_box_$2 python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/s4s_ncu_$2.log 2>&1
done
OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 0 -c 1 -f -o gpurun_out/s4s_gemv python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/s4s_ncu_gemv.log 2>&1
ls -la gpurun_out/*.ncu-rep | tail -5
