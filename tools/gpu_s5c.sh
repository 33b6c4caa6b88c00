mkdir -p gpurun_out
( time python bench.py ) > gpurun_out/s5c_bench.json 2> gpurun_out/s5c_bench.err
echo "bench rc=$?"; tail -3 gpurun_out/s5c_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none -c 60 --csv --log-file gpurun_out/s5c_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/s5c_ncu.log 2>&1
tail -c 300 gpurun_out/s5c_ncu.log
OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_panel -s 4 -c 1 -f -o gpurun_out/s5c_panel python tools/prof_apply.py --config green_cubes_n256 --construct-only > gpurun_out/s5c_ncu_panel.log 2>&1
tail -2 gpurun_out/s5c_ncu_panel.log
