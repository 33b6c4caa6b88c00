mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none -k regex:"k_box|k_gemv" -c 28 --csv --log-file gpurun_out/fin_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/fin_ncu.log 2>&1
tail -c 200 gpurun_out/fin_ncu.log
