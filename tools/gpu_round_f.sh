set -x
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/rf_bench.json 2> gpurun_out/rf_bench.err
tail -c 3000 gpurun_out/rf_bench.json
tail -5 gpurun_out/rf_bench.err
timeout 300 python tools/prof_apply.py --config green_cubes_n256 --reps 2 > gpurun_out/rf_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/rf_launches.csv python tools/prof_apply.py --config green_cubes_n256 --reps 2 > gpurun_out/rf_ncu.log 2>&1
