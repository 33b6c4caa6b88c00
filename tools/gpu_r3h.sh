mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu --durations=10 > gpurun_out/r3h_tests.log 2>&1
tail -14 gpurun_out/r3h_tests.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r3h_bench.json 2> gpurun_out/r3h_bench.err
tail -c 300 gpurun_out/r3h_bench.json; tail -2 gpurun_out/r3h_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none -k regex:"k_box|k_gemv" -c 70 --csv --log-file gpurun_out/r3h_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/r3h_ncu.log 2>&1
tail -2 gpurun_out/r3h_ncu.log
