mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/r2n_tests.log 2>&1
tail -22 gpurun_out/r2n_tests.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err
tail -c 600 gpurun_out/r2n_bench.json; tail -3 gpurun_out/r2n_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_box|k_gemv" --log-file gpurun_out/r2n_launches.csv python tools/prof_apply.py --config green_cubes_n256 --reps 2 > gpurun_out/r2n_ncu.log 2>&1
OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 0 -c 1 -o gpurun_out/r2n_gemv_c3 python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/r2n_ncu2.log 2>&1
bash tools/gpu_r2m.sh
