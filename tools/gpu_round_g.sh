set -x
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/rg_bench.json 2> gpurun_out/rg_bench.err
tail -c 1500 gpurun_out/rg_bench.json
tail -3 gpurun_out/rg_bench.err
OIOBF_NO_GRAPH=1 timeout 300 python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/rg_plain.log 2>&1 && \
OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_box -s 0 -c 1 -o gpurun_out/rg_box_v0 python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/rg_ncu.log 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/rg_tests.log 2>&1
tail -3 gpurun_out/rg_tests.log
