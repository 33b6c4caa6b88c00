mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r4a_smi.txt
timeout 2400 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/r4a_tests.log 2>&1
tail -20 gpurun_out/r4a_tests.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r4a_bench.json 2> gpurun_out/r4a_bench.err
tail -c 400 gpurun_out/r4a_bench.json; tail -3 gpurun_out/r4a_bench.err
