set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -x -q -m gpu --durations=25 > gpurun_out/r2a_tests.log 2>&1
tail -40 gpurun_out/r2a_tests.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
tail -c 2500 gpurun_out/r2a_bench.json
tail -5 gpurun_out/r2a_bench.err
