mkdir -p gpurun_out
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/s5f_tests.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/s5f_tests.log
( time python bench.py ) > gpurun_out/s5f_bench.json 2> gpurun_out/s5f_bench.err
echo "bench rc=$?"; tail -3 gpurun_out/s5f_bench.err
