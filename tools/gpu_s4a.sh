mkdir -p gpurun_out
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/s4a_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/s4a_tests.log
python bench.py > gpurun_out/s4a_bench.json 2> gpurun_out/s4a_bench.err
echo "bench rc=$?"; tail -c 3000 gpurun_out/s4a_bench.json
