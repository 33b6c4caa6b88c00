mkdir -p gpurun_out
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/s5b_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/s5b_tests.log
