mkdir -p gpurun_out
( time python -m pytest tests/test_sharded.py tests/test_sharded_cpp.py -x -q ) > gpurun_out/s4c_tests.log 2>&1
echo "tests rc=$?"; tail -8 gpurun_out/s4c_tests.log
