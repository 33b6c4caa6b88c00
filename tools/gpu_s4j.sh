mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dropin_cpp.py tests/test_capi.py -x -q > gpurun_out/s4j_tests.log 2>&1; tail -15 gpurun_out/s4j_tests.log
