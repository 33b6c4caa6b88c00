mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin_cpp.py -x -q -k "column_id or dropin or tucker" > gpurun_out/s4i_tests.log 2>&1; tail -15 gpurun_out/s4i_tests.log
