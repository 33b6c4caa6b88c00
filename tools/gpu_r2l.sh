mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
timeout 600 python tools/apply_ab.py green_cubes_n256 - OIOBF_GEMV_SHORT=0 > gpurun_out/r2l_ab3.jsonl 2>&1; cat gpurun_out/r2l_ab3.jsonl
timeout 1200 python -m pytest tests/test_sharded_cpp.py tests/test_sharded.py tests/test_capi.py -x -q -m gpu > gpurun_out/r2l_tests.log 2>&1
tail -15 gpurun_out/r2l_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "butterfly_parity or config3 or multi_rhs or host_pipeline or contract_async" > gpurun_out/r2l_tests2.log 2>&1
tail -3 gpurun_out/r2l_tests2.log
timeout 600 python tools/panel_ab.py green_cubes_n64,green_cubes_n256 '' > gpurun_out/r2l_pab.jsonl 2>&1; cat gpurun_out/r2l_pab.jsonl
