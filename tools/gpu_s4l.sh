mkdir -p gpurun_out
timeout 600 python tools/apply_ab.py green_cubes_n256 - OIOBF_BOX_ASYNC_FAC=0 - > gpurun_out/s4l_ab.jsonl 2> gpurun_out/s4l_ab.err
cat gpurun_out/s4l_ab.jsonl; tail -3 gpurun_out/s4l_ab.err
timeout 600 python tools/apply_ab.py green_cubes_n64 - > gpurun_out/s4l_ab2.jsonl 2> gpurun_out/s4l_ab2.err
cat gpurun_out/s4l_ab2.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "variants or box2 or contract or apply" > gpurun_out/s4l_tests.log 2>&1; tail -4 gpurun_out/s4l_tests.log
