mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "butterfly_parity or cta_variants or register_cached or sampled_slots or config3 or golden or column_id" > gpurun_out/r2v_tests.log 2>&1
tail -3 gpurun_out/r2v_tests.log
timeout 600 python tools/apply_ab.py green_cubes_n256 - > gpurun_out/r2v_ab3.jsonl 2>&1; cat gpurun_out/r2v_ab3.jsonl
timeout 2700 python tools/proxy_sweep.py radon2d_n1024 1,12,23 > gpurun_out/r2v_radon1024.jsonl 2>&1
cat gpurun_out/r2v_radon1024.jsonl
