mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
timeout 600 python tools/apply_ab.py green_cubes_n256 - OIOBF_GEMV_L2AHEAD=0 > gpurun_out/r2p_ab3.jsonl 2>&1; cat gpurun_out/r2p_ab3.jsonl
timeout 600 python tools/apply_ab.py green_cubes_n64 - > gpurun_out/r2p_ab2.jsonl 2>&1; cat gpurun_out/r2p_ab2.jsonl
timeout 600 python tools/apply_ab.py dft6_n16 - > gpurun_out/r2p_ab4.jsonl 2>&1; cat gpurun_out/r2p_ab4.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_sharded.py tests/test_sharded_cpp.py -x -q -m gpu -k "butterfly_parity or tiny_engine or config3 or config5 or host_pipeline or contract_async or multi_rhs or linearity or box2 or rank1 or sharded or fused" > gpurun_out/r2p_tests.log 2>&1
tail -3 gpurun_out/r2p_tests.log
