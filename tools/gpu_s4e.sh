mkdir -p gpurun_out
( time python -m pytest tests/test_sharded.py tests/test_sharded_cpp.py -x -q ) > gpurun_out/s4e_tests.log 2>&1
echo "sharded tests rc=$?"; tail -8 gpurun_out/s4e_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "variants or box2 or engines or rank" > gpurun_out/s4e_tests2.log 2>&1; tail -4 gpurun_out/s4e_tests2.log
timeout 600 python tools/apply_ab.py green_cubes_n256 OIOBF_BOX_MMA=0 OIOBF_BOX_MMA=1 > gpurun_out/s4e_ab.jsonl 2> gpurun_out/s4e_ab.err
cat gpurun_out/s4e_ab.jsonl; tail -3 gpurun_out/s4e_ab.err
