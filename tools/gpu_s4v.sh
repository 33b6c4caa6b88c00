mkdir -p gpurun_out
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/s4v_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/s4v_tests.log
timeout 600 python tools/apply_ab.py green_cubes_n256 - OIOBF_BOX_MMA=0 - > gpurun_out/s4v_ab.jsonl 2> gpurun_out/s4v_ab.err
cat gpurun_out/s4v_ab.jsonl
