mkdir -p gpurun_out
timeout 600 python tools/apply_ab.py green_cubes_n256 OIOBF_BOX_MMA=0 OIOBF_BOX_MMA=1 OIOBF_BOX_MMA=0 OIOBF_BOX_MMA=1 > gpurun_out/s4d_ab.jsonl 2> gpurun_out/s4d_ab.err
cat gpurun_out/s4d_ab.jsonl; tail -3 gpurun_out/s4d_ab.err
timeout 600 python tools/apply_ab.py green_cubes_n64 OIOBF_BOX_MMA=0 OIOBF_BOX_MMA=1 > gpurun_out/s4d_ab2.jsonl 2> gpurun_out/s4d_ab2.err
cat gpurun_out/s4d_ab2.jsonl; tail -3 gpurun_out/s4d_ab2.err
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "apply or contract or box or full_config" > gpurun_out/s4d_tests.log 2>&1; tail -5 gpurun_out/s4d_tests.log
