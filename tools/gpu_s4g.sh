mkdir -p gpurun_out
timeout 600 python tools/apply_ab.py green_cubes_n256 OIOBF_BOX_MMA=1 OIOBF_BOX_MMA=0 OIOBF_BOX_MMA=1 > gpurun_out/s4g_ab.jsonl 2> gpurun_out/s4g_ab.err
cat gpurun_out/s4g_ab.jsonl; tail -3 gpurun_out/s4g_ab.err
