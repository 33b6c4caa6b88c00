mkdir -p gpurun_out
timeout 600 python tools/apply_ab.py green_cubes_n256 OIOBF_BOX_PF=0 OIOBF_BOX_PF=1 OIOBF_BOX_PF=2 OIOBF_BOX_PF=0 OIOBF_BOX_PF=1 OIOBF_BOX_PF=2 > gpurun_out/s5g_ab.jsonl 2> gpurun_out/s5g_ab.err
cat gpurun_out/s5g_ab.jsonl; tail -3 gpurun_out/s5g_ab.err
timeout 600 python tools/apply_ab.py green_cubes_n64 OIOBF_BOX_PF=0 OIOBF_BOX_PF=1 OIOBF_BOX_PF=2 > gpurun_out/s5g_ab2.jsonl 2> gpurun_out/s5g_ab2.err
cat gpurun_out/s5g_ab2.jsonl
