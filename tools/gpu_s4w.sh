mkdir -p gpurun_out
timeout 600 python tools/apply_ab.py green_cubes_n256 OIOBF_BOX_MMA=2 OIOBF_BOX_MMA=4 OIOBF_BOX_MMA=2 OIOBF_BOX_MMA=4 > gpurun_out/s4w_ab.jsonl 2> gpurun_out/s4w_ab.err
cat gpurun_out/s4w_ab.jsonl; tail -3 gpurun_out/s4w_ab.err
timeout 600 python tools/apply_ab.py green_cubes_n64 OIOBF_BOX_MMA=2 OIOBF_BOX_MMA=4 OIOBF_BOX_MMA=2 OIOBF_BOX_MMA=4 > gpurun_out/s4w_ab2.jsonl 2> gpurun_out/s4w_ab2.err
cat gpurun_out/s4w_ab2.jsonl
