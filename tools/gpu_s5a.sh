mkdir -p gpurun_out
timeout 1500 python tools/panel_ab.py radon256,radon2d_n1024 'OIOBF_PANEL_PIPE=0' '' > gpurun_out/s5e_ab.jsonl 2> gpurun_out/s5e_ab.err
cat gpurun_out/s5e_ab.jsonl; tail -3 gpurun_out/s5e_ab.err
