mkdir -p gpurun_out
timeout 900 python tools/panel_ab.py green_cubes_n256,green_cubes_n64 '' 'OIOBF_PANEL_PIPE=2' '' 'OIOBF_PANEL_PIPE=2' > gpurun_out/s5a_ab.jsonl 2> gpurun_out/s5a_ab.err
cat gpurun_out/s5a_ab.jsonl; tail -3 gpurun_out/s5a_ab.err
