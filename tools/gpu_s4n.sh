mkdir -p gpurun_out
timeout 600 python tools/apply_ab.py green_cubes_n256 - OIOBF_BOX_SPLIT_AT=0:0:2 OIOBF_BOX_SPLIT_AT=1:0:4 OIOBF_BOX_SPLIT_AT=0:1:2 OIOBF_BOX_SPLIT_AT=0:2:2 - > gpurun_out/s4n_ab.jsonl 2> gpurun_out/s4n_ab.err
cat gpurun_out/s4n_ab.jsonl; tail -3 gpurun_out/s4n_ab.err
