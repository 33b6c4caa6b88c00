mkdir -p gpurun_out
timeout 600 python tools/apply_ab.py green_cubes_n256 - OIOBF_BOX_NT_AT=1:0:256 OIOBF_BOX_NT_AT=1:1:256 OIOBF_BOX_NT_AT=1:2:256 OIOBF_BOX_NT_AT=0:0:256 OIOBF_BOX_NT_AT=0:1:256 OIOBF_BOX_NT_AT=0:2:256 - > gpurun_out/s4q_ab.jsonl 2> gpurun_out/s4q_ab.err
cat gpurun_out/s4q_ab.jsonl; tail -3 gpurun_out/s4q_ab.err
