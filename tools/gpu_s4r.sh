mkdir -p gpurun_out
timeout 600 python tools/apply_ab.py green_cubes_n256 - OIOBF_BOX6_KB=36 OIOBF_BOX6_KB=51 OIOBF_BOX6_KB=200 - > gpurun_out/s4r_ab.jsonl 2> gpurun_out/s4r_ab.err
cat gpurun_out/s4r_ab.jsonl; tail -3 gpurun_out/s4r_ab.err
timeout 600 python tools/apply_ab.py green_cubes_n64 - OIOBF_BOX6_KB=36 > gpurun_out/s4r_ab2.jsonl 2> gpurun_out/s4r_ab2.err
cat gpurun_out/s4r_ab2.jsonl
timeout 600 python tools/apply_ab.py radon2d_n1024 - OIOBF_BOX6_KB=36 > gpurun_out/s4r_ab3.jsonl 2> gpurun_out/s4r_ab3.err
cat gpurun_out/s4r_ab3.jsonl
