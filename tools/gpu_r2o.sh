mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
V="- OIOBF_BOX_NT=128 OIOBF_BOX_NT=128,OIOBF_BOX_STAGE=0 OIOBF_BOX_STAGE=0"
timeout 600 python tools/apply_ab.py green_cubes_n256 $V > gpurun_out/r2o_ab3.jsonl 2>&1; cat gpurun_out/r2o_ab3.jsonl
timeout 600 python tools/apply_ab.py green_cubes_n64 $V > gpurun_out/r2o_ab2.jsonl 2>&1; cat gpurun_out/r2o_ab2.jsonl
timeout 600 python tools/apply_ab.py green_plates_n64 $V > gpurun_out/r2o_ab1.jsonl 2>&1; cat gpurun_out/r2o_ab1.jsonl
