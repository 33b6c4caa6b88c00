mkdir -p gpurun_out
OIOBF_DEBUG=1 timeout 300 python tools/prof_apply.py --config green_cubes_n256 --reps 1 2>&1 | grep "box side" > gpurun_out/s4o_plan.log
cat gpurun_out/s4o_plan.log
timeout 600 python tools/apply_ab.py green_cubes_n256 OIOBF_BOX_A16=1 OIOBF_BOX_A16=2 OIOBF_BOX_A16=1 OIOBF_BOX_A16=2 > gpurun_out/s4o_ab.jsonl 2> gpurun_out/s4o_ab.err
cat gpurun_out/s4o_ab.jsonl; tail -3 gpurun_out/s4o_ab.err
timeout 600 python tools/apply_ab.py green_cubes_n64 OIOBF_BOX_A16=1 OIOBF_BOX_A16=2 > gpurun_out/s4o_ab2.jsonl 2> gpurun_out/s4o_ab2.err
cat gpurun_out/s4o_ab2.jsonl
