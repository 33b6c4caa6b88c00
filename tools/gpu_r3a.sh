mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
timeout 600 python tools/apply_ab.py green_cubes_n256 - > gpurun_out/r3a_ab3.jsonl 2>&1; cat gpurun_out/r3a_ab3.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv -k regex:"k_box|k_gemv" --log-file gpurun_out/r3a_launches.csv python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/r3a_ncu.log 2>&1
python tools/launch_list.py gpurun_out/r3a_launches.csv x | head -12
