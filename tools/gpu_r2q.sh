mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_box|k_gemv" --log-file gpurun_out/r2q_launches.csv python tools/prof_apply.py --config green_cubes_n256 --reps 2 > gpurun_out/r2q_ncu.log 2>&1
OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_box -s 4 -c 1 -o gpurun_out/r2q_box_p1 python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/r2q_ncu2.log 2>&1
OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_box -s 1 -c 1 -o gpurun_out/r2q_box_v1 python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/r2q_ncu3.log 2>&1
