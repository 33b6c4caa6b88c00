set -x
mkdir -p gpurun_out
python paper_2411_03029_b200/build.py
timeout 300 python tools/prof_apply.py --config green_cubes_n256 --reps 2 > gpurun_out/r2g_plain.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_box|k_gemv" --log-file gpurun_out/r2g_launches.csv python tools/prof_apply.py --config green_cubes_n256 --reps 2 > gpurun_out/r2g_ncu.log 2>&1
OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_box -s 0 -c 1 -o gpurun_out/r2g_box_v0 python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/r2g_ncu2.log 2>&1
OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_box -s 5 -c 1 -o gpurun_out/r2g_box_u0 python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/r2g_ncu3.log 2>&1
tail -n 2 gpurun_out/r2g_*.log
