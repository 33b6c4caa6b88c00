mkdir -p gpurun_out
python paper_2411_03029_b200/build.py >/dev/null 2>&1
OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_box -s 1 -c 1 -o gpurun_out/r2h_box_v1 python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/r2h_ncu1.log 2>&1
OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_box -s 4 -c 1 -o gpurun_out/r2h_box_p1 python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/r2h_ncu2.log 2>&1
tail -n 1 gpurun_out/r2h_ncu*.log
