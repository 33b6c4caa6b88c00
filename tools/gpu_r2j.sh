mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
OIOBF_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 0 -c 1 -o gpurun_out/r2j_gemv_c3 python tools/prof_apply.py --config green_cubes_n256 --reps 1 > gpurun_out/r2j_ncu1.log 2>&1
tail -n 1 gpurun_out/r2j_ncu1.log
