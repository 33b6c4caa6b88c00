set -x
mkdir -p gpurun_out
python paper_2411_03029_b200/build.py
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_panel -s 2 -c 1 -o gpurun_out/r2f_panel_r256 python tools/construct_once.py radon256 > gpurun_out/r2f_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_panel -s 2 -c 1 -o gpurun_out/r2f_panel_c3 python tools/construct_once.py green_cubes_n256 > gpurun_out/r2f_ncu2.log 2>&1
tail -n 3 gpurun_out/r2f_ncu1.log gpurun_out/r2f_ncu2.log
