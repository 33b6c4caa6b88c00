set -x
mkdir -p gpurun_out
python paper_2411_03029_b200/build.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tsqr -s 2 -c 1 -o gpurun_out/r2c_tsqr_c3 python tools/construct_once.py green_cubes_n256 > gpurun_out/r2c_ncu1.log 2>&1
OIOBF_PANEL_OLD=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_panel -s 2 -c 1 -o gpurun_out/r2c_panel_c3 python tools/construct_once.py green_cubes_n256 > gpurun_out/r2c_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tsqr -s 2 -c 1 -o gpurun_out/r2c_tsqr_r256 python tools/construct_once.py radon256 > gpurun_out/r2c_ncu3.log 2>&1
tail -3 gpurun_out/r2c_ncu*.log
