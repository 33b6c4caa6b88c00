set -x
mkdir -p gpurun_out
timeout 300 python tools/construct_once.py radon256 > gpurun_out/rd_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_panel -s 2 -c 1 -o gpurun_out/rd_panel_wide python tools/construct_once.py radon256 > gpurun_out/rd_ncu.log 2>&1
