mkdir -p gpurun_out
export OIOBF_SERIAL_SIDES=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wtsqr -s 2 -c 1 -o gpurun_out/r4f_wtsqr python tools/construct_cfg.py green_cubes_n256 1 > gpurun_out/r4f_ncu.log 2>&1
tail -3 gpurun_out/r4f_ncu.log
