mkdir -p gpurun_out
export OIOBF_SERIAL_SIDES=1 OIOBF_DEBUG=1
timeout 300 python tools/construct_cfg.py green_cubes_n256 2 > gpurun_out/r4c_c3.log 2>&1
grep -h "construct" gpurun_out/r4c_c3.log | tail -12
timeout 300 python tools/construct_cfg.py radon2d_n1024 1 > gpurun_out/r4c_c5.log 2>&1
grep -h "construct" gpurun_out/r4c_c5.log | tail -12
