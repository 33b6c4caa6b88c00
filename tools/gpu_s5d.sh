mkdir -p gpurun_out
OIOBF_DEBUG=1 OIOBF_SERIAL_SIDES=1 timeout 600 python tools/construct_dbg.py radon2d_n1024 1 > gpurun_out/s5d_serial.log 2>&1
grep -v "box side\|plan" gpurun_out/s5d_serial.log | tail -40
