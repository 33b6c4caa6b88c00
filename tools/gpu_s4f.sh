mkdir -p gpurun_out
OIOBF_DEBUG=1 OIOBF_SERIAL_SIDES=1 timeout 300 python tools/construct_dbg.py green_cubes_n256 2 > gpurun_out/s4f_serial.log 2>&1
OIOBF_DEBUG=1 timeout 300 python tools/construct_dbg.py green_cubes_n256 2 > gpurun_out/s4f_conc.log 2>&1
grep -c . gpurun_out/s4f_serial.log gpurun_out/s4f_conc.log
timeout 600 nsys --version 2>/dev/null | head -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4f_construct_launches.csv python tools/construct_dbg.py green_cubes_n256 1 > gpurun_out/s4f_ncu.log 2>&1
tail -2 gpurun_out/s4f_ncu.log
