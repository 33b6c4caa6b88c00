PROBE_TAG=default python tools/e2e_probe.py > gpurun_out/probe.log 2>&1
OIOBF_NO_PDL=1 PROBE_TAG=nopdl python tools/e2e_probe.py >> gpurun_out/probe.log 2>&1
OIOBF_NO_GRAPH=1 PROBE_TAG=nograph python tools/e2e_probe.py >> gpurun_out/probe.log 2>&1
OIOBF_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/lq2.csv python tools/prof_apply.py --reps 1 > gpurun_out/nq2.log 2>&1
