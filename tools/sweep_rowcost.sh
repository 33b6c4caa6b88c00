for k in 0 64 256 1024 100000000; do OIOBF_GEMV_ROW_COST=$k PROBE_TAG=k$k python tools/e2e_probe.py >> gpurun_out/rowcost.log 2>&1; done
