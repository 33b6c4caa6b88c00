mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
timeout 2700 python tools/proxy_sweep.py green_cubes_n256 1,6,27 > gpurun_out/r2t_cubes256.jsonl 2>&1
cat gpurun_out/r2t_cubes256.jsonl
