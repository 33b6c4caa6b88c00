mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
P="timeout 1500 python tools/proxy_sweep.py"
$P green_cubes_n256 1,4,23 1,4,25 > gpurun_out/r2k_cubes256.jsonl 2>&1
cat gpurun_out/r2k_cubes256.jsonl
$P radon2d_n1024 1,8,21 > gpurun_out/r2k_radon1024.jsonl 2>&1
cat gpurun_out/r2k_radon1024.jsonl
