set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/sw1_smi.txt
P="timeout 900 python tools/proxy_sweep.py"
$P green_plates_n64 1,3,17 1,4,17 1,3,18 1,4,18 1,6,17 0,3,17 > gpurun_out/sw1_plates.jsonl 2>&1
$P green_cubes_n64 1,3,17 1,3,19 1,3,21 1,4,21 1,3,23 > gpurun_out/sw1_cubes64.jsonl 2>&1
$P radon256:4 1,3,17 1,3,19 1,3,21 1,6,21 0,3,17 > gpurun_out/sw1_radon256.jsonl 2>&1
$P green_cubes_n256 1,3,17 1,3,19 1,3,21 > gpurun_out/sw1_cubes256.jsonl 2>&1
$P radon2d_n1024 1,3,19 > gpurun_out/sw1_radon1024.jsonl 2>&1
