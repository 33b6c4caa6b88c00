set -x
mkdir -p gpurun_out
timeout 600 python tools/bigproxy_check.py > gpurun_out/sw2_bigproxy.txt 2>&1
P="timeout 1200 python tools/proxy_sweep.py"
$P radon256:4 1,6,21 1,8,21 1,12,21 1,8,23 > gpurun_out/sw2_radon256.jsonl 2>&1
$P green_cubes_n64 1,2,20 1,2,22 1,3,22 1,2,23 > gpurun_out/sw2_cubes64.jsonl 2>&1
$P radon512 1,3,17 1,8,21 > gpurun_out/sw2_radon512.jsonl 2>&1
$P green_cubes_n256 1,2,22 1,3,23 > gpurun_out/sw2_cubes256.jsonl 2>&1
