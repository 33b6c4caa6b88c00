# 1000-sample accuracy of every BASELINE config with its accuracy ProxyStrategy (configs.ACCURACY_STRATEGY), final kernels
mkdir -p gpurun_out
: > gpurun_out/acc_final.jsonl
timeout 300 python tools/proxy_sweep.py green_plates_n64 1,4,17 >> gpurun_out/acc_final.jsonl 2>> gpurun_out/acc_final.err
timeout 300 python tools/proxy_sweep.py green_cubes_n64 1,3,23 >> gpurun_out/acc_final.jsonl 2>> gpurun_out/acc_final.err
timeout 300 python tools/proxy_sweep.py dft6_n16 1,3,17 >> gpurun_out/acc_final.jsonl 2>> gpurun_out/acc_final.err
timeout 1200 python tools/proxy_sweep.py radon2d_n1024 1,12,23 >> gpurun_out/acc_final.jsonl 2>> gpurun_out/acc_final.err
timeout 1800 python tools/proxy_sweep.py green_cubes_n256 1,6,27 >> gpurun_out/acc_final.jsonl 2>> gpurun_out/acc_final.err
cat gpurun_out/acc_final.jsonl
