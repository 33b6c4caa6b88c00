set -x
mkdir -p gpurun_out
timeout 600 python tools/panel_bitcheck.py > gpurun_out/re_bitcheck.log 2>&1
tail -2 gpurun_out/re_bitcheck.log
OIOBF_DEBUG=1 timeout 900 python tools/construct_once.py radon2d_n1024 2>&1 | grep -v finish_level > gpurun_out/re_c5.log
timeout 600 python tools/construct_ab2.py green_cubes_n256 > gpurun_out/re_c3.jsonl 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "full_config or config3 or config5 or accuracy" -s > gpurun_out/re_fullcfg.log 2>&1
tail -15 gpurun_out/re_fullcfg.log
