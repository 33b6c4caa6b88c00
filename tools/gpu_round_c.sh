set -x
mkdir -p gpurun_out
timeout 600 python tools/panel_bitcheck.py > gpurun_out/rc_bitcheck.log 2>&1
tail -3 gpurun_out/rc_bitcheck.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/rc_parity.log 2>&1
tail -2 gpurun_out/rc_parity.log
OIOBF_DEBUG=1 timeout 900 python tools/construct_once.py radon2d_n1024 > gpurun_out/rc_c5_rs.log 2>&1
OIOBF_DEBUG=1 OIOBF_PAIR_ABSORB=1 timeout 900 python tools/construct_once.py radon2d_n1024 > gpurun_out/rc_c5_pair.log 2>&1
