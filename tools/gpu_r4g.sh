mkdir -p gpurun_out
export OIOBF_SERIAL_SIDES=1
for sg in 1 0; do
  echo "== OIOBF_PANEL_STAGGER=$sg"
  for c in green_cubes_n256 green_cubes_n64; do OIOBF_PANEL_STAGGER=$sg timeout 300 python tools/construct_cfg.py $c 2 2>&1 | grep "^construct" | tail -1; done
done
timeout 300 python tools/panel_diag.py radon256 2>&1 | grep "^construct"
OIOBF_PANEL_STAGGER=0 timeout 300 python tools/panel_diag.py radon256 2>&1 | grep "^construct"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "butterfly_parity or sampled_slots or golden or bit_identical" > gpurun_out/r4g_tests.log 2>&1
tail -3 gpurun_out/r4g_tests.log
