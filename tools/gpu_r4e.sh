mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "butterfly_parity or sampled_slots or golden" > gpurun_out/r4e_tests.log 2>&1
tail -5 gpurun_out/r4e_tests.log
export OIOBF_SERIAL_SIDES=1
for wt in 16 0; do
  echo "== OIOBF_PANEL_WT=$wt"
  OIOBF_PANEL_WT=$wt timeout 300 python tools/construct_cfg.py green_cubes_n256 2 2>&1 | grep "^construct"
  OIOBF_PANEL_WT=$wt timeout 300 python tools/construct_cfg.py green_cubes_n64 2 2>&1 | grep "^construct"
done
OIOBF_PANEL_PR=32 timeout 300 python tools/construct_cfg.py green_cubes_n256 2 2>&1 | grep "^construct"
