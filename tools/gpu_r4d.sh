mkdir -p gpurun_out
export OIOBF_SERIAL_SIDES=1
for c in green_cubes_n256 radon256; do
  timeout 600 python tools/panel_diag.py $c > gpurun_out/r4d_diag_$c.log 2>&1
  grep -h "panel-diag\|construct" gpurun_out/r4d_diag_$c.log
done
OIOBF_PANEL_NARROW_RC=0 timeout 600 python tools/panel_diag.py green_cubes_n256 2>&1 | grep -h "panel-diag\|construct"
