mkdir -p gpurun_out
for c in green_cubes_n64 green_cubes_n256 radon256 radon2d_n1024; do
  timeout 600 python tools/panel_diag.py $c > gpurun_out/r4b_diag_$c.log 2>&1
  grep -h "panel-diag\|construct" gpurun_out/r4b_diag_$c.log
done
