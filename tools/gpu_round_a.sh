set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/ra_parity.log 2>&1
tail -3 gpurun_out/ra_parity.log
for c in green_plates_n64 green_cubes_n64 green_cubes_n256; do
  timeout 600 python tools/construct_ab2.py $c >> gpurun_out/ra_ab.jsonl 2>&1
  OIOBF_PANEL_LEGACY=1 timeout 600 python tools/construct_ab2.py $c >> gpurun_out/ra_ab.jsonl 2>&1
done
timeout 900 python tools/construct_ab2.py green_cubes_n64 3 23 >> gpurun_out/ra_ab.jsonl 2>&1
timeout 900 python tools/construct_ab2.py green_cubes_n256 3 23 >> gpurun_out/ra_ab.jsonl 2>&1
