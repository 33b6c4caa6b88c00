set -x
mkdir -p gpurun_out
for c in green_cubes_n64 green_cubes_n256; do
  timeout 600 python tools/construct_ab2.py $c >> gpurun_out/rb_ab.jsonl 2>&1
done
timeout 300 python tools/construct_once.py green_cubes_n64 > gpurun_out/rb_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tsqr -s 1 -c 1 -o gpurun_out/rb_tsqr python tools/construct_once.py green_cubes_n64 > gpurun_out/rb_ncu.log 2>&1
