set -x
mkdir -p gpurun_out
python paper_2411_03029_b200/build.py
timeout 900 python tools/tsqr_ab.py green_cubes_n64,radon256,green_cubes_n256 > gpurun_out/r2d_ab.jsonl 2>&1
cat gpurun_out/r2d_ab.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "butterfly_parity or sampled_slots or column_id or golden" > gpurun_out/r2d_tests.log 2>&1
tail -5 gpurun_out/r2d_tests.log
