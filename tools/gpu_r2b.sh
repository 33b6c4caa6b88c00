set -x
mkdir -p gpurun_out
python paper_2411_03029_b200/build.py
timeout 900 python tools/tsqr_ab.py cubes32,green_cubes_n64,green_plates_n64,radon256,green_cubes_n256 > gpurun_out/r2b_ab.jsonl 2>&1
cat gpurun_out/r2b_ab.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "butterfly_parity or sampled_slots or config3 or column_id or dense_accuracy or catalog or accuracy_gate or golden" > gpurun_out/r2b_tests.log 2>&1
tail -15 gpurun_out/r2b_tests.log
timeout 600 python tools/tsqr_ab.py radon2d_n1024 > gpurun_out/r2b_ab5.jsonl 2>&1
cat gpurun_out/r2b_ab5.jsonl
