set -x
mkdir -p gpurun_out
python paper_2411_03029_b200/build.py
timeout 600 python tools/panel_ab.py green_cubes_n64,green_cubes_n256 '' 'OIOBF_PANEL_PR=128' > gpurun_out/r2e_ab.jsonl 2>&1
timeout 600 python tools/panel_ab.py radon256 '' 'OIOBF_PANEL_PR=64' 'OIOBF_PANEL_PR=96' >> gpurun_out/r2e_ab.jsonl 2>&1
cat gpurun_out/r2e_ab.jsonl
timeout 600 python tools/panel_ab.py radon2d_n1024 '' > gpurun_out/r2e_ab5.jsonl 2>&1
cat gpurun_out/r2e_ab5.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "butterfly_parity or sampled_slots or column_id or golden or register_cached" > gpurun_out/r2e_tests.log 2>&1
tail -5 gpurun_out/r2e_tests.log
