mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
OIOBF_DEBUG=1 timeout 300 python tools/prof_apply.py --config green_cubes_n256 --reps 1 2>&1 | grep -E "box side" | head
timeout 1200 python tools/panel_ab.py green_cubes_n64,green_cubes_n256,dft6_n16,green_plates_n64 '' 'OIOBF_SERIAL_SIDES=1' > gpurun_out/r2w_pab.jsonl 2>&1; cat gpurun_out/r2w_pab.jsonl
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2w_tests.log 2>&1
tail -3 gpurun_out/r2w_tests.log
OIOBF_SERIAL_SIDES=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_panel -s 3 -c 1 -o gpurun_out/r2w_panel_c5l3 python tools/construct_once.py radon2d_n1024 > gpurun_out/r2w_ncu.log 2>&1
tail -2 gpurun_out/r2w_ncu.log
