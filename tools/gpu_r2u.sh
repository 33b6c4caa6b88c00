mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
OIOBF_DEBUG=1 timeout 300 python tools/prof_apply.py --config green_cubes_n256 --reps 1 2>&1 | grep -E "box side|rror" | head
timeout 600 python tools/apply_ab.py green_cubes_n256 - OIOBF_BOX_PIPE=0 > gpurun_out/r2u_ab3.jsonl 2>&1; cat gpurun_out/r2u_ab3.jsonl
timeout 600 python tools/apply_ab.py green_cubes_n64 - > gpurun_out/r2u_ab2.jsonl 2>&1; cat gpurun_out/r2u_ab2.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "butterfly_parity or tiny_engine or config3 or host_pipeline or contract_async or multi_rhs or linearity or cta_variants" > gpurun_out/r2u_tests.log 2>&1
tail -3 gpurun_out/r2u_tests.log
timeout 900 python tools/panel_ab.py green_cubes_n64,green_cubes_n256 '' 'OIOBF_PANEL_NARROW_RC=1' 'OIOBF_PANEL_NARROW_RC=1;OIOBF_PANEL_PR=128' > gpurun_out/r2u_pab.jsonl 2>&1; cat gpurun_out/r2u_pab.jsonl
