set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python tools/prof_apply.py --reps 2 > gpurun_out/p_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_graph.csv python tools/prof_apply.py --reps 2 > gpurun_out/ncu_l.log 2>&1
python tools/prof_apply.py --reps 1 > gpurun_out/p_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 0 -c 1 -o gpurun_out/prof_gemv_final python tools/prof_apply.py --reps 1 > gpurun_out/ncu_g.log 2>&1
python tools/prof_apply.py --construct-only > gpurun_out/p_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_panel -s 0 -c 1 -o gpurun_out/prof_panel_final python tools/prof_apply.py --construct-only > gpurun_out/ncu_p.log 2>&1
