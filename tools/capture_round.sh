# Round artifacts: bench (both arms), launch list, ncu full captures of the
# GEMV and the first box launch (each only after the same command ran clean).
set -x
TAG=${TAG:-r1b}
python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
python tools/prof_apply.py --reps 2 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/prof_apply.py --reps 2 > gpurun_out/${TAG}_ncu_l.log 2>&1
OIOBF_NO_GRAPH=1 python tools/prof_apply.py --reps 1 > gpurun_out/${TAG}_plain2.log 2>&1 && \
OIOBF_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 0 -c 1 -o gpurun_out/${TAG}_gemv python tools/prof_apply.py --reps 1 > gpurun_out/${TAG}_ncu_g.log 2>&1
OIOBF_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:k_box -s 0 -c 1 -o gpurun_out/${TAG}_box python tools/prof_apply.py --reps 1 > gpurun_out/${TAG}_ncu_b.log 2>&1
