timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | grep -E "^E|passed|failed|rel err" | head -30 > gpurun_out/tq.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bq.json 2> gpurun_out/bq.err
OIOBF_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/lq.csv python tools/prof_apply.py --reps 1 > gpurun_out/nq.log 2>&1
