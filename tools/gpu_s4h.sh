mkdir -p gpurun_out
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/s4h_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/s4h_tests.log
python bench.py > gpurun_out/s4h_bench.json 2> gpurun_out/s4h_bench.err
echo "bench rc=$?"; tail -c 600 gpurun_out/s4h_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none -k regex:"k_box|k_gemv" -c 70 --csv --log-file gpurun_out/s4h_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/s4h_ncu.log 2>&1
tail -2 gpurun_out/s4h_ncu.log
OIOBF_BENCH_DIST=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/s4h_bench_w2_gloo.json 2> gpurun_out/s4h_bench_w2.err
tail -c 1500 gpurun_out/s4h_bench_w2_gloo.json; tail -3 gpurun_out/s4h_bench_w2.err
