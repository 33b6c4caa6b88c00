mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2y_build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y_smoke.log 2>&1; tail -2 gpurun_out/r2y_smoke.log
time timeout 1700 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2y_ref.json 2> gpurun_out/r2y_ref.err
tail -c 1200 gpurun_out/r2y_ref.json; tail -3 gpurun_out/r2y_ref.err
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2y_bench.json 2> gpurun_out/r2y_bench.err
tail -c 800 gpurun_out/r2y_bench.json; tail -3 gpurun_out/r2y_bench.err
