mkdir -p gpurun_out
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/fin_tests.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/fin_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; tail -1 gpurun_out/fin_smoke.log
python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
echo "bench rc=$?"
