mkdir -p gpurun_out
( time python bench.py --impl reference ) > gpurun_out/s4y_ref.json 2> gpurun_out/s4y_ref.err
echo "ref rc=$?"; tail -c 900 gpurun_out/s4y_ref.json; tail -3 gpurun_out/s4y_ref.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4y_smoke.log 2>&1; tail -2 gpurun_out/s4y_smoke.log
( time python bench.py ) > gpurun_out/s4y_bench.json 2> gpurun_out/s4y_bench.err
echo "bench rc=$?"; tail -3 gpurun_out/s4y_bench.err
