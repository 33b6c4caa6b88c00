mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "bfp or butterfly_parity" > gpurun_out/r3c_tests.log 2>&1
tail -5 gpurun_out/r3c_tests.log
timeout 1500 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r3c_bench.json 2> gpurun_out/r3c_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r3c_bench.json').read().strip().splitlines()[-1])
print('value',d['value'],d['ms_per_step']); print(json.dumps(d['compressed_cores']))
"
tail -3 gpurun_out/r3c_bench.err
