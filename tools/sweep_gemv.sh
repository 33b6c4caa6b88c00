for cfg in "OIOBF_GEMV_NO_TMA=1" "OIOBF_TMA_STAGES=8" "OIOBF_TMA_STAGES=16" "OIOBF_TMA_CTAS_PER_SM=2 OIOBF_TMA_STAGES=8" "OIOBF_TMA_CTAS_PER_SM=3 OIOBF_TMA_STAGES=8"; do
  echo "== $cfg"
  env $cfg python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.load(sys.stdin); print(round(j['ms_per_step']*1000,1), 'us/step; core', round(j['roofline']['launch_ms']*1000,1), 'us frac', round(j['roofline']['frac'],3))"
done
