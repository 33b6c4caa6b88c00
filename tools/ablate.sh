for ab in "" "3" "1" "4" "34" "134"; do
  echo "== skip kinds '$ab' (1=gemv 3=box 4=sum)"
  OIOBF_ABLATE=$ab python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.load(sys.stdin); print(round(j['ms_per_step']*1000,1), 'us/step (L2 flushed); graph', round(j['roofline']['phase_ms']['graph_total']*1000,1),'us warm')"
done
