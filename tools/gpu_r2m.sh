mkdir -p gpurun_out
python paper_2411_03029_b200/build.py > /dev/null 2>&1
python tools/sanitize_driver.py > gpurun_out/r2m_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/r2m_plain.log; exit 1; }
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > gpurun_out/r2m_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r2m_$tool.log
done
