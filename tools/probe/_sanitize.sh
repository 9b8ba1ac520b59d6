timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for tool in memcheck synccheck racecheck; do
  echo "== $tool"
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_$tool.log 2>&1; echo "rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Error|error" gpurun_out/san_$tool.log | head -8
done
