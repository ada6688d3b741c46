#!/bin/bash
# compute-sanitizer over tools/sanitize.py: memcheck, racecheck, synccheck (summary lines kept)
out=${1:-gpurun_out/r02_sanitizer.txt}
: > $out
for tool in memcheck racecheck synccheck; do
  echo "=== $tool" >> $out
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/san_$tool.log 2>&1
  echo "exit $?" >> $out
  grep -E "^OK|complete|ERROR SUMMARY|RACECHECK SUMMARY|Error|error|hazard|Invalid" gpurun_out/san_$tool.log | head -60 >> $out
done
