#!/bin/bash
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 40 python tools/sanitize.py > gpurun_out/r02_racecheck_full.txt 2>&1
echo "exit $?" >> gpurun_out/r02_racecheck_full.txt
