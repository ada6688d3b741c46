#!/bin/bash
# Late round-2 evidence: full GPU suite, smoke, bench lines (C2 default, C3, C4), the reference arm,
# the ncu launch list of the C2 bench command. Outputs under gpurun_out/s3_*.
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s3_gputest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/s3_c2.json 2> gpurun_out/s3_c2.err
timeout 900 python bench.py --config C3 > gpurun_out/s3_c3.json 2> gpurun_out/s3_c3.err
timeout 1200 python bench.py --config C4 --steps 64 --warmup 8 > gpurun_out/s3_c4.json 2> gpurun_out/s3_c4.err
timeout 900 python bench.py --impl reference --steps 16 --warmup 3 > gpurun_out/s3_ref_c2.json 2> gpurun_out/s3_ref_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_launches_c2.csv python bench.py --steps 32 --warmup 4 --no-cpu-baseline --no-l2-variant > gpurun_out/s3_launches_c2.json 2>/dev/null
ls -la gpurun_out/ | grep s3_
