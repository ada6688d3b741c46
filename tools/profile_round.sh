#!/bin/bash
# Round-2 evidence: bench lines (C2 default, C3, C4), the reference arm, ncu launch lists of bench
# commands, ncu --set full captures of the dominant kernels. Outputs under gpurun_out/r02_*.
set -x
timeout 900 python bench.py > gpurun_out/r02_final_c2.json 2> gpurun_out/r02_final_c2.err
timeout 900 python bench.py --config C3 > gpurun_out/r02_final_c3.json 2> gpurun_out/r02_final_c3.err
timeout 1200 python bench.py --config C4 --steps 64 --warmup 8 > gpurun_out/r02_final_c4.json 2> gpurun_out/r02_final_c4.err
timeout 900 python bench.py --impl reference --steps 16 --warmup 2 > gpurun_out/r02_final_ref_c2.json 2> gpurun_out/r02_final_ref_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c2.csv python bench.py --steps 32 --warmup 4 --no-cpu-baseline --no-l2-variant > gpurun_out/r02_launches_c2.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c4.csv python bench.py --config C4 --steps 16 --warmup 4 --no-cpu-baseline --no-l2-variant > gpurun_out/r02_launches_c4.json 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 200 -c 6 -o gpurun_out/r02_full_lk_c2 python tools/probe_step.py --config C2 --layer --taus default --steps 16 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_full -s 4 -c 2 -o gpurun_out/r02_full_fa_c4 python tools/probe_step.py --config C4 --layer --taus default --steps 4 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 200 -c 4 -o gpurun_out/r02_full_lk_c4 python tools/probe_step.py --config C4 --layer --taus default --steps 12 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kmeans_assign -s 2 -c 1 -o gpurun_out/r02_full_km_c2 python tools/probe_kmeans.py > /dev/null 2>&1
ls -la gpurun_out/
