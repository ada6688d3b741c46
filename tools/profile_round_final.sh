#!/bin/bash
# End-of-round evidence with the final code: full GPU suite, smoke, bench lines (C2, C3, C4, C5 share),
# the reference arm, the ncu launch list of the C2 bench command, --set full captures of the layer
# kernel (C2, steady-state launches) and the full-cache attention (C2). Outputs under gpurun_out/fin_*.
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fin_gputest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/fin_c2.json 2> gpurun_out/fin_c2.err
timeout 900 python bench.py --config C3 > gpurun_out/fin_c3.json 2> gpurun_out/fin_c3.err
timeout 1200 python bench.py --config C4 --steps 64 --warmup 8 > gpurun_out/fin_c4.json 2> gpurun_out/fin_c4.err
timeout 1500 python bench.py --config C5 --shard-of 8 --batch 16 --steps 64 --warmup 8 --no-cpu-baseline > gpurun_out/fin_c5.json 2> gpurun_out/fin_c5.err
timeout 900 python bench.py --impl reference --steps 16 --warmup 3 > gpurun_out/fin_ref_c2.json 2> gpurun_out/fin_ref_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c2.csv python bench.py --steps 32 --warmup 4 --no-cpu-baseline --no-l2-variant > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 400 -c 8 -o gpurun_out/fin_full_lk_c2 python tools/probe_step.py --config C2 --layer --taus default --steps 20 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_full -s 10 -c 2 -o gpurun_out/fin_full_fa_c2 python tools/probe_step.py --config C2 --layer --taus default --steps 8 > /dev/null 2>&1
ls -la gpurun_out/ | grep fin_
