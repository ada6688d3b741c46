#!/bin/bash
# A/B: the default library vs a variant build (liblouiskv_$1.so), C2 and C4 bench lines, alternating
v=$1
for rep in 1 2; do
  for lib in liblouiskv.so liblouiskv_$v.so; do
    LOUISKV_LIB=$PWD/paper_2510_11292_b200/$lib timeout 600 python bench.py --steps 128 --warmup 8 --no-cpu-baseline --no-l2-variant > gpurun_out/ab_c2_${lib}_$rep.json 2>/dev/null
    LOUISKV_LIB=$PWD/paper_2510_11292_b200/$lib timeout 600 python bench.py --config C4 --steps 32 --warmup 4 --no-cpu-baseline --no-l2-variant > gpurun_out/ab_c4_${lib}_$rep.json 2>/dev/null
  done
done
