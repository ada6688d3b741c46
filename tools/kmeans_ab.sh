#!/bin/bash
# A/B of k-means kernels: the default library vs liblouiskv_$1.so, prefill-timer phases at C2 and C4
v=$1; out=${2:-gpurun_out/km_ab.txt}
for rep in 1 2; do for lib in liblouiskv.so liblouiskv_$v.so; do for c in C2 C4; do
LOUISKV_LIB=$PWD/paper_2510_11292_b200/$lib timeout 300 python tools/probe_kmeans_phases.py $c 3 >> $out 2>>$out.err
done; done; done
