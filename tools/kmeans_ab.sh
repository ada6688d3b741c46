for rep in 1 2; do for lib in liblouiskv.so liblouiskv_scw.so; do for c in C2 C4; do
LOUISKV_LIB=$PWD/paper_2510_11292_b200/$lib timeout 300 python tools/probe_kmeans_phases.py $c 3 >> gpurun_out/v7_km.txt 2>>gpurun_out/v7_km.err
done; done; done
