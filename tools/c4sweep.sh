for v in "8 liblouiskv.so" "4 liblouiskv.so" "4 liblouiskv_minb2.so" "2 liblouiskv_minb2.so"; do
  set -- $v
  LOUISKV_LAYER_CL=$1 LOUISKV_LIB=$PWD/paper_2510_11292_b200/$2 timeout 600 python bench.py --config C4 --steps 32 --warmup 4 --no-cpu-baseline --no-l2-variant > gpurun_out/r02_c4_cl$1_$2.json 2>/dev/null
done
LOUISKV_LIB=$PWD/paper_2510_11292_b200/liblouiskv_minb2.so timeout 600 python bench.py --steps 64 --warmup 8 --no-cpu-baseline --no-l2-variant > gpurun_out/r02_c2_minb2.json 2>/dev/null
