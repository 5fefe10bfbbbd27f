# Streaming kernels k_select_s1 and k6_assign: resident-wave / capped grid with grid-stride loops
# (default) vs uncapped grids (g0).  Results: gpurun_out/grid/
set -u
O=gpurun_out/grid
L=$PWD/paper_2502_06798_b200/lib
mkdir -p $O
PAS_LIB=$L/libpas_g0.so timeout 600 python -m pytest tests/test_gpu_redirect.py tests/test_gpu_parity.py -x -q -k "redirect or c1_parity or c2_parity or ragged or merge or select" > $O/tests_g0.log 2>&1; echo "rc=$?" >> $O/tests_g0.log
for v in pas pas_g0; do
  PAS_LIB=$L/lib$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k6_assign|k_select" --csv --log-file $O/ncu_stream_$v.csv python tools/bench_stream.py --reps 1 > /dev/null 2>&1
done
for rep in 1 2; do
  for v in pas pas_g0; do
    PAS_LIB=$L/lib$v.so timeout 300 python tools/bench_stream.py --reps 5 > $O/stream_${v}_$rep.json 2> /dev/null
  done
done
