# K7 rank kernel register budget (class + rank packed in one register per row; PAS_K7_MINB resident
# CTAs): 64M-prompt streaming bench and routing parity.  Results: gpurun_out/k7m/
set -u
O=gpurun_out/k7m
L=$PWD/paper_2502_06798_b200/lib
mkdir -p $O
for v in k7m5 k7m6; do
  PAS_LIB=$L/libpas_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dispatch.py tests/test_gpu_redirect.py -x -q -k "c1_parity or c2_parity or many or ragged or dispatch or redirect or uniform or virtual" > $O/tests_$v.log 2>&1; echo "rc=$?" >> $O/tests_$v.log
done
for rep in 1 2; do
  for v in pas_k7m4 pas_k7m5 pas_k7m6; do
    PAS_LIB=$L/lib$v.so timeout 300 python tools/bench_stream.py --reps 5 > $O/stream_${v}_$rep.json 2> $O/stream_${v}_$rep.err
  done
done
for v in pas_k7m4 pas_k7m5 pas_k7m6; do
  PAS_LIB=$L/lib$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_cls" --csv --log-file $O/ncu_$v.csv python tools/bench_stream.py --reps 1 > /dev/null 2>&1
done
