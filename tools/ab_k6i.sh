# K6 assign: 1 (default) vs 2 / 4 prompts per thread per grid step (loads issued together).
# Results: gpurun_out/k6i/
set -u
O=gpurun_out/k6i
L=$PWD/paper_2502_06798_b200/lib
mkdir -p $O
for v in pas pas_k6i2 pas_k6i4; do
  PAS_LIB=$L/lib$v.so timeout 600 python -m pytest tests/test_gpu_redirect.py tests/test_gpu_parity.py -x -q -k "redirect or c1_parity or c2_parity or ragged" > $O/tests_$v.log 2>&1; echo "rc=$?" >> $O/tests_$v.log
  PAS_LIB=$L/lib$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k6_" --csv --log-file $O/ncu_stream_$v.csv python tools/bench_stream.py --reps 1 > /dev/null 2>&1
done
for rep in 1 2; do
  for v in pas pas_k6i2 pas_k6i4; do
    PAS_LIB=$L/lib$v.so timeout 300 python tools/bench_stream.py --reps 5 > $O/stream_${v}_$rep.json 2> /dev/null
  done
done
