# K1 grid: resident-CTA grid with grid-stride rows (default) vs one CTA per 8 rows (k1g0), and
# the latter at 8 CTAs/SM (k1g0m8).  Results: gpurun_out/k1g/
set -u
O=gpurun_out/k1g
L=$PWD/paper_2502_06798_b200/lib
mkdir -p $O
for v in k1g0 k1g0m8; do
  PAS_LIB=$L/libpas_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_parity or ragged or bf16 or c2_parity or widths" > $O/tests_$v.log 2>&1; echo "rc=$?" >> $O/tests_$v.log
done
for v in pas pas_k1g0 pas_k1g0m8; do
  PAS_LIB=$L/lib$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_normalize -s 153 -c 4 --csv --log-file $O/ncu_c4_$v.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
for rep in 1 2; do
  for v in pas pas_k1g0 pas_k1g0m8; do
    PAS_LIB=$L/lib$v.so timeout 300 python tools/bench_stream.py --reps 5 > $O/stream_${v}_$rep.json 2> $O/stream_${v}_$rep.err
  done
done
