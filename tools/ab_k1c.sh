# K1 variants: 4 resident CTAs holding the row (m4r0) vs re-reading the row for the stores at 5 / 6
# resident CTAs (m5r1, m6r1).  Results: gpurun_out/k1c/
set -u
O=gpurun_out/k1c
L=$PWD/paper_2502_06798_b200/lib
mkdir -p $O
for v in k1m6r1 k1m5r1; do
  PAS_LIB=$L/libpas_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or c1_parity or cold or ragged or bf16 or c2_parity or widths" > $O/tests_$v.log 2>&1; echo "rc=$?" >> $O/tests_$v.log
done
for rep in 1 2; do
  for v in pas pas_k1m4r0 pas_k1m5r1 pas_k1m6r1; do
    PAS_LIB=$L/lib$v.so timeout 300 python tools/bench_stream.py --reps 5 > $O/stream_${v}_$rep.json 2> $O/stream_${v}_$rep.err
    PAS_LIB=$L/lib$v.so timeout 300 python bench.py --config C3 --steps 30 --no-cpu-baseline --no-e2e > $O/c3_${v}_$rep.json 2> $O/c3_${v}_$rep.err
  done
done
for v in pas_k1m4r0 pas_k1m6r1; do
  PAS_LIB=$L/lib$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_normalize -s 153 -c 4 --csv --log-file $O/ncu_c4_$v.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
