# K1 occupancy / dependency-chain variants (PAS_K1_MINB resident CTAs, PAS_K1_ACC partial sums):
# cache insert at 1M fp32 rows and the in-pipeline normalise at C3 / C4.  Results: gpurun_out/k1b/
set -u
O=gpurun_out/k1b
L=$PWD/paper_2502_06798_b200/lib
mkdir -p $O
for v in k1m4a2 k1m3a2; do
  PAS_LIB=$L/libpas_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or c1_parity or cold or ragged or bf16 or c2_parity" > $O/tests_$v.log 2>&1; echo "rc=$?" >> $O/tests_$v.log
done
for rep in 1 2; do
  for v in pas pas_k1m3a2 pas_k1m4a1 pas_k1m4a2 pas_k1m4a4; do
    PAS_LIB=$L/lib$v.so timeout 300 python tools/bench_stream.py --reps 5 > $O/stream_${v}_$rep.json 2> $O/stream_${v}_$rep.err
    PAS_LIB=$L/lib$v.so timeout 300 python bench.py --config C3 --steps 30 --no-cpu-baseline --no-e2e > $O/c3_${v}_$rep.json 2> $O/c3_${v}_$rep.err
  done
done
for v in pas pas_k1m4a2; do
  PAS_LIB=$L/lib$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_normalize -s 306 -c 4 --csv --log-file $O/ncu_c4_$v.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
