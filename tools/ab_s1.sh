# K3+K4 k_select_s1: loads in flight per thread (PAS_S1_UNROLL 1 / 2 / 4 default / 8) at 64M prompts.
set -u
O=gpurun_out/s1
L=$PWD/paper_2502_06798_b200/lib
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_redirect.py -q -x -k "c1_parity or c2_parity or cold or redirect or many or widths" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
for v in pas_s1u1 pas_s1u2 pas pas_s1u8; do
  PAS_LIB=$L/lib$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_select" --csv --log-file $O/ncu_$v.csv python tools/bench_stream.py --reps 1 > /dev/null 2>&1
  PAS_LIB=$L/lib$v.so timeout 300 python tools/bench_stream.py --reps 5 > $O/stream_$v.json 2> $O/stream_$v.err
done
