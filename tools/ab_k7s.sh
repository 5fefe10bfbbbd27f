# K7 batch lists: staged per-instance runs (default) vs the direct scatter (libpas_nostage.so).
set -u
O=gpurun_out/k7s
L=$PWD/paper_2502_06798_b200/lib
mkdir -p $O
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dispatch.py tests/test_gpu_forecast.py tests/test_gpu_cache.py tests/test_gpu_redirect.py -q -x -k "not c4_parity and not c5_load" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
for v in pas pas_nostage; do
  PAS_LIB=$L/lib$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_cls" --csv --log-file $O/ncu_$v.csv python tools/bench_stream.py --reps 1 > /dev/null 2>&1
done
