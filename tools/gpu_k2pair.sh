OUT=${OUT:-r2zd}
mkdir -p gpurun_out/$OUT
python -m paper_2502_06798_b200.build > /dev/null
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_cache.py -m gpu -q -x -k "not c4 and not c5_parity" > gpurun_out/$OUT/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/$OUT/tests.log
for v in "" epiw8; do
  L=$PWD/paper_2502_06798_b200/lib/libpas${v:+_$v}.so
  PAS_LIB=$L timeout 300 python tools/c1_latency.py > gpurun_out/$OUT/c1_latency_${v:-default}.json 2>&1
  PAS_LIB=$L REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/$OUT/c1_launches_warm_${v:-default}.csv python tools/c1_latency.py > /dev/null 2>&1
  PAS_LIB=$L timeout 900 python bench.py --config C5 --prompts 256 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/$OUT/bench_c5_256_${v:-default}.json 2> gpurun_out/$OUT/bench_c5_256_${v:-default}.err
done
tail -2 gpurun_out/$OUT/tests.log; cat gpurun_out/$OUT/c1_latency_*.json; for f in gpurun_out/$OUT/bench_c5_256_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d.get('clocks'))"; done
