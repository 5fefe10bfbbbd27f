mkdir -p gpurun_out/r2l
python -m paper_2502_06798_b200.build > /dev/null
timeout 300 python tools/c1_latency.py > gpurun_out/r2l/c1_latency.json 2>&1
REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/r2l/c1_launches_warm.csv python tools/c1_latency.py > gpurun_out/r2l/c1_ncu2.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_k1_exact.py -m gpu -q -k "not c4 and not c5" > gpurun_out/r2l/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2l/tests.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2l/bench_c4.json 2> gpurun_out/r2l/bench_c4.err
timeout 600 python bench.py --config C2 --steps 2000 --no-cpu-baseline --no-e2e > gpurun_out/r2l/bench_c2.json 2> gpurun_out/r2l/bench_c2.err
timeout 600 python bench.py --config C3 --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/r2l/bench_c3.json 2> gpurun_out/r2l/bench_c3.err
