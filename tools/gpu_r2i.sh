mkdir -p gpurun_out/r2i
python -m paper_2502_06798_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_plan.py -m gpu -q -s -k "not c4 and not c5 and not c3 and not fuzz and not dynamic" > gpurun_out/r2i/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2i/tests.log
timeout 300 python tools/c1_latency.py > gpurun_out/r2i/c1_latency.json 2>&1
REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/r2i/c1_launches_warm.csv python tools/c1_latency.py > gpurun_out/r2i/c1_ncu2.log 2>&1
tail -2 gpurun_out/r2i/tests.log
