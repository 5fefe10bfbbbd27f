mkdir -p gpurun_out/r2e
python -m paper_2502_06798_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_redirect.py tests/test_gpu_graph.py -m gpu -q -s > gpurun_out/r2e/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2e/tests.log
timeout 300 python tools/c1_latency.py > gpurun_out/r2e/c1_latency.json 2>&1
REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e/c1_launches.csv python tools/c1_latency.py > gpurun_out/r2e/c1_ncu.log 2>&1
timeout 600 python tools/bench_n2.py > gpurun_out/r2e/bench_n2.json 2> gpurun_out/r2e/bench_n2.err
CMD="python tools/bench_stream.py --reps 1"
timeout 600 python tools/bench_stream.py > gpurun_out/r2e/stream.json 2> gpurun_out/r2e/stream.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(normalize|merge|select|scan|tile|route|cls|offsets|bucket|plan|fc|small)|k6_" --csv --log-file gpurun_out/r2e/stream_launches.csv $CMD > gpurun_out/r2e/stream_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2e/stream_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k6_fused" -c 1 -o gpurun_out/r2e/k6_fused_full $CMD > gpurun_out/r2e/ncu_full.log 2>&1
tail -3 gpurun_out/r2e/tests.log
