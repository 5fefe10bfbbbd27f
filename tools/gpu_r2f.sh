mkdir -p gpurun_out/r2f
python -m paper_2502_06798_b200.build > /dev/null
timeout 1500 python -m pytest tests/test_gpu_redirect.py tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_dispatch.py tests/test_gpu_forecast.py tests/test_gpu_cache.py tests/test_gpu_multi.py -m gpu -q -s -k "not c4 and not c5 and not fuzz" > gpurun_out/r2f/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2f/tests.log
timeout 300 python tools/c1_latency.py > gpurun_out/r2f/c1_latency.json 2>&1
PAS_K2_PAIR_MAX_TILES=0 timeout 300 python tools/c1_latency.py > gpurun_out/r2f/c1_latency_nopair.json 2>&1
REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f/c1_launches.csv python tools/c1_latency.py > gpurun_out/r2f/c1_ncu.log 2>&1
REPS=20 PAS_K2_PAIR_MAX_TILES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f/c1_launches_nopair.csv python tools/c1_latency.py > gpurun_out/r2f/c1_ncu2.log 2>&1
CMD="python tools/bench_stream.py --reps 1"
timeout 600 python tools/bench_stream.py > gpurun_out/r2f/stream.json 2> gpurun_out/r2f/stream.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(normalize|merge|select|scan|tile|route|cls|offsets|bucket|plan|fc|small)|k6_" --csv --log-file gpurun_out/r2f/stream_launches.csv $CMD > gpurun_out/r2f/stream_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2f/stream_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k6_fused|k_cls_rank" -c 2 -o gpurun_out/r2f/k6k7_full $CMD > gpurun_out/r2f/ncu_full.log 2>&1
tail -3 gpurun_out/r2f/tests.log
