mkdir -p gpurun_out/r2c
python -m paper_2502_06798_b200.build > /dev/null
timeout 1500 python -m pytest tests/test_gpu_graph.py tests/test_gpu_redirect.py tests/test_gpu_multi.py tests/test_gpu_plan.py tests/test_gpu_parity.py tests/test_gpu_forecast.py tests/test_gpu_cache.py tests/test_gpu_dispatch.py -m gpu -q -s -k "not c4 and not c5 and not c3_parity_full" > gpurun_out/r2c/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2c/tests.log
for g in "" "--graph"; do
  timeout 300 python bench.py --config C1 --steps 2000 --no-cpu-baseline --no-e2e $g > gpurun_out/r2c/bench_c1$g.json 2>&1
  timeout 300 python bench.py --config C2 --steps 2000 --no-cpu-baseline --no-e2e $g > gpurun_out/r2c/bench_c2$g.json 2>&1
done
CMD="python tools/bench_stream.py --reps 1"
timeout 600 python tools/bench_stream.py > gpurun_out/r2c/stream.json 2> gpurun_out/r2c/stream.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(normalize|merge|select|scan|tile|route|cls|offsets|bucket|plan|fc|small)|k6_" --csv --log-file gpurun_out/r2c/stream_launches.csv $CMD > gpurun_out/r2c/stream_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2c/stream_ncu.log
tail -3 gpurun_out/r2c/tests.log
