# K1 check: GPU tests touching K1, streaming bench (cache insert), bench C4 stage times
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cache.py -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python tools/bench_stream.py --reps 3 > gpurun_out/k1_stream.json 2>/dev/null
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/k1_bench.json 2> gpurun_out/k1_bench.err
