# After the N-dispatched pair tile: GPU tests, C5 load curve, C4 bench.
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 1200 python tools/sweep.py --kind load --steps 5 --warmup 1 > gpurun_out/c5_load.jsonl 2> gpurun_out/c5_load.err
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c4.json 2> gpurun_out/c4.err
