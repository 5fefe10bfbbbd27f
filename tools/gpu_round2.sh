# round-2 evidence: smoke, the whole -m gpu suite, the default bench (C4) and C2 / C3 lines
mkdir -p gpurun_out/r2
python -m paper_2502_06798_b200.build > /dev/null
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2/smoke.log
timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q -s ${PYTEST_ARGS:-} > gpurun_out/r2/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2/gpu_tests.log
timeout 900 python bench.py > gpurun_out/r2/bench_c4.json 2> gpurun_out/r2/bench_c4.err; echo "bench rc=$?" >> gpurun_out/r2/bench_c4.err
timeout 600 python bench.py --config C3 --steps 100 --no-cpu-baseline > gpurun_out/r2/bench_c3.json 2> gpurun_out/r2/bench_c3.err
timeout 600 python bench.py --config C2 --steps 2000 --no-cpu-baseline > gpurun_out/r2/bench_c2.json 2> gpurun_out/r2/bench_c2.err
timeout 600 python bench.py --config C1 --steps 2000 --no-cpu-baseline > gpurun_out/r2/bench_c1.json 2> gpurun_out/r2/bench_c1.err
tail -2 gpurun_out/r2/gpu_tests.log
