# smoke + the whole -m gpu suite (no profiler); logs under gpurun_out/
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -s ${PYTEST_ARGS:-} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
