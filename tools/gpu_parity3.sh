python -m paper_2502_06798_b200.build > /dev/null
timeout 1500 python -m pytest tests/test_gpu_plan.py tests/test_gpu_k1_exact.py tests/test_gpu_parity.py -m gpu -q -s -k "plan or degradation or k1 or qhat or store_rows or c2 or c3 or c4" > gpurun_out/gpu_tests3.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests3.log
tail -3 gpurun_out/gpu_tests3.log
