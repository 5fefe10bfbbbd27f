free -g > gpurun_out/box.txt; nproc >> gpurun_out/box.txt; lscpu | grep -E "Model name|Flags" | cut -c1-300 >> gpurun_out/box.txt
python -m paper_2502_06798_b200.build > /dev/null
timeout 1500 python -m pytest tests/test_gpu_k1_exact.py tests/test_gpu_parity.py -m gpu -q -s -k "k1 or qhat or store_rows or error_distribution or c1 or c2 or c3 or widths or ragged or bf16 or embedding_widths" > gpurun_out/gpu_tests2.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests2.log
tail -3 gpurun_out/gpu_tests2.log
