for i in 1 2; do
python tools/bench_stream.py --reps 3 > gpurun_out/ab_k7_r16_$i.json 2>/dev/null
PAS_LIB=$PWD/paper_2502_06798_b200/lib/libpas_k7r8.so python tools/bench_stream.py --reps 3 > gpurun_out/ab_k7_r8_$i.json 2>/dev/null
done
PAS_LIB=$PWD/paper_2502_06798_b200/lib/libpas_k7r8.so timeout 600 python -m pytest tests/test_gpu_dispatch.py tests/test_gpu_parity.py -x -q > gpurun_out/ab_k7_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_k7_tests.log
