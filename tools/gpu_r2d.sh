mkdir -p gpurun_out/r2d
python -m paper_2502_06798_b200.build > /dev/null
timeout 1500 python -m pytest tests/test_gpu_redirect.py tests/test_gpu_graph.py tests/test_gpu_plan.py tests/test_gpu_parity.py -m gpu -q -s -k "not c4 and not c5 and not c3_parity_full and not fuzz" > gpurun_out/r2d/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2d/tests.log
# the checked build (device-side bounds / protocol checks) over the whole non-slow suite
PAS_LIB=$PWD/paper_2502_06798_b200/lib/libpas_checked.so timeout 1800 python -m pytest tests -m "gpu" -q -x -k "not c4 and not c5 and not c3_parity_full" > gpurun_out/r2d/tests_checked.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2d/tests_checked.log
timeout 300 python bench.py --config C2 --steps 2000 --no-cpu-baseline --no-e2e > gpurun_out/r2d/bench_c2.json 2>&1
CMD="python tools/bench_stream.py --reps 1"
timeout 600 python tools/bench_stream.py > gpurun_out/r2d/stream.json 2> gpurun_out/r2d/stream.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(normalize|merge|select|scan|tile|route|cls|offsets|bucket|plan|fc|small)|k6_" --csv --log-file gpurun_out/r2d/stream_launches.csv $CMD > gpurun_out/r2d/stream_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2d/stream_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k6_fused|k6_zone|k_cls_rank" -c 4 -o gpurun_out/r2d/k6k7_full $CMD > gpurun_out/r2d/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2d/ncu_full.log
tail -3 gpurun_out/r2d/tests.log; tail -3 gpurun_out/r2d/tests_checked.log
