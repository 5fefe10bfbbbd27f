OUT=${OUT:-r2s}
mkdir -p gpurun_out/$OUT
python -m paper_2502_06798_b200.build > /dev/null
timeout 1500 python -m pytest tests/test_gpu_nvtx.py tests/test_gpu_redirect.py tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_dispatch.py tests/test_gpu_forecast.py tests/test_gpu_plan.py -m gpu -q -s -x -k "not c4 and not c5 and not fuzz" > gpurun_out/$OUT/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/$OUT/tests.log
CMD="python tools/bench_stream.py --reps 1"
timeout 600 python tools/bench_stream.py > gpurun_out/$OUT/stream.json 2> gpurun_out/$OUT/stream.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(normalize|merge|select|scan|tile|route|cls|offsets|bucket|plan|fc|small)|k6_" --csv --log-file gpurun_out/$OUT/stream_launches.csv $CMD > gpurun_out/$OUT/stream_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/$OUT/stream_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cls_rank" -c 1 -o gpurun_out/$OUT/k7_full $CMD > gpurun_out/$OUT/ncu_full.log 2>&1
for v in ${VARIANTS:-}; do
  PAS_LIB=paper_2502_06798_b200/lib/libpas_$v.so timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_cls_rank" --csv --log-file gpurun_out/$OUT/k7_$v.csv $CMD > gpurun_out/$OUT/k7_$v.log 2>&1
done
tail -3 gpurun_out/$OUT/tests.log
