# Streaming kernels at >= 1 GB: tests first, plain run, then the ncu launch list (time + DRAM bytes).
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python tools/bench_stream.py > gpurun_out/stream.json 2> gpurun_out/stream.err; echo "rc=$?" >> gpurun_out/stream.err
CMD="python tools/bench_stream.py --reps 1"
timeout 600 $CMD > gpurun_out/stream_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(normalize|merge|select|scan|tile|route|cls|offsets|bucket|plan|fc)|k6_" --csv --log-file gpurun_out/stream_launches.csv $CMD > gpurun_out/stream_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/stream_ncu.log
