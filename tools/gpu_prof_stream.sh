timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
CMD="python tools/bench_stream.py --reps 1"
timeout 600 $CMD > gpurun_out/stream_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(normalize|merge|select|keys|scan|tile|scatter|rank|cls|offsets|bucket|plan)" --csv --log-file gpurun_out/stream_launches.csv $CMD > gpurun_out/stream_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_(select_s1|cls_rank|cls_count|bucket)" -c 4 -o gpurun_out/stream_full $CMD > gpurun_out/stream_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/stream_full.log
