# ncu --set full of the streaming kernels at 64M prompts (stream bench): K6 (k6_hist, k6_assign) and
# K7 (k_cls_count, k_cls_rank); read back with ncu -i ... --page raw/source.
CMD="python tools/bench_stream.py --reps 1"
timeout 600 $CMD > gpurun_out/sf_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k6_hist|k6_assign|k_cls_(rank|count)" -c 4 -o gpurun_out/stream_full $CMD > gpurun_out/stream_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/stream_full.log
