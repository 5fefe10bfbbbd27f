# ncu --set full of the K7 rank kernels at 64M prompts (stream bench); read back with ncu -i.
CMD="python tools/bench_stream.py --reps 1"
timeout 600 $CMD > gpurun_out/k7_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cls_(rank|count)" -c 2 -o gpurun_out/k7_full $CMD > gpurun_out/k7_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/k7_full.log
