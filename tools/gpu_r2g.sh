mkdir -p gpurun_out/r2g
python -m paper_2502_06798_b200.build > /dev/null
REPS=5 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_simtopk|k_small|k_normalize" -s 6 -c 6 -o gpurun_out/r2g/c1_full python tools/c1_latency.py > gpurun_out/r2g/c1_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2g/c1_ncu.log
REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/r2g/c1_launches_warm.csv python tools/c1_latency.py > gpurun_out/r2g/c1_ncu2.log 2>&1
timeout 300 python tools/c1_latency.py > gpurun_out/r2g/c1_latency.json 2>&1
CMD="python tools/bench_stream.py --reps 1"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(normalize|merge|select|scan|tile|route|cls|offsets|bucket|plan|fc|small)|k6_" --csv --log-file gpurun_out/r2g/stream_launches.csv $CMD > gpurun_out/r2g/stream_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2g/stream_ncu.log
