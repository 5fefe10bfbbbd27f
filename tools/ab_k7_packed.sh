# K7 greedy ranking: register-packed (default) vs match.any (PAS_K7_MATCH=1) at 64M prompts, + GPU tests
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for i in 1 2; do
python tools/bench_stream.py --reps 3 > gpurun_out/ab_k7p_packed_$i.json 2>/dev/null
PAS_K7_MATCH=1 python tools/bench_stream.py --reps 3 > gpurun_out/ab_k7p_match_$i.json 2>/dev/null
done
CMD="python tools/bench_stream.py --reps 1"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(normalize|merge|select|scan|tile|route|cls|offsets|bucket|plan|fc)|k6_" --csv --log-file gpurun_out/stream_launches.csv $CMD > gpurun_out/stream_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/stream_ncu.log
