OUT=${OUT:-r2x}
mkdir -p gpurun_out/$OUT
python -m paper_2502_06798_b200.build > /dev/null
PAS_LIB=$PWD/paper_2502_06798_b200/lib/libpas_clk.so REPS=5 timeout 300 python tools/c1_latency.py 2>&1 | grep -E "SMALLCLK|PLANCLK" | tail -4 > gpurun_out/$OUT/clk.log
timeout 300 python tools/c1_latency.py > gpurun_out/$OUT/c1_latency.json 2>&1
REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/$OUT/c1_launches_warm.csv python tools/c1_latency.py > gpurun_out/$OUT/c1_ncu.log 2>&1
if [ -n "$STREAM" ]; then
  CMD="python tools/bench_stream.py --reps 1"
  timeout 600 python tools/bench_stream.py > gpurun_out/$OUT/stream.json 2> gpurun_out/$OUT/stream.err
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(normalize|merge|select|scan|tile|route|cls|offsets|bucket|plan|fc|small)|k6_" --csv --log-file gpurun_out/$OUT/stream_launches.csv $CMD > gpurun_out/$OUT/stream_ncu.log 2>&1
fi
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -m gpu -q -x -k "not c4 and not c5 and not fuzz" > gpurun_out/$OUT/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/$OUT/tests.log
  tail -3 gpurun_out/$OUT/tests.log
fi
cat gpurun_out/$OUT/clk.log gpurun_out/$OUT/c1_latency.json
