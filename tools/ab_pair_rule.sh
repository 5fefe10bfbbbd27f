O=gpurun_out/ab_pair_rule
mkdir -p $O
python -m paper_2502_06798_b200.build > /dev/null
timeout 300 python tools/c1_latency.py > $O/c1_latency.json 2>&1
REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $O/c1_launches_warm.csv python tools/c1_latency.py > /dev/null 2>&1
for n in 128 256 384 512; do
  timeout 900 python bench.py --config C5 --prompts $n --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5_n${n}.json 2> $O/c5_n${n}.err
  python -c "import json; d=json.loads(open('$O/c5_n${n}.json').read().strip().splitlines()[-1]); print($n, round(d['value'],1), d['clocks']['sm_mhz'])"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_cache.py -m gpu -q -x -k "not c4" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
tail -2 $O/tests.log; cat $O/c1_latency.json
