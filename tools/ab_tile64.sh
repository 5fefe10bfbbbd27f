# K2 small-problem tile: 64 rows (default) vs 128 rows (PAS_K2_NO_TILE64), same box, alternating
O=gpurun_out/ab_tile64
mkdir -p $O
python -m paper_2502_06798_b200.build > /dev/null
for rep in 1 2; do
  for v in t64 t128; do
    if [ $v = t128 ]; then export PAS_K2_NO_TILE64=1; else unset PAS_K2_NO_TILE64; fi
    for n in 1 64; do
      C1_N=$n timeout 300 python tools/c1_latency.py > $O/c1_${v}_n${n}_$rep.json 2>&1
      echo "$v n=$n $rep $(cat $O/c1_${v}_n${n}_$rep.json)"
    done
  done
done
unset PAS_K2_NO_TILE64
REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $O/c1_launches_t64.csv python tools/c1_latency.py > /dev/null 2>&1
PAS_K2_NO_TILE64=1 REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $O/c1_launches_t128.csv python tools/c1_latency.py > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_cache.py tests/test_gpu_nvtx.py tests/test_gpu_host_pipeline.py tests/test_gpu_dispatch.py -m gpu -q -x -k "not c4 and not c5" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log; tail -2 $O/tests.log
