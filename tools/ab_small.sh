# K2's 128-row small-problem tile (simtopk_small) on vs off (PAS_K2_NO_SMALL), same box, alternating
O=gpurun_out/ab_small
mkdir -p $O
python -m paper_2502_06798_b200.build > /dev/null
for rep in 1 2; do
  for v in small nosmall; do
    if [ $v = nosmall ]; then export PAS_K2_NO_SMALL=1; else unset PAS_K2_NO_SMALL; fi
    for n in 1 64; do
      C1_N=$n timeout 300 python tools/c1_latency.py > $O/c1_${v}_n${n}_$rep.json 2>&1
      echo "$v n=$n $rep $(cat $O/c1_${v}_n${n}_$rep.json)"
    done
  done
done
unset PAS_K2_NO_SMALL
REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $O/c1_launches_small.csv python tools/c1_latency.py > /dev/null 2>&1
PAS_K2_NO_SMALL=1 REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $O/c1_launches_nosmall.csv python tools/c1_latency.py > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_cache.py tests/test_gpu_nvtx.py tests/test_gpu_host_pipeline.py tests/test_gpu_dispatch.py -m gpu -q -x -k "not c4 and not c5" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log; tail -2 $O/tests.log
