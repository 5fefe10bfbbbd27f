# C1: K2's duplicated-row epilogue on vs off (PAS_K2_NO_DUP), same box, alternating
O=gpurun_out/ab_dup
mkdir -p $O
python -m paper_2502_06798_b200.build > /dev/null
for rep in 1 2 3; do
  for v in dup nodup; do
    if [ $v = nodup ]; then export PAS_K2_NO_DUP=1; else unset PAS_K2_NO_DUP; fi
    timeout 300 python tools/c1_latency.py > $O/c1_${v}_$rep.json 2>&1
    echo "$v $rep $(cat $O/c1_${v}_$rep.json)"
  done
done
unset PAS_K2_NO_DUP
REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $O/c1_launches_dup.csv python tools/c1_latency.py > /dev/null 2>&1
PAS_K2_NO_DUP=1 REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $O/c1_launches_nodup.csv python tools/c1_latency.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_k1_exact.py tests/test_gpu_parity.py -m gpu -q -x -k "c1 or small or graph or k1 or odd_tile or topk_widths" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log; tail -2 $O/tests.log
