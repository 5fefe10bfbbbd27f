# K2 epilogue: warp-vote column skipping (default build) vs the per-lane divergent insert path
# (libpas_novote.so, -DPAS_K2_EPI_VOTE=0), back to back.  Results: gpurun_out/vote/
set -u
O=gpurun_out/vote
L=$PWD/paper_2502_06798_b200/lib
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "k2_dyn or c1_parity or c2_parity or c3_parity or topk_widths or ragged or fewer or many" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
grep -q "rc=0" $O/tests.log || exit 1
B="python bench.py --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  for v in pas pas_novote; do
    PAS_LIB=$L/lib$v.so timeout 300 $B --config C2 --steps 50 > $O/c2_${v}_$rep.json 2> $O/c2_${v}_$rep.err
    PAS_LIB=$L/lib$v.so timeout 300 $B --config C3 --steps 30 > $O/c3_${v}_$rep.json 2> $O/c3_${v}_$rep.err
    PAS_LIB=$L/lib$v.so timeout 600 $B --steps 5 --warmup 3 > $O/c4_${v}_$rep.json 2> $O/c4_${v}_$rep.err
  done
done
for v in pas pas_novote; do
  PAS_LIB=$L/lib$v.so timeout 900 python tools/sweep.py --kind load --ns 256,512,1024,2048,4096 --steps 4 --warmup 2 > $O/c5_$v.jsonl 2> $O/c5_$v.err
done
