# Post-argmax tuning: C2 static vs dynamic schedule, pair-tile threshold at small N (prewarmed), C1;
# ncu --set full of the K7 rank and K6 histogram kernels at 64M prompts.  Results: gpurun_out/tune/
set -u
O=gpurun_out/tune
mkdir -p $O
B="python bench.py --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  timeout 300 $B --config C2 --steps 50 > $O/c2_default_$rep.json 2> $O/c2_default_$rep.err
  PAS_K2_DYN_MIN_STEPS=2 timeout 300 $B --config C2 --steps 50 > $O/c2_dyn_$rep.json 2> $O/c2_dyn_$rep.err
  timeout 300 $B --config C1 --steps 200 > $O/c1_$rep.json 2> $O/c1_$rep.err
done
for v in 0 2 4 8; do
  PAS_K2_PAIR_MAX_TILES=$v timeout 900 python tools/sweep.py --kind load --ns 256,512,1024,2048 --steps 6 --warmup 2 --prewarm-s 5 > $O/c5_pair$v.jsonl 2> $O/c5_pair$v.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cls_rank|k6_hist|k6_assign" -c 3 -o $O/stream_k67 python tools/bench_stream.py --reps 1 > $O/ncu_k67.log 2>&1; echo "rc=$?" >> $O/ncu_k67.log
