# C2 (4,096 x 100k): K2 schedule choices after the argmax epilogue (static R, dynamic forced).
set -u
O=gpurun_out/c2ab
mkdir -p $O
B="python bench.py --config C2 --steps 100 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  timeout 300 $B > $O/default_$rep.json 2>/dev/null
  for r in 5 8 37 74; do PAS_K2_RANGES=$r timeout 300 $B > $O/static_R${r}_$rep.json 2>/dev/null; done
  for mb in 16 40 100; do PAS_K2_DYN_MIN_STEPS=1 PAS_K2_DYN_MB=$mb timeout 300 $B > $O/dyn_mb${mb}_$rep.json 2>/dev/null; done
  timeout 300 python bench.py --config C3 --steps 30 --no-cpu-baseline --no-e2e > $O/c3_default_$rep.json 2>/dev/null
  PAS_K2_SCHED=static timeout 300 python bench.py --config C3 --steps 30 --no-cpu-baseline --no-e2e > $O/c3_static_$rep.json 2>/dev/null
done
