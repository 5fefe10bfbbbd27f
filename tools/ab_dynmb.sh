# Dynamic-schedule chunk length at small/mid N vs the 50M cache: L2 budget 100 (default) / 200 / 400 MB
# (T grows with it).  Results: gpurun_out/dynmb/
set -u
O=gpurun_out/dynmb
mkdir -p $O
for rep in 1 2; do
  for mb in 100 200 400; do
    PAS_K2_DYN_MB=$mb timeout 900 python tools/sweep.py --kind load --ns 1024,2048,4096,8192 --steps 4 --warmup 2 --prewarm-s 3 > $O/c5_mb${mb}_$rep.jsonl 2> $O/c5_mb${mb}_$rep.err
  done
done
