# C5 mid-N: K2 leash budget A/B (0 = off) on one box.  Results: gpurun_out/leash_mb/
mkdir -p gpurun_out/leash_mb
L=paper_2502_06798_b200/lib
for mb in 0 24 96; do
  python -m paper_2502_06798_b200.build -DPAS_K2_LEASH_MB=$mb --out=$L/libpas_lm$mb.so > /dev/null
done
for mb in 0 24 48 96; do
  lib=$PWD/$L/libpas_lm$mb.so; [ $mb = 48 ] && lib=$PWD/$L/libpas.so
  PAS_LIB=$lib timeout 900 python tools/sweep.py --kind load --ns 512,1024,2048 --steps 3 --warmup 1 > gpurun_out/leash_mb/c5_mb$mb.jsonl 2>gpurun_out/leash_mb/c5_mb$mb.err
done
