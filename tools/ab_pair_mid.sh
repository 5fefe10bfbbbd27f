# C5 load curve: CTA-pair (cta_group::2, 256x256) vs single-CTA K2 (leash on / off) on one box.
mkdir -p gpurun_out/pair_mid
L=paper_2502_06798_b200/lib
python -m paper_2502_06798_b200.build -DPAS_K2_PAIR=1 --out=$L/libpas_pair.so > /dev/null
for rep in 1 2; do
for v in ss pair ssfree; do
  lib=$PWD/$L/libpas.so; [ $v = pair ] && lib=$PWD/$L/libpas_pair.so
  if [ $v = ssfree ]; then export PAS_K2_NOLEASH=1; else unset PAS_K2_NOLEASH; fi
  PAS_LIB=$lib timeout 1200 python tools/sweep.py --kind load --ns 256,512,1024,2048,4096 --steps 5 --warmup 1 > gpurun_out/pair_mid/c5_${v}_$rep.jsonl 2>gpurun_out/pair_mid/c5_${v}_$rep.err
done
done
