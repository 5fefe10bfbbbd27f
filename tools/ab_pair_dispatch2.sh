L=paper_2502_06798_b200/lib
python -m paper_2502_06798_b200.build -DPAS_K2_PAIR_MAX_TILES=0 --out=$L/libpas_nopair.so > /dev/null
for rep in 1 2; do
for v in cur nopair; do
  lib=$PWD/$L/libpas.so; [ $v = nopair ] && lib=$PWD/$L/libpas_nopair.so
  PAS_LIB=$lib timeout 1200 python tools/sweep.py --kind load --ns 4096,8192,16384,32768 --steps 5 --warmup 1 > gpurun_out/c5_${v}_$rep.jsonl 2>/dev/null
done; done
