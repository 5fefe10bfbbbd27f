# Small batches vs the 50M cache: A-in-TMEM tile (libpas_atmem.so, -DPAS_K2_ATMEM=1) vs the default
# dispatch (CTA pair for N <= 512, single-CTA dynamic above).  Results: gpurun_out/atmem/
set -u
O=gpurun_out/atmem
L=$PWD/paper_2502_06798_b200/lib
mkdir -p $O
PAS_LIB=$L/libpas_atmem.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_parity or gemm or ragged or fewer" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for rep in 1 2; do
  for v in pas pas_atmem; do
    PAS_LIB=$L/lib$v.so timeout 900 python tools/sweep.py --kind load --ns 256,512,1024 --steps 6 --warmup 2 --prewarm-s 5 > $O/c5_${v}_$rep.jsonl 2> $O/c5_${v}_$rep.err
  done
done
