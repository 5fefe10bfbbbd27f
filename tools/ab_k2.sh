# Factorial A/B of K2 choices on one box (same GPU, back to back).  Results: gpurun_out/ab_*.json
B="python bench.py --steps 8 --warmup 2 --no-cpu-baseline --no-e2e"
L=paper_2502_06798_b200/lib
for v in "1 1" "3 1" "3 0"; do set -- $v
  python -m paper_2502_06798_b200.build -DPAS_K2_EPI=$1 -DPAS_MBAR_SUSPEND=$2 --out=$L/libpas_e$1s$2.so > /dev/null
done
PAS_LIB=$PWD/$L/libpas_e3s1.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or c1_parity or c3 or virtual or fewer or ragged" > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
for rep in 1 2; do
  for v in e1s1 e3s1 e3s0; do
    PAS_K2_RANGES=1 PAS_LIB=$PWD/$L/libpas_$v.so timeout 600 $B > gpurun_out/ab_${v}_R1_$rep.json 2>/dev/null
  done
  PAS_LIB=$PWD/$L/libpas_e3s1.so timeout 600 $B > gpurun_out/ab_e3s1_Rauto_$rep.json 2>/dev/null
done
