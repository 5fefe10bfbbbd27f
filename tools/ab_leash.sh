# A/B of the K2 progress leash on one box (same GPU, back to back).  Results: gpurun_out/leash/
mkdir -p gpurun_out/leash
O=gpurun_out/leash
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or c1_parity or c2 or c3 or virtual or fewer or ragged" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  timeout 600 $B > $O/c4_leash_$rep.json 2>/dev/null
  PAS_K2_NOLEASH=1 timeout 600 $B > $O/c4_free_$rep.json 2>/dev/null
done
timeout 900 python tools/sweep.py --kind load --ns 512,1024,2048,4096,8192 --steps 3 --warmup 1 > $O/c5_leash.jsonl 2>$O/c5_leash.err
PAS_K2_NOLEASH=1 timeout 900 python tools/sweep.py --kind load --ns 512,1024,2048,4096,8192 --steps 3 --warmup 1 > $O/c5_free.jsonl 2>$O/c5_free.err
# DRAM bytes of one K2 launch at C4, leash on / off (profiler run: traffic only, no timing claims)
for v in leash free; do
  if [ $v = free ]; then export PAS_K2_NOLEASH=1; else unset PAS_K2_NOLEASH; fi
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_simtopk -s 1 -c 1 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c4_$v.csv 2>$O/ncu_c4_$v.err
done
