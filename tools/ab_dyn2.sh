# K2 dynamic schedule tuning: L2 budget for in-flight chunks at C4, C2 fallback, C5 mid-range
# (dynamic vs static).  Results: gpurun_out/dyn2/
set -u
O=gpurun_out/dyn2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "k2_dyn or c2_parity or c3_parity" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
grep -q "rc=0" $O/tests.log || exit 1
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 300 $B --config C2 --steps 50 > $O/c2_default.json 2> $O/c2_default.err
for rep in 1 2; do
  for mb in 20 40 80; do
    PAS_K2_DYN_MB=$mb timeout 600 $B --steps 5 --warmup 3 > $O/c4_mb${mb}_$rep.json 2> $O/c4_mb${mb}_$rep.err
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for mb in 20 80; do
  PAS_K2_DYN_MB=$mb timeout 600 ncu --metrics $M --clock-control none -k regex:k_simtopk -c 1 --csv --log-file $O/ncu_c4_mb$mb.csv $B --steps 1 --warmup 1 > /dev/null 2>&1
done
for s in dynamic static; do
  PAS_K2_SCHED=$s timeout 900 python tools/sweep.py --kind load --ns 4096,8192,16384,32768,65536 --steps 4 --warmup 2 > $O/c5_$s.jsonl 2> $O/c5_$s.err
done
