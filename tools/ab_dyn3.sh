# K2 dynamic schedule: prompt-tile groups (A budget) and chunk length at C4; DRAM bytes per launch.
# Results: gpurun_out/dyn3/
set -u
O=gpurun_out/dyn3
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "k2_dyn or c3_parity" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
grep -q "rc=0" $O/tests.log || exit 1
B="python bench.py --no-cpu-baseline --no-e2e"
V="AMB=4096,TMAX=64 AMB=56,TMAX=64 AMB=40,TMAX=64 AMB=4096,TMAX=128"
for rep in 1 2; do
  for v in $V; do
    a=${v%%,*}; t=${v##*,}
    env PAS_K2_DYN_$a PAS_K2_DYN_$t timeout 600 $B --steps 5 --warmup 3 > $O/c4_${a}_${t}_$rep.json 2> $O/c4_${a}_${t}_$rep.err
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for v in $V; do
  a=${v%%,*}; t=${v##*,}
  env PAS_K2_DYN_$a PAS_K2_DYN_$t timeout 600 ncu --metrics $M --clock-control none -k regex:k_simtopk -c 1 --csv --log-file $O/ncu_c4_${a}_${t}.csv $B --steps 1 --warmup 1 > /dev/null 2>&1
done
