# K2 dynamic vs static schedule on one box, back to back: parity first, then C3 / C4 device timing
# and one ncu launch of K2 each (DRAM bytes per launch).  Results: gpurun_out/dyn/
set -u
O=gpurun_out/dyn
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "k2_dyn or c1_parity or c2_parity or c3_parity or ragged or virtual or topk_widths or many" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
grep -q "rc=0" $O/tests.log || exit 1
B="python bench.py --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  for s in dynamic static; do
    PAS_K2_SCHED=$s timeout 300 $B --config C3 --steps 20 > $O/c3_${s}_$rep.json 2> $O/c3_${s}_$rep.err
    PAS_K2_SCHED=$s timeout 300 $B --config C2 --steps 50 > $O/c2_${s}_$rep.json 2> $O/c2_${s}_$rep.err
  done
done
for rep in 1 2; do
  for s in dynamic static; do
    PAS_K2_SCHED=$s timeout 600 $B --steps 5 --warmup 3 > $O/c4_${s}_$rep.json 2> $O/c4_${s}_$rep.err
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed
for s in dynamic static; do
  PAS_K2_SCHED=$s timeout 600 ncu --metrics $M --clock-control none -k regex:k_simtopk -c 2 --csv --log-file $O/ncu_c4_$s.csv $B --steps 1 --warmup 1 > /dev/null 2>&1
  PAS_K2_SCHED=$s timeout 600 ncu --metrics $M --clock-control none -k regex:k_simtopk -c 2 --csv --log-file $O/ncu_c3_$s.csv $B --config C3 --steps 1 --warmup 1 > /dev/null 2>&1
done
