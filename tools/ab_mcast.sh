# K2 B multicast across CTA pairs (PAS_K2_MCAST=1) vs the default single-CTA dynamic schedule:
# byte-identity tests first (bounded), then C4 / C3 timing and ncu.  Results: gpurun_out/mcast/
set -u
O=gpurun_out/mcast
mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "matches_static" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
grep -q "rc=0" $O/tests.log || exit 1
B="python bench.py --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  for m in 0 1; do
    PAS_K2_MCAST=$m timeout 600 $B --steps 5 --warmup 3 > $O/c4_mc${m}_$rep.json 2> $O/c4_mc${m}_$rep.err
    PAS_K2_MCAST=$m timeout 300 $B --config C3 --steps 30 > $O/c3_mc${m}_$rep.json 2> $O/c3_mc${m}_$rep.err
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for m in 0 1; do
  PAS_K2_MCAST=$m timeout 600 ncu --metrics $M --clock-control none -k regex:k_simtopk -c 1 --csv --log-file $O/ncu_c4_mc$m.csv $B --steps 1 --warmup 1 > /dev/null 2>&1
done
