# K2 dynamic schedule: chunk length sweep at C4 and C3 (L2 budget lifted).  Results: gpurun_out/dyn4/
set -u
O=gpurun_out/dyn4
mkdir -p $O
B="python bench.py --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  for t in 106 128 192 256 384; do
    PAS_K2_DYN_MB=4000 PAS_K2_DYN_TMAX=$t timeout 600 $B --steps 5 --warmup 3 > $O/c4_T${t}_$rep.json 2> $O/c4_T${t}_$rep.err
  done
  for t in 64 128 256; do
    PAS_K2_DYN_MB=4000 PAS_K2_DYN_TMAX=$t timeout 600 $B --config C3 --steps 30 > $O/c3_T${t}_$rep.json 2> $O/c3_T${t}_$rep.err
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for t in 192 256; do
  PAS_K2_DYN_MB=4000 PAS_K2_DYN_TMAX=$t timeout 600 ncu --metrics $M --clock-control none -k regex:k_simtopk -c 1 --csv --log-file $O/ncu_c4_T$t.csv $B --steps 1 --warmup 1 > /dev/null 2>&1
done
