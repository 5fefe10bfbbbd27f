# K2 dynamic schedule: prompt-tile groups (A budget) at T = 128, C4 throughput and DRAM per launch.
set -u
O=gpurun_out/amb
mkdir -p $O
B="python bench.py --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  for a in 4096 56 40; do
    PAS_K2_DYN_AMB=$a timeout 600 $B --steps 5 --warmup 3 > $O/c4_amb${a}_$rep.json 2> $O/c4_amb${a}_$rep.err
  done
done
for a in 4096 56 40; do
  PAS_K2_DYN_AMB=$a timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_simtopk -c 1 --csv --log-file $O/ncu_c4_amb$a.csv $B --steps 1 --warmup 1 > /dev/null 2>&1
done
