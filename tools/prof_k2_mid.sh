# K2 at mid-N (C5 load-curve regime): plain timings, then one ncu --set full capture per shape.
for N in 1024 4096 16384; do
  timeout 600 python tools/k2_probe.py --N $N --M 20000000 --reps 3 > gpurun_out/k2mid_$N.jsonl 2>&1
done
for N in 1024 16384; do
  timeout 900 ncu --set full --clock-control none -k regex:k_simtopk -s 1 -c 1 -o gpurun_out/k2mid_$N \
    python tools/k2_probe.py --N $N --M 20000000 --reps 2 > gpurun_out/k2mid_ncu_$N.log 2>&1
done
