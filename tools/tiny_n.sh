O=gpurun_out/tiny_n
mkdir -p $O
python -m paper_2502_06798_b200.build > /dev/null
for n in 1 8 32 64; do
  C1_N=$n timeout 300 python tools/c1_latency.py > $O/lat_$n.json 2>&1; echo "$n $(cat $O/lat_$n.json)"
  C1_N=$n REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $O/launches_$n.csv python tools/c1_latency.py > /dev/null 2>&1
done
