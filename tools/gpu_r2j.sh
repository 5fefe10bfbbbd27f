mkdir -p gpurun_out/r2j
python -m paper_2502_06798_b200.build > /dev/null
timeout 600 python bench.py --config C1 --steps 5000 --no-cpu-baseline > gpurun_out/r2j/bench_c1_g1.json 2> gpurun_out/r2j/bench_c1_g1.err
timeout 600 python bench.py --config C1 --steps 5000 --graph --no-cpu-baseline --no-e2e > gpurun_out/r2j/bench_c1_graph.json 2> gpurun_out/r2j/bench_c1_graph.err
# launch list of the bench command: skip the 3 launches per 65,536-row block of the 10M cache load (153 blocks)
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_|k6_" -s 459 -c 60 --csv --log-file gpurun_out/r2j/c4_g1_launches.csv $CMD > gpurun_out/r2j/ncu_launch.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/r2j/ncu_launch.log
