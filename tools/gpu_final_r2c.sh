# Round-2 evidence: smoke, all GPU tests (product and checked builds), benches (C4 default + reference
# arm, C3, C2, C1 eager / graph, f3 dispatcher, f1 forecast, explicit collectives through a 1-rank
# communicator), N2 / C1 / f4 microbenchmarks, sweeps, ncu launch lists + full captures.
# Results: gpurun_out/final4/
set -u
O=gpurun_out/final4
mkdir -p $O
python -m paper_2502_06798_b200.build > /dev/null
python -m paper_2502_06798_b200.build -DPAS_CHECKED=1 --out=paper_2502_06798_b200/lib/libpas_checked.so > /dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > $O/smi.txt
nproc >> $O/smi.txt; free -g >> $O/smi.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 3000 python -m pytest tests -m gpu -q -s > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
PAS_LIB=$PWD/paper_2502_06798_b200/lib/libpas_checked.so timeout 2400 python -m pytest tests -m gpu -q -k "not c4 and not c5 and not c3_parity_full and not error_distribution" > $O/gpu_tests_checked.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests_checked.log
timeout 900 python bench.py > $O/bench_c4_g1.json 2> $O/bench_c4_g1.err; echo "rc=$?" >> $O/bench_c4_g1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_c4.json 2> $O/bench_reference_c4.err
timeout 900 python bench.py --config C3 --steps 100 > $O/bench_c3_g1.json 2> $O/bench_c3_g1.err
timeout 900 python bench.py --config C2 --steps 2000 > $O/bench_c2_g1.json 2> $O/bench_c2_g1.err
timeout 600 python bench.py --config C2 --steps 2000 --graph --no-cpu-baseline --no-e2e > $O/bench_c2_graph.json 2> $O/bench_c2_graph.err
timeout 600 python bench.py --config C1 --steps 5000 --no-cpu-baseline > $O/bench_c1_g1.json 2> $O/bench_c1_g1.err
timeout 600 python bench.py --config C1 --steps 5000 --graph --no-cpu-baseline --no-e2e > $O/bench_c1_graph.json 2> $O/bench_c1_graph.err
timeout 900 python bench.py --dispatcher --no-cpu-baseline --no-e2e > $O/bench_c4_dispatcher.json 2> $O/bench_c4_dispatcher.err
timeout 900 python bench.py --forecast 1000 --no-cpu-baseline --no-e2e > $O/bench_c4_forecast.json 2> $O/bench_c4_forecast.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --config C2 --steps 2000 --force-collective --collectives explicit --no-cpu-baseline --no-e2e > $O/bench_c2_explicit_1rank.json 2> $O/bench_c2_explicit_1rank.err
timeout 600 python tools/bench_n2.py > $O/bench_n2.json 2> $O/bench_n2.err
timeout 300 python tools/c1_latency.py > $O/c1_latency.json 2> $O/c1_latency.err
timeout 600 python tools/bench_controller.py > $O/controller.jsonl 2> $O/controller.err
if [ "${SWEEPS:-1}" = 1 ]; then
timeout 1500 python tools/sweep.py --kind load --steps 4 --warmup 2 > $O/c5_load_sweep_50M_g1.jsonl 2> $O/c5_sweep.err
timeout 1200 python tools/sweep.py --kind cache --steps 4 --warmup 2 > $O/cache_sweep_n16384.jsonl 2> $O/cache_sweep.err
fi
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_|k6_" -s 459 -c 60 --csv --log-file $O/c4_g1_launches.csv $CMD > $O/ncu_launch.log 2>&1; echo "ncu1 rc=$?" >> $O/ncu_launch.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_simtopk -c 1 -o $O/k2_c4_g1 $CMD > $O/ncu_full.log 2>&1; echo "ncu2 rc=$?" >> $O/ncu_full.log
timeout 600 python tools/bench_stream.py > $O/stream_64M.json 2> $O/stream.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_|k6_" --csv --log-file $O/stream_launches_64M.csv python tools/bench_stream.py --reps 1 > $O/stream_ncu.log 2>&1; echo "ncu3 rc=$?" >> $O/stream_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_normalize|k_select_s1|k6_fused|k_cls_rank" -c 4 -o $O/stream_full python tools/bench_stream.py --reps 1 > $O/ncu_stream_full.log 2>&1; echo "ncu4 rc=$?" >> $O/ncu_stream_full.log
REPS=20 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $O/c1_launches_warm.csv python tools/c1_latency.py > $O/c1_ncu.log 2>&1
echo done > $O/DONE
