# Round evidence: smoke, all GPU tests, bench (C4 default, reference arm, f3 dispatcher, C3, C2), f4
# solver timing, sweeps (cache size, C5 load), ncu launch list + K2 --set full capture, streaming
# kernels at 64M prompts.  Results: gpurun_out/final/
set -u
O=gpurun_out/final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > $O/smi.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -s > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_c4_g1.json 2> $O/bench_c4_g1.err; echo "rc=$?" >> $O/bench_c4_g1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_c4.json 2> $O/bench_reference_c4.err
timeout 900 python bench.py --dispatcher --no-cpu-baseline --no-e2e > $O/bench_c4_g1_dispatcher.json 2> $O/bench_c4_g1_dispatcher.err
timeout 900 python bench.py --config C3 --steps 100 > $O/bench_c3_g1.json 2> $O/bench_c3_g1.err
timeout 900 python bench.py --config C2 --steps 2000 > $O/bench_c2_g1.json 2> $O/bench_c2_g1.err
timeout 600 python tools/bench_controller.py > $O/controller.jsonl 2> $O/controller.err
if [ "${SWEEPS:-1}" = 1 ]; then
timeout 1200 python tools/sweep.py --kind load --steps 4 --warmup 2 > $O/c5_load_sweep_50M_g1.jsonl 2> $O/c5_sweep.err
timeout 1200 python tools/sweep.py --kind cache --steps 4 --warmup 2 > $O/cache_sweep_n16384.jsonl 2> $O/cache_sweep.err
fi
# launch list of the bench command: skip the 2 launches per 65,536-row block of the 10M cache load
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_|k6_" -s 306 -c 60 --csv --log-file $O/c4_g1_launches.csv $CMD > $O/ncu_launch.log 2>&1; echo "ncu1 rc=$?" >> $O/ncu_launch.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_simtopk -c 1 -o $O/k2_c4_g1 $CMD > $O/ncu_full.log 2>&1; echo "ncu2 rc=$?" >> $O/ncu_full.log
timeout 600 python tools/bench_stream.py > $O/stream_64M.json 2> $O/stream.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_|k6_" --csv --log-file $O/stream_launches_64M.csv python tools/bench_stream.py --reps 1 > $O/stream_ncu.log 2>&1; echo "ncu3 rc=$?" >> $O/stream_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_normalize|k_select_s1|k_cls_rank" -c 3 -o $O/stream_k1k3k7 python tools/bench_stream.py --reps 1 > $O/ncu_stream_full.log 2>&1; echo "ncu4 rc=$?" >> $O/ncu_stream_full.log
