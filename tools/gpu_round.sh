# Full round evidence: smoke, all GPU tests, bench (C4, G=1), ncu launch list + K2 --set full.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(simtopk|normalize|merge|select|plan|keys|scan|tile|scatter|rank|cls|offsets|bucket|fill|zero|fc)" -s 153 -c 60 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_simtopk -c 1 -o gpurun_out/k2_c4 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?" >> gpurun_out/ncu_full.log
