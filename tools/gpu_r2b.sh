mkdir -p gpurun_out/r2b
python -m paper_2502_06798_b200.build > /dev/null
timeout 1200 python -m pytest tests/test_gpu_graph.py tests/test_gpu_multi.py tests/test_gpu_plan.py tests/test_gpu_parity.py -m gpu -q -s -k "graph or small or multi or explicit or plan or c1 or ragged or widths or cold or shards or nccl" > gpurun_out/r2b/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2b/tests.log
for g in "" "--graph"; do
  timeout 300 python bench.py --config C1 --steps 2000 --no-cpu-baseline --no-e2e $g > gpurun_out/r2b/bench_c1$g.json 2>&1
  timeout 300 python bench.py --config C2 --steps 2000 --no-cpu-baseline --no-e2e $g > gpurun_out/r2b/bench_c2$g.json 2>&1
done
OUT=gpurun_out/r2b/sanitizer SAN_TIMEOUT=900 bash tools/sanitize.sh
tail -3 gpurun_out/r2b/tests.log
