OUT=${OUT:-r2ze}
mkdir -p gpurun_out/$OUT
python -m paper_2502_06798_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_host_pipeline.py tests/test_gpu_nvtx.py -m gpu -q -x > gpurun_out/$OUT/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/$OUT/tests.log
timeout 600 python bench.py --config C2 --steps 2000 --no-cpu-baseline > gpurun_out/$OUT/bench_c2.json 2> gpurun_out/$OUT/bench_c2.err
timeout 600 python bench.py --config C1 --steps 5000 --no-cpu-baseline > gpurun_out/$OUT/bench_c1.json 2> gpurun_out/$OUT/bench_c1.err
timeout 600 python bench.py --config C3 --steps 100 --no-cpu-baseline > gpurun_out/$OUT/bench_c3.json 2> gpurun_out/$OUT/bench_c3.err
timeout 900 python bench.py > gpurun_out/$OUT/bench_c4.json 2> gpurun_out/$OUT/bench_c4.err
tail -2 gpurun_out/$OUT/tests.log
for c in c1 c2 c3 c4; do python -c "
import json; d=json.loads(open('gpurun_out/$OUT/bench_$c.json').read().strip().splitlines()[-1]); e=d['e2e']
print('$c', round(d['value'],1), 'e2e', round(e['value'],1), 'sync', round(e['value_sync'],1), d['clocks']['sm_mhz'])"; done
