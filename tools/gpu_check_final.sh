# Last-commit check: smoke, the whole -m gpu suite, the C4 / C2 / C1 bench lines (gpurun_out/check/)
O=${O:-gpurun_out/check}
mkdir -p $O
python -m paper_2502_06798_b200.build > /dev/null
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_c4_g1.json 2> $O/bench_c4_g1.err
timeout 600 python bench.py --config C2 --steps 2000 > $O/bench_c2_g1.json 2> $O/bench_c2_g1.err
timeout 600 python bench.py --config C1 --steps 5000 > $O/bench_c1_g1.json 2> $O/bench_c1_g1.err
tail -1 $O/smoke.log; tail -2 $O/gpu_tests.log
for c in c4 c2 c1; do python -c "
import json; d=json.loads(open('$O/bench_${c}_g1.json').read().strip().splitlines()[-1]); e=d['e2e']
print('$c', round(d['value'],1), 'frac', d['roofline'] and round(d['roofline']['frac'],3), 'e2e', round(e['value'],1), 'sync', round(e['value_sync'],1), 'cpu', d['cpu_baseline']['value'], d['clocks']['sm_mhz'], d['gpu_launches'])"; done
