# C5 (50M rows) at intermediate batch sizes, and N = 512 on the pair vs the single-CTA tile
O=gpurun_out/ab_c5_fine
mkdir -p $O
python -m paper_2502_06798_b200.build > /dev/null
run() {  # n tag env...
  n=$1; tag=$2; shift 2
  env "$@" timeout 900 python bench.py --config C5 --prompts $n --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5_n${n}_$tag.json 2> $O/c5_n${n}_$tag.err
  python -c "import json; d=json.loads(open('$O/c5_n${n}_$tag.json').read().strip().splitlines()[-1]); print($n, '$tag', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"
}
for rep in 1 2; do
  run 512 pair$rep PAS_K2_PAIR_MAX_TILES=4
  run 512 single$rep PAS_K2_PAIR_MAX_TILES=0
done
for n in 640 768 1024 1536 2048; do run $n default X=1; done
