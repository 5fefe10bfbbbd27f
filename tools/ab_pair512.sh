# C5 at small N: CTA pair vs the single-CTA dynamic tile (PAS_K2_PAIR_MAX_TILES = 4 default / 0 = never)
O=gpurun_out/ab_pair512
mkdir -p $O
python -m paper_2502_06798_b200.build > /dev/null
for rep in 1 2; do
for n in ${NS:-128 256 384}; do
  for t in 4 0; do
    PAS_K2_PAIR_MAX_TILES=$t timeout 900 python bench.py --config C5 --prompts $n --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5_n${n}_t${t}_r$rep.json 2> $O/c5_n${n}_t${t}_r$rep.err
    python -c "import json; d=json.loads(open('$O/c5_n${n}_t${t}_r$rep.json').read().strip().splitlines()[-1]); print($n, $t, $rep, round(d['value'],1), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"
  done
done
done
