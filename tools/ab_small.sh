# C5 small batches (N = 256..2048 vs 50M): CTA-pair tile with the static schedule (default) vs the
# single-CTA tile with the dynamic schedule (PAS_K2_PAIR_MAX_TILES=0); C3 K2 DRAM bytes (ncu).
# Results: gpurun_out/small/
set -u
O=gpurun_out/small
mkdir -p $O
PAS_K2_PAIR_MAX_TILES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "c1_parity or ragged or fewer or topk_widths or k2_dyn" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for v in 16 0; do
  PAS_K2_PAIR_MAX_TILES=$v timeout 900 python tools/sweep.py --kind load --ns 256,512,1024,2048,4096 --steps 4 --warmup 2 > $O/c5_pair$v.jsonl 2> $O/c5_pair$v.err
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
timeout 600 ncu --metrics $M --clock-control none -k regex:k_simtopk -c 1 --csv --log-file $O/ncu_c3.csv python bench.py --no-cpu-baseline --no-e2e --config C3 --steps 1 --warmup 1 > /dev/null 2>&1
