# A/B: A-in-TMEM K2 (default build) vs the SS K2 (PAS_K2_ATMEM=0), same box, back to back.
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/t.log 2>&1; echo "tests rc=$?" >> gpurun_out/t.log
L=$PWD/paper_2502_06798_b200/lib
for rep in 1 2; do
  for c in C4 C2; do
    timeout 600 python bench.py --config $c --steps 8 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ab_ta_${c}_$rep.json 2>/dev/null
    PAS_LIB=$L/libpas_ss.so timeout 600 python bench.py --config $c --steps 8 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ab_ss_${c}_$rep.json 2>/dev/null
  done
done
