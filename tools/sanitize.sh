# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_driver.py workloads
OUT=${OUT:-gpurun_out/sanitizer}
mkdir -p $OUT
python -m paper_2502_06798_b200.build > /dev/null
for tool in memcheck racecheck synccheck; do
  for wl in ${WORKLOADS:-c1 c1chain c2 dyn graph plan lru}; do
    timeout ${SAN_TIMEOUT:-600} compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 \
      python tools/sanitize_driver.py $wl > $OUT/${tool}_${wl}.log 2>&1
    echo "$tool $wl rc=$?" | tee -a $OUT/summary.txt
  done
done
