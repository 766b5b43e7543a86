# compute-sanitizer gates (each bounded); DESC_DYN_MIN=1 forces the dynamic tile scheduler
for t in racecheck synccheck memcheck initcheck; do
  DESC_DYN_MIN=1 DESC_SCAN_SINGLE_MAX_TILES=2 timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_driver.py > gpurun_out/sanitizer_$t.log 2>&1; echo "$t rc=$?"; grep -E "SUMMARY|Race reported|Error" gpurun_out/sanitizer_$t.log | head -3
done
