# compute-sanitizer over the hot-path launches (memcheck, racecheck, synccheck, initcheck)
mkdir -p gpurun_out
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 --error-exitcode 9 python scripts/sanitize.py > gpurun_out/sanitizer_$t.txt 2>&1
  echo "$t exit=$?" | tee -a gpurun_out/sanitizer_summary.txt
  tail -3 gpurun_out/sanitizer_$t.txt >> gpurun_out/sanitizer_summary.txt
done
