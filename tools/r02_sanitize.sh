mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  for case in knn fallback lof nwr ring; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py $case > gpurun_out/san/${tool}_${case}.txt 2>&1
    echo "$tool $case rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/${tool}_${case}.txt | tail -1)"
  done
done
