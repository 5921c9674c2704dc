# Re-entry (session 3): GPU tests, smoke, bench lines at HEAD, C3 launch list, sanitizers.
O=gpurun_out/p; mkdir -p $O $O/san
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.txt
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 -rf > $O/pytest_gpu.txt 2>&1; tail -25 $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench_c3_line.json 2> $O/bench_c3.err; tail -c 2500 $O/bench_c3_line.json; tail -3 $O/bench_c3.err
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > $O/bench_c2_line.json 2> $O/bench_c2.err; tail -c 1500 $O/bench_c2_line.json
timeout 1200 python bench.py --config c4 --steps 3 --warmup 3 > $O/bench_c4_line.json 2> $O/bench_c4.err; tail -c 600 $O/bench_c4_line.json; tail -3 $O/bench_c4.err
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 > $O/bench_c5_line.json 2> $O/bench_c5.err; tail -c 600 $O/bench_c5_line.json; tail -3 $O/bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
for tool in memcheck synccheck racecheck; do
  for case in knn fallback lof nwr ring; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py $case > $O/san/${tool}_${case}.txt 2>&1
    echo "$tool $case rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/san/${tool}_${case}.txt | tail -1)"
  done
done
ls -la $O
