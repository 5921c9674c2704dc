# Round-2 re-entry: full GPU test suite, smoke, bench lines per config, launch list and main-kernel capture.
O=gpurun_out/a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.txt
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 -rf > $O/pytest_gpu.txt 2>&1; tail -25 $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench_c3_line.json 2> $O/bench_c3.err; tail -c 2500 $O/bench_c3_line.json; tail -3 $O/bench_c3.err
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > $O/bench_c2_line.json 2> $O/bench_c2.err; tail -c 400 $O/bench_c2_line.json
timeout 1200 python bench.py --config c4 --steps 3 --warmup 3 > $O/bench_c4_line.json 2> $O/bench_c4.err; tail -c 400 $O/bench_c4_line.json; tail -3 $O/bench_c4.err
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 > $O/bench_c5_line.json 2> $O/bench_c5.err; tail -c 400 $O/bench_c5_line.json; tail -3 $O/bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc4 -c 1 -o $O/knn_tc4_c3bf16 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc3 --launch-skip 1 -c 1 -o $O/knn_tc3_c2 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 > /dev/null 2>&1
ls -la $O
