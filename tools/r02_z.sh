# Round-2 final evidence at HEAD: GPU tests, smoke, bench lines (C3 default, C2, C4 shard, C5), launch lists, main-kernel captures.
O=gpurun_out/z; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.txt
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 -rf > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench_c3_line.json 2> $O/bench_c3.err; head -c 300 $O/bench_c3_line.json; echo
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > $O/bench_c2_line.json 2> $O/bench_c2.err; head -c 300 $O/bench_c2_line.json; echo
timeout 1200 python bench.py --config c4 --steps 3 --warmup 3 > $O/bench_c4_line.json 2> $O/bench_c4.err; head -c 300 $O/bench_c4_line.json; echo
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 > $O/bench_c5_line.json 2> $O/bench_c5.err; head -c 300 $O/bench_c5_line.json; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref_line.json 2> /dev/null; head -c 300 $O/bench_ref_line.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_bench.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc4 -c 1 -o $O/knn_tc4_c3bf16 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc3 --launch-skip 1 -c 1 -o $O/knn_tc3_c2 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rerank_groups -c 1 -o $O/rerank_c3 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1 > /dev/null 2>&1
ls $O
