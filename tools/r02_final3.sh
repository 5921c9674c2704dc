# Round-2 closing evidence at HEAD (a171e97+): full GPU suite, smoke, all bench lines, C5/C4 launch share.
O=gpurun_out/final3; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.txt
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 -rf > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench_c3_line.json 2> $O/bench_c3.err; head -c 200 $O/bench_c3_line.json; echo
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > $O/bench_c2_line.json 2> $O/bench_c2.err; head -c 200 $O/bench_c2_line.json; echo
timeout 1200 python bench.py --config c4 --steps 3 --warmup 3 > $O/bench_c4_line.json 2> $O/bench_c4.err; head -c 200 $O/bench_c4_line.json; echo
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 > $O/bench_c5_line.json 2> $O/bench_c5.err; head -c 200 $O/bench_c5_line.json; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref_line.json 2> /dev/null; head -c 200 $O/bench_ref_line.json; echo
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5_bench.csv python bench.py --config c5 --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
du -sh $O
