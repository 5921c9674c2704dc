# Round-2 closing check at HEAD: full GPU suite, smoke, C3 default line, C5 line.
O=gpurun_out/final2; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.txt
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 -rf > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench_c3_line.json 2> $O/bench_c3.err; head -c 200 $O/bench_c3_line.json; echo
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 > $O/bench_c5_line.json 2> $O/bench_c5.err; head -c 200 $O/bench_c5_line.json; echo
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > $O/bench_c2_line.json 2> $O/bench_c2.err; head -c 200 $O/bench_c2_line.json; echo
du -sh $O
