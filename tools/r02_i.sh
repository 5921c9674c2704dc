# Column candidates: parity + timings.
O=gpurun_out/i; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; tail -5 $O/pytest.txt
for cm in 1 0; do
 for f in "--n 1000000 --d 64 --k 10 --fmt bf16 --reps 3" "--n 1000000 --d 64 --k 10 --fmt fp16 --reps 2" "--n 500000 --d 512 --k 50 --fmt fp16 --reps 2"; do
  echo "== colmode $cm $f"; TOD_COLMODE=$cm timeout 300 python tools/prof_knn.py $f 2>&1 | tail -1; done
done
timeout -s KILL 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > $O/pytest_full.txt 2>&1; tail -3 $O/pytest_full.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > $O/bench_c3_line.json 2> $O/bench_c3.err; tail -c 1200 $O/bench_c3_line.json
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu > $O/bench_c5_line.json 2> $O/bench_c5.err; tail -c 800 $O/bench_c5_line.json
