# Staging drops appends >= vmin; chunk size A/B; bench lines.
O=gpurun_out/m; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
for mb in 48 24 16; do
  echo "== chunk $mb bf16"; TOD_MAIN_CHUNK_MB=$mb timeout 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 2 2>&1 | tail -1
done
echo "== c3 fp16"; timeout 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt fp16 --reps 2 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > $O/bench_c3_line.json 2> $O/bench_c3.err; tail -c 1200 $O/bench_c3_line.json
timeout 1200 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > $O/bench_c4_line.json 2> $O/bench_c4.err; tail -c 900 $O/bench_c4_line.json; tail -2 $O/bench_c4.err
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu > $O/bench_c2_line.json 2> $O/bench_c2.err; tail -c 600 $O/bench_c2_line.json
