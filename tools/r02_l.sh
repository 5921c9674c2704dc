# Three-stage candidate selection at d = 64 (default) vs the list-based sample.
O=gpurun_out/l; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
for rep in 1 2; do
 for s3 in 1 0; do
  echo "== sample3 $s3 bf16"; TOD_SAMPLE3=$s3 timeout 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 2 2>&1 | tail -1
  echo "== sample3 $s3 fp16"; TOD_SAMPLE3=$s3 timeout 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt fp16 --reps 2 2>&1 | tail -1
 done
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > $O/bench_c3_line.json 2> $O/bench_c3.err; tail -c 1500 $O/bench_c3_line.json; tail -3 $O/bench_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1 > /dev/null 2>&1; python tools/launch_share.py $O/launches_c3.csv 1 | head -12
