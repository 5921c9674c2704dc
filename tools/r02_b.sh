# Filter rewrite (part-min vote) check: parity, phase timings, micro-benchmarks.
O=gpurun_out/b; mkdir -p $O
timeout 120 ./build/mma_bench > $O/mma_bench.txt 2>&1; cat $O/mma_bench.txt
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
for f in "--n 100000 --d 32 --k 20 --fmt fp16 --reps 4" "--n 1000000 --d 64 --k 10 --fmt bf16 --reps 3" "--n 1000000 --d 64 --k 10 --fmt fp16 --reps 3"; do
  echo "== $f"; timeout 300 python tools/prof_knn.py $f 2>&1 | tail -2; done
for v in "TOD_SAMPLE_R=16" "TOD_SAMPLE_V1=0"; do
  echo "== bf16 $v"; env $v timeout 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 3 2>&1 | tail -1
done
timeout 300 python tools/dbg_modes.py > $O/dbg_modes_c2.txt 2>&1; cat $O/dbg_modes_c2.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $O/bench_c3_line.json 2> $O/bench_c3.err; tail -c 1500 $O/bench_c3_line.json
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu > $O/bench_c2_line.json 2> $O/bench_c2.err; tail -c 600 $O/bench_c2_line.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc4 -c 1 -o $O/knn_tc4_c3bf16 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc3 --launch-skip 1 -c 1 -o $O/knn_tc3_c2 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 > /dev/null 2>&1
ls $O
