# knn_tc5 (3-deep accumulator ring): parity, timing, trace.
O=gpurun_out/e; mkdir -p $O
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ring3 or two_pass" > $O/pytest_ring3.txt 2>&1; tail -5 $O/pytest_ring3.txt
for f in "--n 100000 --d 32 --k 20 --fmt fp16 --reps 4"; do
  echo "== $f"; timeout 300 python tools/prof_knn.py $f 2>&1 | tail -1
  echo "== ring3=0 $f"; TOD_MAIN_RING3=0 timeout 300 python tools/prof_knn.py $f 2>&1 | tail -1; done
echo "== c3 shape ring3 (key-only sample)"; TOD_MAIN_RING3=1 TOD_SAMPLE_V1=0 TOD_MAIN_PAIR=0 timeout 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 3 2>&1 | tail -1
TOD_MAIN_RING3=1 timeout 300 python tools/trace_main.py > $O/trace_c2.txt 2>&1; cat $O/trace_c2.txt
TOD_MAIN_RING3=1 TOD_SAMPLE_V1=0 timeout 300 python tools/trace_main.py --n 1000000 --d 64 --k 10 > $O/trace_c3.txt 2>&1; cat $O/trace_c3.txt
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu > $O/bench_c2_line.json 2> $O/bench_c2.err; tail -c 900 $O/bench_c2_line.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc5 -c 1 -o $O/knn_tc5_c2 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 > /dev/null 2>&1
ls $O
