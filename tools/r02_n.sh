# After removing trace/spin/stagger code from production kernels: parity, timings, tc4 trace.
O=gpurun_out/n; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
for f in "--n 100000 --d 32 --k 20 --fmt fp16 --reps 4" "--n 1000000 --d 64 --k 10 --fmt bf16 --reps 2" "--n 500000 --d 512 --k 50 --fmt fp16 --reps 2"; do
  echo "== $f"; timeout 300 python tools/prof_knn.py $f 2>&1 | tail -1; done
timeout 300 python tools/dbg_modes.py > $O/dbg_modes_c2.txt 2>&1; cat $O/dbg_modes_c2.txt
TOD_MAIN_PAIR=1 timeout 300 python tools/trace_main.py --n 1000000 --d 64 --k 10 --fmt bf16 > $O/trace_c3_tc4.txt 2>&1; cat $O/trace_c3_tc4.txt
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu > $O/bench_c2_line.json 2> $O/bench_c2.err; tail -c 700 $O/bench_c2_line.json
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > $O/bench_c3_line.json 2> $O/bench_c3.err; tail -c 700 $O/bench_c3_line.json
