timeout -s KILL 120 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 3 2>&1 | tail -1
timeout -s KILL 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --reps 2 2>&1 | tail -1
for f in 256 0; do
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/l_$f.csv python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 --flags $f > /dev/null 2>&1
done
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "two_pass or identical" 2>&1 | tail -2
