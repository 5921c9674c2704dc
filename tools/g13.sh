for f in 256 288 512 544; do
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/l_$f.csv python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 --flags $f > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc4 -c 1 -o gpurun_out/knn_tc4_c2 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 > /dev/null 2>&1
