for R in 8 16 32; do
echo "R=$R"; TOD_SAMPLE_R=$R timeout -s KILL 300 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 3 2>&1 | tail -1
TOD_SAMPLE_R=$R timeout -s KILL 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --reps 2 2>&1 | tail -1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_null.csv python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 2 --flags 256 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_null2.csv python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 2 --flags 512 > /dev/null 2>&1
