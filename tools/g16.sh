for cfg in "8 8" "16 8" "16 4" "32 4"; do set -- $cfg
echo "R=$1 KR=$2"; TOD_SAMPLE_R=$1 TOD_SAMPLE_KR=$2 timeout -s KILL 120 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 3 2>&1 | tail -1
TOD_SAMPLE_R=$1 TOD_SAMPLE_KR=$2 timeout -s KILL 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --reps 2 2>&1 | tail -1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_prep.csv python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 > /dev/null 2>&1
