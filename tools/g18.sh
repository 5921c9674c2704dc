for v in 0 1; do echo "SAMPLE_V1=$v"
TOD_SAMPLE_V1=$v timeout -s KILL 120 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 3 > gpurun_out/c2.txt 2>&1; tail -1 gpurun_out/c2.txt
TOD_SAMPLE_V1=$v timeout -s KILL 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --reps 2 2>&1 | tail -1
done
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -2
