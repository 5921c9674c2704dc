timeout -s KILL 120 python tools/dbg_small.py 2>&1 | tail -2
timeout -s KILL 120 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 3 2>&1 | tail -1
timeout -s KILL 120 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 3 --flags 32 2>&1 | tail -1
timeout -s KILL 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --reps 2 2>&1 | tail -1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -3
