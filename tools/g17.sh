for m in 4 6 8 16 64 100000; do echo "grid mult $m"; TOD_RR_GRID=$m timeout -s KILL 120 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 3 2>&1 | tail -1; done
