summ() { python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); print('$1', 'cert', d['certified'], 'fb', d['fallback_rows'], 'kp', d['kprime'], 'S', d['chunks'], 'prep %.3f main %.3f cert %.3f fb %.3f' % (d['ms_prep'], d['ms_main'], d['ms_certify'], d['ms_fallback']))" 2>&1 | tail -1; }
timeout -s KILL 300 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 3 2>&1 | summ "C2 2p"
timeout -s KILL 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --reps 2 2>&1 | summ "C3 2p"
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -3
