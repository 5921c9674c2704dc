summ() { python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); print('$1', 'cert', d['certified'], 'fb', d['fallback_rows'], 'kp', d['kprime'], 'S', d['chunks'], 'prep %.2f main %.2f cert %.2f fb %.2f' % (d['ms_prep'], d['ms_main'], d['ms_certify'], d['ms_fallback']))"; }
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -2
for sp in 1 2; do python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 3 --split $sp | summ "C2 BN64 split=$sp"; done
TOD_TRACE_FILE=gpurun_out/trace_c2.bin python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 --flags 2048 | tail -1
