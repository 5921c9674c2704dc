summ() { python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); print('$1', 'cert', d['certified'], 'fb', d['fallback_rows'], 'kp', d['kprime'], 'main %.2f cert %.2f' % (d['ms_main'], d['ms_certify']))"; }
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -2
for sp in 4 2; do
python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 3 --split $sp | summ "C2 sp$sp"
python tools/prof_knn.py --n 1000000 --d 64 --k 10 --reps 1 --split $sp | summ "C3 sp$sp"
done
