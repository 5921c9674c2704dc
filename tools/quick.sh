#!/bin/bash
# Quick GPU check: parity tests + main-kernel timings at C2 / C3 shapes.
set -o pipefail
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -2
summ() { python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); print('$1', 'cert', d['certified'], 'fb', d['fallback_rows'], 'kp', d['kprime'], 'S', d['chunks'], 'prep %.2f main %.2f cert %.2f fb %.2f' % (d['ms_prep'], d['ms_main'], d['ms_certify'], d['ms_fallback']))"; }
for sp in 1 2; do
python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 3 --split $sp 2>&1 | summ "C2 split=$sp"
python tools/prof_knn.py --n 1000000 --d 64 --k 10 --reps 2 --split $sp 2>&1 | summ "C3f16 split=$sp"
done
python tools/prof_knn.py --n 1000000 --d 64 --k 10 --reps 1 --split 1 --kprime 24 2>&1 | summ "C3 kp=24 split=1"
