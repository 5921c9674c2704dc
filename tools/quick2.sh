#!/bin/bash
for sp in 1 2; do
for f in 0 1536 512 256; do
python tools/prof_knn.py --n 1000000 --d 64 --k 10 --reps 2 --split $sp --flags $f 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('split',$sp,'flags',$f,'main',round(d['ms_main'],1))"
done; done
