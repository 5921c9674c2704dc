summ() { python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); print('$1', 'cert', d['certified'], 'fb', d['fallback_rows'], 'kp', d['kprime'], 'S', d['chunks'], 'prep %.3f main %.3f cert %.3f fb %.3f' % (d['ms_prep'], d['ms_main'], d['ms_certify'], d['ms_fallback']))"; }
for sp in 1 2 4; do
for f in 0 256; do
python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 3 --split $sp --flags $f 2>&1 | summ "C2 split=$sp flags=$f"
done
python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 3 --split $sp --chunks 1 2>&1 | summ "C2 split=$sp S=1"
done
for sp in 1 2 4; do
TOD_TRACE_FILE=gpurun_out/trace_sp$sp.bin python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 --split $sp --flags 2048 2>&1 | summ "trace sp$sp"
python tools/trace_analyze.py gpurun_out/trace_sp$sp.bin
done
