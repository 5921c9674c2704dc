# Hand-off wait: suspend (default) vs poll (TOD_SPIN=1), per main kernel.
O=gpurun_out/f; mkdir -p $O
for sp in 0 1; do
  echo "== spin $sp c2 tc3"; TOD_SPIN=$sp TOD_MAIN_RING3=0 timeout 300 python tools/prof_knn.py --n 100000 --d 32 --k 20 --fmt fp16 --reps 4 2>&1 | tail -1
  echo "== spin $sp c2 tc5"; TOD_SPIN=$sp TOD_MAIN_RING3=1 timeout 300 python tools/prof_knn.py --n 100000 --d 32 --k 20 --fmt fp16 --reps 4 2>&1 | tail -1
  echo "== spin $sp c3 tc4"; TOD_SPIN=$sp timeout 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 3 2>&1 | tail -1
done
TOD_SPIN=1 TOD_MAIN_RING3=0 timeout 300 python tools/trace_main.py > $O/trace_c2_tc3_spin.txt 2>&1; cat $O/trace_c2_tc3_spin.txt
TOD_SPIN=1 TOD_MAIN_RING3=1 timeout 300 python tools/trace_main.py > $O/trace_c2_tc5_spin.txt 2>&1; cat $O/trace_c2_tc5_spin.txt
