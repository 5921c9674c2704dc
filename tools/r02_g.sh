# Finer main-pass trace (16 stamps per tile); fp16 second tier; tc5 parity.
O=gpurun_out/g; mkdir -p $O
TOD_MAIN_RING3=0 timeout 300 python tools/trace_main.py > $O/trace_c2_tc3.txt 2>&1; cat $O/trace_c2_tc3.txt
TOD_MAIN_RING3=1 timeout 300 python tools/trace_main.py > $O/trace_c2_tc5.txt 2>&1; cat $O/trace_c2_tc5.txt
TOD_MAIN_RING3=0 TOD_SAMPLE_V1=0 timeout 300 python tools/trace_main.py --n 1000000 --d 64 --k 10 > $O/trace_c3_tc3.txt 2>&1; cat $O/trace_c3_tc3.txt
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "second_tier or ring3" > $O/pytest.txt 2>&1; tail -5 $O/pytest.txt
echo "== c5s"; timeout 300 python tools/prof_knn.py --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
echo "== c2"; timeout 300 python tools/prof_knn.py --n 100000 --d 32 --k 20 --fmt fp16 --reps 3 2>&1 | tail -1
