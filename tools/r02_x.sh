# A/B: alternating filter groups + pipelined 16-column TMEM reads in knn_tc3.
O=gpurun_out/x; mkdir -p $O
for rep in 1 2 3; do
  TOD_MAIN_RING3=0 timeout 300 python tools/ab_lib.py abl/base_libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
  timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
done
TOD_MAIN_RING3=0 timeout 300 python tools/trace_main.py --n 100000 --d 32 --k 20 2>&1 | tail -16
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > $O/pytest_parity.txt 2>&1; tail -3 $O/pytest_parity.txt
