# A/B: alternating filter groups in knn_tc3 (warps 0-7 even tiles, 8-15 odd tiles, 128 columns each).
O=gpurun_out/w; mkdir -p $O
for rep in 1 2 3; do
  TOD_MAIN_RING3=0 timeout 300 python tools/ab_lib.py abl/base_libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
  timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
done
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > $O/pytest_parity.txt 2>&1; tail -3 $O/pytest_parity.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc3 --launch-skip 1 -c 1 -o $O/knn_tc3_c2 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 > /dev/null 2>&1
ls $O
