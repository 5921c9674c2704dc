# K-pipelined CTA-pair main pass (dpad > 64): parity, then A/B against the single-SM K-pipelined pass at the C5 shape.
O=gpurun_out/kp; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "kpipelined or high_dimensional" > $O/pytest_kp.txt 2>&1; tail -5 $O/pytest_kp.txt
for rep in 1 2; do
  TOD_MAIN_PAIR=0 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
  TOD_MAIN_PAIR=1 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
done
TOD_MAIN_PAIR=0 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 128 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
TOD_MAIN_PAIR=1 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 128 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
TOD_MAIN_PAIR=0 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 256 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
TOD_MAIN_PAIR=1 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 256 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
