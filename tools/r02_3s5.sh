# Three-stage selection for dpad > 64 on the K-pipelined pair (TOD_SAMPLE3=1) vs the key-only sample pass.
for rep in 1 2; do
  TOD_SAMPLE3=0 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
  TOD_SAMPLE3=1 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
done
TOD_SAMPLE3=0 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 128 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
TOD_SAMPLE3=1 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 128 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
TOD_SAMPLE3=1 timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "kpipelined or high_dimensional" 2>&1 | tail -2
