# Re-rank spatial row order: A/B (TOD_RR_ORDER=0/1) at C3 bf16/fp16, C2, d=128; parity.
O=gpurun_out/ord; mkdir -p $O
for f in bf16 fp16; do
  TOD_RR_ORDER=0 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 1000000 --d 64 --k 10 --fmt $f --reps 2 2>&1 | tail -1
  timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 1000000 --d 64 --k 10 --fmt $f --reps 2 2>&1 | tail -1
done
for rep in 1 2; do
  TOD_RR_ORDER=0 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
  TOD_RR_ORDER=1 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
done
TOD_RR_ORDER=0 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 128 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 128 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
timeout -s KILL 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "c3 or c2" > $O/pytest_full.txt 2>&1; tail -3 $O/pytest_full.txt
