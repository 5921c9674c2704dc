# Re-rank per-column pre-bound: parity + A/B (TOD_RR_PREBOUND=0/1) at C2, C3 bf16, C3 fp16, d=128.
O=gpurun_out/pb; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_abi.py -m gpu -x -q -p no:cacheprovider > $O/pytest_parity.txt 2>&1; tail -3 $O/pytest_parity.txt
for rep in 1 2; do
  TOD_RR_PREBOUND=0 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
  timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
done
for f in bf16 fp16; do
  TOD_RR_PREBOUND=0 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 1000000 --d 64 --k 10 --fmt $f --reps 2 2>&1 | tail -1
  timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 1000000 --d 64 --k 10 --fmt $f --reps 2 2>&1 | tail -1
done
TOD_RR_PREBOUND=0 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 128 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 128 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
timeout -s KILL 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "c3 or c2" > $O/pytest_full.txt 2>&1; tail -3 $O/pytest_full.txt
